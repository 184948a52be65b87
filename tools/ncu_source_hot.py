#!/usr/bin/env python
"""Top SASS lines by warp-stall samples for one kernel of an .ncu-rep:
python tools/ncu_source_hot.py rep.ncu-rep <launch-index> [N]"""
import csv, subprocess, sys

def main(path, idx, n=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--launch-skip", str(idx),
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    print(rows[0][:2])
    h = rows[1]
    si, src, ex = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
    data = []
    for r in rows[2:]:
        try:
            data.append((float(r[si]), r[ex], r[src].strip(), r[0]))
        except (ValueError, IndexError):
            continue
    tot = sum(d[0] for d in data) or 1
    print(f"total samples {tot:.0f}, {len(data)} SASS lines")
    for s, e, line, addr in sorted(data, key=lambda d: -d[0])[:n]:
        print(f"{s / tot * 100:5.1f}%  ex={e:>10s}  {addr[-5:]}  {line[:95]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 40)
