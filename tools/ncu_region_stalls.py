#!/usr/bin/env python
"""Stall reasons of an ncu source page, aggregated per SASS address window
(execution-count groups) -- python tools/ncu_region_stalls.py rep [launch] [min_ex]"""
import csv
import subprocess
import sys

REASONS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_drain", "stall_lg",
           "stall_long_sb", "stall_math", "stall_membar", "stall_mio", "stall_misc", "stall_no_inst",
           "stall_not_selected", "stall_selected", "stall_short_sb", "stall_sleep", "stall_tex",
           "stall_wait"]


def main(path, idx=0, min_ex=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--launch-skip", str(idx),
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    ci = {r: h.index(r) for r in REASONS}
    ex, src, tot = h.index("Instructions Executed"), h.index("Source"), h.index(
        "Warp Stall Sampling (All Samples)")
    groups = {}
    total = 0.0
    for r in rows[2:]:
        try:
            e = int(float(r[ex]))
            s = float(r[tot])
        except (ValueError, IndexError):
            continue
        total += s
        if e < min_ex:
            continue
        g = groups.setdefault(e, {"n": 0, "samples": 0.0, **{k: 0.0 for k in REASONS}, "ops": {}})
        g["n"] += 1
        g["samples"] += s
        for k in REASONS:
            g[k] += float(r[ci[k]] or 0)
        op = r[src].strip().split()[0] if r[src].strip() else "?"
        if op.startswith("@"):
            op = r[src].strip().split()[1]
        op = op.split(".")[0]
        g["ops"][op] = g["ops"].get(op, 0) + 1
    print(f"total samples {total:.0f}")
    for e, g in sorted(groups.items(), key=lambda kv: -kv[1]["samples"])[:12]:
        top = sorted(((g[k], k) for k in REASONS), reverse=True)[:5]
        ops = sorted(g["ops"].items(), key=lambda kv: -kv[1])[:8]
        print(f"ex={e:>10d} lines={g['n']:5d} samples={g['samples'] / total * 100:5.1f}%  " +
              " ".join(f"{k[6:]}={v / total * 100:.1f}" for v, k in top))
        print("      ops: " + " ".join(f"{o}:{c}" for o, c in ops))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0,
         int(sys.argv[3]) if len(sys.argv) > 3 else 0)
