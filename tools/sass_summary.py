#!/usr/bin/env python
"""Per-kernel SASS instruction counts of libsrpb.so (profiles/r2_sass_summary.txt):
python tools/sass_summary.py [lib]"""
import re
import subprocess
import sys

COLS = [("UTC", r"\bUTC\w*MMA\b"), (".2CTA", r"\bUTC\w*MMA\.2CTA\b"), ("UTMALDG", r"\bUTMALDG\b"),
        ("UTMASTG", r"\bUTMASTG\b"), ("LDTM", r"\bLDTM\b"), ("STTM", r"\bSTTM\b"),
        ("F*2", r"\b(FADD2|FMUL2|FFMA2)\b")]


def main(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs, name = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            name = m.group(1)
            funcs[name] = []
        elif name and re.search(r"/\*[0-9a-f]{4,}\*/", line):
            funcs[name].append(line)
    dem = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True,
                         text=True).stdout.splitlines()
    for (mangled, lines), d in sorted(zip(funcs.items(), dem), key=lambda x: x[1]):
        if not any(k in d for k in ("srp_tc_kernel", "lattice")):
            continue
        short = re.sub(r"\(.*", "", d).replace("srpb::", "")
        counts = [sum(1 for l in lines if re.search(rx, l)) for _, rx in COLS]
        print(f"{short:60s} {len(lines):6d} " + " ".join(f"{c:4d}" for c in counts))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2012_09499_b200/libsrpb.so")
