#!/usr/bin/env python
"""Stall-reason breakdown of an ncu source page grouped by execution count
(code regions that run the same number of times): stall_by_exec.py csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
ex = h.index("Instructions Executed")
agg = {}
for r in rows[2:]:
    try:
        e = int(r[ex])
    except (ValueError, IndexError):
        continue
    d = agg.setdefault(e, {k: 0.0 for k in reasons})
    for k in reasons:
        try:
            d[k] += float(r[h.index(k)])
        except ValueError:
            pass
tot_all = sum(sum(d.values()) for d in agg.values()) or 1
for e, d in sorted(agg.items(), key=lambda x: -sum(x[1].values()))[:int(sys.argv[2]) if len(sys.argv) > 2 else 6]:
    s = sum(d.values())
    top = sorted(d.items(), key=lambda x: -x[1])[:6]
    print(f"exec={e:>8d} {s / tot_all * 100:5.1f}%: " + ", ".join(f"{k[6:]} {v / s * 100:.0f}%" for k, v in top if v))
