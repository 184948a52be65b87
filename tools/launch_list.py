#!/usr/bin/env python
"""Summarise an ncu launch list (``ncu --metrics gpu__time_duration.sum --csv
--log-file X.csv ...``): per kernel, launches, mean/total duration and share
of the profiled time.  ncu times are cold-cache and serialised: compare the
SHARES with bench.py's live per-kernel times, not the absolute values."""
import collections
import csv
import sys


def main(path, skip=0):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
    agg = collections.OrderedDict()
    for r in rows[1 + skip:]:
        name = r[kn].split("(")[0].strip()
        try:
            us = float(r[mv].replace(",", "")) * scale.get(r[mu], 1.0)
        except ValueError:
            continue
        if us != us:  # nan: a launch ncu could not time
            continue
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    total = sum(t for _, t in agg.values())
    print(f"{'kernel':58s} {'launches':>8s} {'mean_us':>10s} {'total_us':>10s} {'share':>7s}")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[-58:]:58s} {n:8d} {t / n:10.2f} {t:10.2f} {100 * t / total:6.1f}%")
    print(f"{'total':58s} {sum(n for n, _ in agg.values()):8d} {'':10s} {total:10.2f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
