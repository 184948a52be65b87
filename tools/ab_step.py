#!/usr/bin/env python
"""A/B of the approx graph step under environment toggles, same process
family and box: python tools/ab_step.py VAR=1 [VAR2=1 ...] (each arg = one
extra variant; the baseline runs first and last)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline",
                          "--steps", "20"], capture_output=True, text=True, env=env).stdout
    d = json.loads(out.strip().splitlines()[-1])
    return d["ms_per_step"] * 1e3, d["roofline"]["kernels_ms"], d["conventional"]["ms_per_step"]


variants = [{}] + [dict([a.split("=", 1)]) for a in sys.argv[1:]] + [{}]
for v in variants:
    ms, k, conv = run(v)
    print(f"{str(v):40s} approx {ms:7.2f} us  conv {conv:6.3f} ms  "
          + "  ".join(f"{n}={t * 1e3:.1f}us" for n, t in k.items()))
