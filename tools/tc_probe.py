#!/usr/bin/env python
"""Per-role cycle breakdown of the tcgen05 kernels (instrumentation build).

    make prof && python tools/tc_probe.py

Loads libsrpb_prof.so (compiled with -DSRPB_TC_PROFILE) instead of the
product library and reports, per kernel, where the MMA issuer, the TMA
producer and the epilogue/generator warps spend their cycles (sums over
CTAs; divide by the CTA count for per-CTA figures).
"""

import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_09499_b200 import _native  # noqa: E402

lib = _native.load(os.path.join(ROOT, "paper_2012_09499_b200", "libsrpb_prof.so"))
lib.srpb_tc_profile_read.argtypes = [ctypes.c_void_p]

import bench  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402

NAMES = {0: "mma_total", 1: "mma_wait_full", 2: "mma_wait_acc_empty", 3: "tma_wait_empty",
         4: "tma_total", 5: "epi_gen_wait_empty", 6: "epi_gen", 7: "epi_drain", 9: "epi_write",
         10: "epi_total", 11: "ctas"}


def read():
    buf = (ctypes.c_ulonglong * 16)()
    assert lib.srpb_tc_profile_read(ctypes.addressof(buf)) == 0
    return list(buf)


def report(tag, c):
    n = max(c[11], 1)
    print(f"== {tag}: {n} CTAs; per-CTA cycles:")
    for i, name in NAMES.items():
        if i == 11:
            continue
        print(f"   {name:22s} {c[i] / n:14.0f}   ({c[i] / max(c[0], 1) * 100:5.1f}% of mma_total)")


def main():
    scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=bench.N_AUX,
                   weights="stored")
    Y = torch.from_numpy(scene.Y).cuda()
    for path in ("approx", "conventional"):
        plan.run(Y, path)  # warm
        torch.cuda.synchronize()
        read()
        plan.run(Y, path)
        torch.cuda.synchronize()
        report(path, read())


if __name__ == "__main__":
    main()
