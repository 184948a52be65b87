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
         4: "tma_total", 5: "epi_gen_wait_empty", 6: "epi_gen", 7: "epi_drain", 8: "staged_argmax", 9: "epi_write",
         10: "epi_total", 11: "ctas", 12: "write_loop", 13: "write_flush|staged_sts", 14: "write_stores|staged_wait",
         15: "write_argmax", 16: "cta_lifetime(all CTAs)", 17: "setup(all CTAs)",
         18: "teardown_wait(all CTAs)", 19: "cta_count"}


def read():
    buf = (ctypes.c_ulonglong * 24)()
    assert lib.srpb_tc_profile_read(ctypes.addressof(buf)) == 0
    return list(buf)


def report(tag, c):
    n = max(c[11], 1)
    M = (1 << 64) - 1
    first_in, last_out = M - c[20], c[21]
    first_out, last_in = M - c[22], c[23]
    print(f"== {tag}: CTA span {(last_out - first_in) / 1e3:.1f} us (globaltimer); entries spread "
          f"{(last_in - first_in) / 1e3:.1f} us, exits spread {(last_out - first_out) / 1e3:.1f} us")
    print(f"== {tag}: {n} CTAs; per-CTA cycles:")
    for i, name in NAMES.items():
        if i in (11, 19, 20, 21, 22, 23):
            continue
        d = max(c[19], 1) if i in (16, 17, 18) else n
        print(f"   {name:24s} {c[i] / d:14.0f}   ({c[i] / d / max(c[0] / n, 1) * 100:5.1f}% of mma_total)")


def main():
    scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
    kbg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=bench.N_AUX,
                   weights=os.environ.get("SRPB_WEIGHTS", "stored"), kb_per_group=kbg)
    Y = torch.from_numpy(scene.Y).cuda()
    paths = sys.argv[2].split(",") if len(sys.argv) > 2 else ["approx", "conventional"]
    for path in paths:
        plan.run(Y, path)  # warm
        torch.cuda.synchronize()
        read()
        plan.run(Y, path)
        torch.cuda.synchronize()
        report(f"{path} kb_per_group={kbg}", read())


if __name__ == "__main__":
    main()
