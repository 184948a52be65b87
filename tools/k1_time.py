#!/usr/bin/env python
"""K1 (GCC-PHAT) timing at C4 (4096 frames x 32 mics x 512 bins, 496 pairs):
psi complex64 and the fp16 operand split, achieved HBM bandwidth."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_09499_b200 import _native as N  # noqa: E402


def main():
    sc = bench.c4_scene(4096)
    plan = bench.build_plan(sc, 2, torch.device("cuda", 0), conventional=False)
    Y = torch.from_numpy(sc.Y).cuda()
    F, P, Kb = Y.shape[0], plan.P, plan.Kb
    psi = torch.empty((F, P, Kb), dtype=torch.complex64, device="cuda")
    fl = torch.empty(F, dtype=torch.float64, device="cuda")
    hi = torch.empty((F, 2 * P * Kb), dtype=torch.float16, device="cuda")
    lo = torch.empty_like(hi)
    byts = F * 32 * Kb * 8 + F * P * Kb * 8
    for name, args in (("psi", ("srpb_gcc_phat", N.ptr(Y), F, 32, Kb, N.ptr(plan.pair_m),
                                N.ptr(plan.pair_mp), P, 0, 1e-12, -1.0, N.ptr(psi), N.ptr(fl),
                                N.stream_handle())),
                       ("split16", ("srpb_gcc_phat_split16", N.ptr(Y), F, 32, Kb,
                                    N.ptr(plan.pair_m), N.ptr(plan.pair_mp), P, 0, 1e-12, -1.0,
                                    None, N.ptr(hi), N.ptr(lo), 16384.0, N.ptr(fl),
                                    N.stream_handle()))):
        N.call(*args)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            N.call(*args)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / 5
        print(f"K1 {name:8s} C4: {ms:.3f} ms  {byts / ms / 1e9:.2f} TB/s "
              f"({byts / ms / 1e9 / 6.5475:.2f} of HBM)")


if __name__ == "__main__":
    main()
