#!/usr/bin/env python
"""Fused lattice (GCC-PHAT + lattice IDFT, fp16-split output) timing on the
C2 (N_aux 4) and C3 (N_aux 0 / 8) workloads: SRPB_LIB selects the library."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_09499_b200 import scenes  # noqa: E402


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    dev = torch.device("cuda", 0)
    for name, sc, naux in (("C2", scenes.make_c2(), 4), ("C3", scenes.make_c3(), 0),
                           ("C3", None, 8)):
        sc = sc if sc is not None else last
        last = sc
        plan = bench.build_plan(sc, naux, dev, weights="onthefly", conventional=False)
        Y = torch.from_numpy(sc.Y).to(dev)
        ms = timeit(lambda: plan.lattice_from_spectra(Y, split="f16"))
        print(f"{name} N_aux {naux}: lattice {ms * 1e3:.1f} us (tc={plan.lattice_tc}, "
              f"F={Y.shape[0]}, P={plan.P}, L={plan.L})")


if __name__ == "__main__":
    main()
