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


def c4_setup(F):
    """C4 shapes (32 mics, 496 pairs, 512 bins, N_aux 2): random spectra."""
    import numpy as np
    from paper_2012_09499_b200 import scenes
    from paper_2012_09499_b200.plan import SrpPlan

    rng = np.random.default_rng(np.random.SeedSequence([4, 0, 0]))
    box = np.array([6.0, 5.0, 3.0])
    mic = rng.uniform(0.0, 1.0, size=(32, 3)) * box
    grid = scenes.box_grid(120, 100, 50, box)[:4096]
    omega = 2.0 * np.pi * np.arange(512) * 16000.0 / 1024
    plan = SrpPlan.from_geometry(mic, grid, omega, speed_of_sound=343.0,
                                 sample_period=1 / 16000.0, n_aux=2, weights="onthefly",
                                 conventional=False)
    g = torch.Generator(device="cuda").manual_seed(0)
    Y = torch.complex(torch.randn((F, 32, 512), device="cuda", generator=g),
                      torch.randn((F, 32, 512), device="cuda", generator=g)).to(torch.complex64)
    return plan, Y


def main():
    dev = torch.device("cuda", 0)
    if len(sys.argv) > 1 and sys.argv[1] == "--c4":  # C4 shapes, random spectra
        for F in (int(x) for x in (sys.argv[2:] or ["320"])):
            plan, Y = c4_setup(F)
            ms = timeit(lambda: plan.lattice_from_spectra(Y, split="f16"), reps=5)
            print(f"C4 F={F}: lattice {ms * 1e3:.1f} us (tc={plan.lattice_tc}, L={plan.L})")
        return
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
