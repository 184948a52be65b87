#!/usr/bin/env python
"""C4 (BASELINE configs[3]) stage timings: M=32 random mics in a 6x5x3 m
room (scenes.make_c4 geometry), 120x100x50 grid (J=600k), N=1024 (Kb=512),
N_aux=2.  Random unit-variance spectra stand in for the scene (timing only).

  python tools/c4_probe.py [--frames F] [--cands J] [--conv-cands Jc]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_09499_b200 import scenes  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402


def timeit(fn, reps=3):
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=320)
    ap.add_argument("--cands", type=int, default=600000)
    ap.add_argument("--conv-cands", type=int, default=40000)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--kbg", type=int, default=None, help="K blocks per accumulator group (K4; default: the plan's)")
    args = ap.parse_args()
    rng = np.random.default_rng(np.random.SeedSequence([4, 0, 0]))
    box = np.array([6.0, 5.0, 3.0])
    mic = rng.uniform(0.0, 1.0, size=(32, 3)) * box
    grid = scenes.box_grid(120, 100, 50, box)[: args.cands]
    omega = 2.0 * np.pi * np.arange(512) * 16000.0 / 1024
    t0 = time.perf_counter()
    plan = SrpPlan.from_geometry(mic, grid, omega, speed_of_sound=343.0,
                                 sample_period=1 / 16000.0, n_aux=2, weights="onthefly",
                                 conventional=False, interp_kb_per_group=args.kbg)
    torch.cuda.synchronize()
    print(f"plan: J={plan.J} P={plan.P} L={plan.L} total={plan.total_samples} "
          f"T_pad={plan.T_pad} build {time.perf_counter() - t0:.2f} s", flush=True)
    F = args.frames
    g = torch.Generator(device="cuda").manual_seed(0)
    Y = torch.complex(torch.randn((F, 32, 512), device="cuda", generator=g),
                      torch.randn((F, 32, 512), device="cuda", generator=g))
    Y = Y.to(torch.complex64)
    ms = timeit(lambda: plan.lattice_from_spectra(Y, split="f16"), args.reps)
    print(f"lattice (F={F}): {ms:.3f} ms  tc={plan.lattice_tc}", flush=True)
    xh, xl = plan.lattice_from_spectra(Y, split="f16")
    flops = 2.0 * plan.total_samples * F * plan.J
    for maps in (False, True):
        out = torch.empty((F, plan.J), dtype=torch.float32, device="cuda") if maps else None
        ms = timeit(lambda: plan._approx_tc16(xh, xl, out), args.reps)
        print(f"K4 onthefly maps={maps} F={F} J={plan.J}: {ms:.2f} ms  "
              f"{F * plan.J / ms * 1e3:.3e} f.c/s  {flops / ms / 1e9:.1f} TF/s "
              f"({flops / ms / 1e9 / (1616.9 / 3):.3f} of 3xFP16)", flush=True)
        del out
    if args.conv_cands:
        cp = SrpPlan.from_geometry(mic, grid[: args.conv_cands], omega, speed_of_sound=343.0)
        ms = timeit(lambda: cp.run(Y, "conventional", maps=False), 1)
        fl = 4.0 * cp.P * 512 * F * cp.J
        print(f"conventional F={F} J={cp.J}: {ms:.2f} ms  {F * cp.J / ms * 1e3:.3e} f.c/s "
              f"{fl / ms / 1e9:.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
