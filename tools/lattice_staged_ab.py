#!/usr/bin/env python
"""C4 lattice: fused (PHAT formed per half-lag group inside the lattice,
speculative floor) vs staged (K1 writes psi once, the lattice streams it),
F frames of random spectra, CUDA events.  python tools/lattice_staged_ab.py [F]"""
import os
import sys

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
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 320
    rng = np.random.default_rng(np.random.SeedSequence([4, 0, 0]))
    box = np.array([6.0, 5.0, 3.0])
    mic = rng.uniform(0.0, 1.0, size=(32, 3)) * box
    grid = scenes.box_grid(120, 100, 50, box)[:1024]
    omega = 2.0 * np.pi * np.arange(512) * 16000.0 / 1024
    plan = SrpPlan.from_geometry(mic, grid, omega, speed_of_sound=343.0,
                                 sample_period=1 / 16000.0, n_aux=2, weights="onthefly",
                                 conventional=False)
    g = torch.Generator(device="cuda").manual_seed(0)
    Y = torch.complex(torch.randn((F, 32, 512), device="cuda", generator=g),
                      torch.randn((F, 32, 512), device="cuda", generator=g)).to(torch.complex64)
    fused = timeit(lambda: plan.lattice_from_spectra(Y, split="f16"))
    psi, _ = plan.cross_spectra(Y)
    k1 = timeit(lambda: plan.cross_spectra(Y))
    lat = timeit(lambda: plan.lattice(psi))
    xi = plan.lattice(psi)
    sp = timeit(lambda: plan.split_f16(xi, plan.xi_scale16))
    print(f"F={F}: fused {fused:.3f} ms | staged: K1 psi {k1:.3f} + lattice {lat:.3f} + split "
          f"{sp:.3f} = {k1 + lat + sp:.3f} ms")
    xh, xl = plan.lattice_from_spectra(Y, split="f16")
    a = xh.float() + xl.float()
    sh, sl = plan.split_f16(xi, plan.xi_scale16)
    b = sh.float() + sl.float()
    print("max rel diff fused vs staged:", float((a - b).abs().max() / a.abs().max()))


if __name__ == "__main__":
    main()
