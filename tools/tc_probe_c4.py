#!/usr/bin/env python
"""Per-role cycle breakdown of the on-the-fly K4 at C4 shapes
(instrumentation build: make prof && python tools/tc_probe_c4.py [F] [J])."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_09499_b200 import _native, scenes  # noqa: E402

lib = _native.load(os.path.join(ROOT, "paper_2012_09499_b200", "libsrpb_prof.so"))
lib.srpb_tc_profile_read.argtypes = [ctypes.c_void_p]

from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402
import tc_probe  # noqa: E402


def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 320
    J = int(sys.argv[2]) if len(sys.argv) > 2 else 600000
    rng = np.random.default_rng(np.random.SeedSequence([4, 0, 0]))
    box = np.array([6.0, 5.0, 3.0])
    mic = rng.uniform(0.0, 1.0, size=(32, 3)) * box
    grid = scenes.box_grid(120, 100, 50, box)[:J]
    omega = 2.0 * np.pi * np.arange(512) * 16000.0 / 1024
    plan = SrpPlan.from_geometry(mic, grid, omega, speed_of_sound=343.0,
                                 sample_period=1 / 16000.0, n_aux=2, weights="onthefly",
                                 conventional=False)
    g = torch.Generator(device="cuda").manual_seed(0)
    Y = torch.complex(torch.randn((F, 32, 512), device="cuda", generator=g),
                      torch.randn((F, 32, 512), device="cuda", generator=g)).to(torch.complex64)
    xh, xl = plan.lattice_from_spectra(Y, split="f16")
    plan._approx_tc16(xh, xl, None)
    torch.cuda.synchronize()
    tc_probe.read()
    plan._approx_tc16(xh, xl, None)
    torch.cuda.synchronize()
    tc_probe.report(f"C4 onthefly F={F} J={J}", tc_probe.read())


if __name__ == "__main__":
    main()
