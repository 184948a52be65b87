#!/usr/bin/env python
"""One eager pass of the C4 headline step's kernels (for ncu captures):
the bench's plan (scenes.make_c4 geometry, 600k candidates, N_aux 2) on
``--frames`` frames of the seeded scene; approx (lattice -> floor fix-up ->
on-the-fly K4) and/or conventional (K1 split -> K2).  Also the standalone
front-end kernels (K0 STFT, K1 GCC-PHAT, K5 argmax) at C4/C2 sizes with
``--frontend``.

  ncu --set full -k regex:srp_tc_kernel -c 1 python tools/profile_c4.py --paths approx
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=4096)
    ap.add_argument("--paths", default="approx,conventional")
    ap.add_argument("--frontend", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    scene = bench.c4_scene(args.frames)
    plan = bench.build_plan(scene, 2, dev)
    Y = torch.from_numpy(scene.Y).to(dev)
    for path in args.paths.split(","):
        if path:
            plan.run(Y, path)
            torch.cuda.synchronize()
    if args.frontend:
        from paper_2012_09499_b200.plan import standalone_argmax

        # K1 over the C4 batch (psi [F, 496, 512] complex64 + floors)
        plan.cross_spectra(Y)
        # K0: STFT of the C4 audio shape (32 x (F-1)*512+1024 samples)
        L = (args.frames - 1) * 512 + 1024
        x = torch.from_numpy(np.random.default_rng(0).standard_normal((32, L)).astype(
            np.float32)).to(dev)
        plan.stft(x, 1024)
        # K5 standalone over C4 maps of 256 frames
        maps = torch.randn((256, plan.J), device=dev)
        standalone_argmax(maps)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
