#!/usr/bin/env python
"""Small driver for ncu: builds the C2 plan and runs `--reps` approximate and
conventional steps (GCC-PHAT -> lattice -> interp / conventional), nothing
else.  Usage under gpurun:

    python tools/profile_step.py && ncu --set full -k regex:srp_tc_kernel ... \
        python tools/profile_step.py
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--backend", default="auto")
    ap.add_argument("--paths", default="approx,conventional")
    args = ap.parse_args()
    scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=bench.N_AUX,
                   weights="stored", backend=args.backend)
    Y = torch.from_numpy(scene.Y).cuda()
    for path in args.paths.split(","):
        for _ in range(args.reps):
            if path == "approx2step":  # unfused K1 -> K3 -> K4
                plan.approx(plan.lattice(plan.cross_spectra(Y)[0]))
            else:
                plan.run(Y, path)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
