#!/usr/bin/env python
"""Fused (in-kernel) argmax vs the standalone K5 over the stored maps, for
several frame counts of the C2 workload (debug aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan, standalone_argmax  # noqa: E402


def main():
    scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=bench.N_AUX,
                   backend="tc")
    Y = torch.from_numpy(scene.Y).cuda()
    for path in ("approx", "conventional"):
        for F in (311, 100, 11, 1):
            for rep in range(2):
                m, am = plan.run(Y[:F].contiguous(), path)
                ref = standalone_argmax(m)
                bad = (am != ref).nonzero().flatten().tolist()
                print(path, F, rep, "mismatches", len(bad), bad[:5],
                      [(int(am[f]), int(ref[f]), float(m[f, am[f]]), float(m[f, ref[f]]))
                       for f in bad[:3]])


if __name__ == "__main__":
    main()
