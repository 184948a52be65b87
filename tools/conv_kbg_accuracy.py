#!/usr/bin/env python
"""K2 (3xFP16) rel-L2 error vs the oracle for TMEM drain periods, at full C2
J (2 frames) and at C4's K (2 P Kb = 507,904; candidate subset)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from oracle import srp_oracle as O  # noqa: E402
from paper_2012_09499_b200 import scenes  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402


def relerr(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)))


def case(name, Y, pm, pmp, bounds, tdoa, omega, frames):
    psi = np.stack([O.cross_spectrum(Y[f].astype(complex), pm, pmp)[0] for f in frames])
    ref = O.conventional_frames(psi, omega, tdoa, candidate_chunk=4096)
    for k in (4, 8, 16, 32):
        plan = SrpPlan(tdoa, pm, pmp, bounds, omega, kb_per_group=k, backend="tc")
        maps, _ = plan.run(torch.from_numpy(np.ascontiguousarray(Y[frames])).cuda(), "conventional")
        print(f"{name} kb_per_group {k:2d}: rel-L2 {relerr(maps.cpu().numpy(), ref):.2e}")


scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
case("C2 full J", scene.Y, pm, pmp, bounds, tdoa, omega, [0, 200])
s4 = scenes.make_c4(num_frames=2)
pairs = O.canonical_pairs(s4.mic_pos.shape[0])
pm4 = np.array([m for m, _ in pairs], np.int32)
pmp4 = np.array([mp for _, mp in pairs], np.int32)
b4 = np.array([np.linalg.norm(s4.mic_pos[m] - s4.mic_pos[mp]) / 343.0 for m, mp in pairs])
g4 = s4.grid[np.linspace(0, s4.grid.shape[0] - 1, 512).astype(int)]
t4 = O.tdoa_table_nearfield(s4.mic_pos, g4, pairs, 343.0)
case("C4 K=507904", s4.Y, pm4, pmp4, b4, t4, O.bin_frequencies(16000.0, 1024), [0, 1])
