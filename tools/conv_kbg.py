#!/usr/bin/env python
"""K2 step time vs TMEM drain period (kb_per_group) on C2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402

scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
Y = torch.from_numpy(scene.Y).cuda()
for k in [int(v) for v in (sys.argv[1:] or ["2", "4", "8"])]:
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, weights="stored", kb_per_group=k)
    for _ in range(2):
        plan.run(Y, "conventional")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        plan.run(Y, "conventional")
    b.record()
    b.synchronize()
    print(f"kb_per_group {k}: {a.elapsed_time(b) / 5:.3f} ms")
