#!/usr/bin/env python
"""Time the K4 tensor-core launch alone for output variants (maps only,
argmax keys only, both) and drain periods, on the C2 workload."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import bench  # noqa: E402
from paper_2012_09499_b200 import _native as N  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402

scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
Y = torch.from_numpy(scene.Y).cuda()
plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=4, weights="stored")
psi, _ = plan.cross_spectra(Y)
xi = plan.lattice(psi)
plan.approx(xi)  # builds W_hi / W_lo
xh, xl = plan.split_tf32(xi)
F, J = xi.shape[0], plan.J
maps = torch.empty((F, J), device="cuda")
keys = torch.zeros(F, dtype=torch.int64, device="cuda")
s = N.stream_handle()
for kbg in (4, 10, 32):
    for tag, m, k in (("maps+keys", maps, keys), ("maps", maps, None), ("keys", None, keys)):
        def run():
            N.call("srpb_interp_tc", N.ptr(plan.W_hi), N.ptr(plan.W_lo), N.ptr(xh), N.ptr(xl), F, J,
                   plan.T_pad, N.ptr(m), N.ptr(k), kbg, s)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(20):
            run()
        b.record()
        b.synchronize()
        print(f"kb_per_group={kbg:2d} {tag:10s}: {a.elapsed_time(b) / 20 * 1e3:7.1f} us")
