#!/usr/bin/env python
"""Device STFT (K0) time on the C2 shape: 8 channels x 159,744 samples,
N = 1024, hop 512 -> 311 frames."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402

scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=bench.N_AUX,
               weights="stored")
for L, n in ((159744, 1024), (160000, 1000)):
    x = torch.randn(8, L, device="cuda")
    for _ in range(3):
        plan.stft(x, n) if n == 1024 else None
    if n != 1024:
        from paper_2012_09499_b200 import FrameSpec, stft_frames
        spec = FrameSpec(16000.0, n)
        f = lambda: stft_frames(x, spec)  # noqa: E731
    else:
        f = lambda: plan.stft(x, n)  # noqa: E731
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000)
    a.record()
    for _ in range(20):
        f()
    b.record()
    b.synchronize()
    print(f"N={n}: {a.elapsed_time(b) / 20 * 1e3:.1f} us per STFT of 8 x {L}")
