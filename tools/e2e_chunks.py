#!/usr/bin/env python
"""End-to-end (pinned host in -> pinned host out) time of ChunkedRunner for
several chunk counts, C2 workload: approx with maps, approx argmax-only,
audio -> argmax-only, conventional with maps.  CUDA events on the caller's
stream, 3 warm-ups, median of 20 calls."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_09499_b200.pipeline import ChunkedRunner  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402


def timed(runner, x, maps, am, reps=20):
    for _ in range(3):
        runner.run(x, maps, am)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        runner.run(x, maps, am)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=bench.N_AUX,
                   weights="stored")
    F, M, Kb = scene.Y.shape
    Yh = torch.from_numpy(scene.Y).pin_memory()
    L = (F - 1) * Kb + 2 * Kb
    xh = torch.from_numpy(np.random.default_rng(0).standard_normal((M, L)).astype(np.float32)
                          ).pin_memory()
    maps = torch.empty((F, tdoa.shape[0]), dtype=torch.float32).pin_memory()
    am = torch.empty((F,), dtype=torch.int32).pin_memory()
    for chunks in (1, 2, 3, 4, 6, 8):
        row = [f"chunks {chunks}:"]
        r = ChunkedRunner(plan, F, M, "approx", chunks=chunks)
        row.append(f"approx maps {timed(r, Yh, maps, am):.3f}")
        r = ChunkedRunner(plan, F, M, "approx", chunks=chunks, maps=False)
        row.append(f"argmax-only {timed(r, Yh, None, am):.3f}")
        r = ChunkedRunner(plan, F, M, "approx", chunks=chunks, maps=False,
                          audio=(2 * Kb, Kb, "sqrt_hann"))
        row.append(f"audio argmax-only {timed(r, xh, None, am):.3f}")
        if chunks <= 4:
            r = ChunkedRunner(plan, F, M, "conventional", chunks=chunks)
            row.append(f"conv maps {timed(r, Yh, maps, am, reps=5):.3f}")
        print("  ".join(row), flush=True)


if __name__ == "__main__":
    main()
