#!/usr/bin/env python
"""Pinned host<->device copy bandwidth (the end-to-end floor for the maps
transfer) and the chunked runner's e2e time per chunk count."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def bw(nbytes, d2h):
    dev = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    host = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    for _ in range(3):
        (host.copy_(dev, non_blocking=True) if d2h else dev.copy_(host, non_blocking=True))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        (host.copy_(dev, non_blocking=True) if d2h else dev.copy_(host, non_blocking=True))
    b.record()
    b.synchronize()
    return nbytes * 10 / (a.elapsed_time(b) * 1e-3) / 1e9


def main():
    for n in (10 << 20, 62 << 20):
        print(f"{n >> 20:4d} MiB  H2D {bw(n, False):6.1f} GB/s  D2H {bw(n, True):6.1f} GB/s")
    import bench
    from paper_2012_09499_b200.pipeline import ChunkedRunner
    from paper_2012_09499_b200.plan import SrpPlan

    scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=bench.N_AUX,
                   weights="stored")
    F = scene.Y.shape[0]
    Yh = torch.from_numpy(scene.Y).pin_memory()
    mh = torch.empty((F, plan.J), dtype=torch.float32).pin_memory()
    ah = torch.empty(F, dtype=torch.int32).pin_memory()
    for path, counts in (("approx", (1, 2, 4, 6, 8)), ("conventional", (1, 2))):
        for c in counts:
            r = ChunkedRunner(plan, F, scene.Y.shape[1], path, chunks=c)
            for _ in range(3):
                r.run(Yh, mh, ah)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(10):
                r.run(Yh, mh, ah)
                torch.cuda.synchronize()
            print(f"{path:12s} chunks={len(r.bounds)}  e2e {(time.perf_counter() - t0) / 10 * 1e3:7.3f} ms")


if __name__ == "__main__":
    main()
