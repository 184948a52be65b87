#!/usr/bin/env python
"""K4 (3xFP16) kernel time with and without the map store (argmax only):
isolates the cost of writing the F x J maps from the epilogue."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402


class T:
    def __init__(self):
        self.ev = {}

    def before(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev.setdefault(name, []).append([e, None])

    def after(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev[name][-1][1] = e


def main():
    scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=bench.N_AUX,
                   weights=os.environ.get("SRPB_WEIGHTS", "stored"))
    Y = torch.from_numpy(scene.Y).cuda()
    for path in sys.argv[1:] or ["approx"]:
        for maps in (True, False):
            for _ in range(3):
                plan.run(Y, path, maps=maps)
            t = T()
            plan.kernel_timer = t
            for _ in range(10):
                plan.run(Y, path, maps=maps)
            plan.kernel_timer = None
            torch.cuda.synchronize()
            for name, evs in t.ev.items():
                ms = sorted(a.elapsed_time(b) for a, b in evs)
                print(f"{path:12s} maps={maps!s:5s} {name:28s} median {ms[len(ms) // 2] * 1e3:8.1f} us")


if __name__ == "__main__":
    main()
