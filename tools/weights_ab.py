#!/usr/bin/env python
"""Stored sinc table vs weights generated in TMEM (on-the-fly K4) on the
sweep configs: captured approx step (graph replay, inputs resident), CUDA
events.  python tools/weights_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_09499_b200 import scenes  # noqa: E402


def step_ms(timer, plan, Y, steps=10):
    cap = plan.capture(Y.shape[0], Y.shape[1], "approx")
    cap.Y.copy_(Y)
    ms, _ = timer(cap.replay, steps, 2)
    return ms


def main():
    dev = torch.device("cuda", 0)
    clocks = type("NoClocks", (), {"resume": lambda s: None, "pause": lambda s: None})()
    timer = bench.Timer(dev, 1, clocks)
    cases = [("C2", scenes.make_c2(), (0, 2, 4), None), ("C3", scenes.make_c3(), (0, 4, 8), None),
             ("C5", scenes.make_c5(4096), (4,), (1, 256, 4096))]
    for name, sc, auxes, batches in cases:
        for n_aux in auxes:
            plans = {w: bench.build_plan(sc, n_aux, dev, weights=w, conventional=False)
                     for w in ("stored", "onthefly")}
            for B in (batches or (sc.Y.shape[0],)):
                Y = torch.from_numpy(sc.Y[:B]).to(dev)
                r = {w: step_ms(timer, p, Y) for w, p in plans.items()}
                print(f"{name} n_aux={n_aux} F={B}: stored {r['stored']:.4f} ms  onthefly "
                      f"{r['onthefly']:.4f} ms", flush=True)
            del plans
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
