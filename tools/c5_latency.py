#!/usr/bin/env python
"""C5 (BASELINE configs[4]): UCA M=8, N=1024, J=200k candidates, N_aux=4 --
per-batch device time of both paths for batch 1 ... 4096 (plan built once
from the device geometry; CUDA-graph replay; inputs resident)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from oracle import srp_oracle as O  # noqa: E402
from paper_2012_09499_b200 import scenes  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402


def main():
    sc = scenes.make_c5(4096)
    plan = SrpPlan.from_geometry(sc.mic_pos, sc.grid, O.bin_frequencies(16000.0, 1024),
                                 speed_of_sound=343.0, sample_period=1 / 16000.0, n_aux=4,
                                 weights="stored")
    Yall = torch.from_numpy(sc.Y).cuda()
    print(f"C5: J={plan.J} P={plan.P} T_pad={plan.T_pad}")
    for B in (1, 16, 256, 4096):
        for path in ("approx", "conventional"):
            if path == "conventional" and B > 256:
                continue
            cap = plan.capture(B, 8, path)
            cap.Y.copy_(Yall[:B])
            for _ in range(3):
                cap.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20 if B < 4096 else 5
            a.record()
            for _ in range(reps):
                cap.replay()
            b.record()
            b.synchronize()
            ms = a.elapsed_time(b) / reps
            print(f"batch {B:5d} {path:12s} {ms:9.3f} ms  {B * plan.J / (ms * 1e-3):.3e} f.c/s")


if __name__ == "__main__":
    main()
