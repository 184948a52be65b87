#!/usr/bin/env python
"""Plan build time: host TDOA table + host splits (SrpPlan(tdoa_table, ...))
vs device geometry (SrpPlan.from_geometry), C2 and C3-shaped grids."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_09499_b200 as B  # noqa: E402
from paper_2012_09499_b200 import scenes  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402
from oracle import srp_oracle as O  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t


def main():
    cases = {"C2": (scenes.make_c2(num_frames=1), 1024, 4),
             "C3": (scenes.make_c3(num_frames=1), 2048, 8)}
    for name, (sc, n, n_aux) in cases.items():
        pts, pos = sc.grid, sc.mic_pos
        omega = O.bin_frequencies(16000.0, n)
        arr = B.MicArray(pos, speed_of_sound=343.0)
        pm = np.array([p.index_m for p in arr.pairs], np.int32)
        pmp = np.array([p.index_m_prime for p in arr.pairs], np.int32)
        bounds = np.array([p.tdoa_bound for p in arr.pairs])
        kw = dict(sample_period=1 / 16000.0, n_aux=n_aux, weights="onthefly")

        def host():
            g = B.build_tdoa_table(arr, B.CandidateGrid("near_field", pts))
            return SrpPlan(g.tdoa_table, pm, pmp, bounds, omega, **kw)

        SrpPlan.from_geometry(pos[:, :], pts[:1000], omega, speed_of_sound=343.0, **kw)  # warm
        _, th = timed(host)
        _, td = timed(lambda: SrpPlan.from_geometry(pos, pts, omega, speed_of_sound=343.0, **kw))
        print(f"{name}: J={pts.shape[0]} P={len(pm)}  host table+splits {th:.2f} s   "
              f"device {td * 1e3:.1f} ms  ({th / td:.0f}x)")


if __name__ == "__main__":
    main()
