#!/usr/bin/env python
"""Kernel timeline of one approx step (instrumentation build, CUDA graph
replay): tensor-core lattice first CTA start / last CTA end and K4 CTA
entries / exits from globaltimer, so launch gaps and PDL overlap show.
    make prof && python tools/step_timeline.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_09499_b200 import _native  # noqa: E402

lib = _native.load(os.path.join(ROOT, "paper_2012_09499_b200", "libsrpb_prof.so"))
lib.srpb_tc_trace_read.argtypes = [ctypes.c_void_p]
lib.srpb_lt_profile_read.argtypes = [ctypes.c_void_p]

import bench  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402


def main():
    scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=bench.N_AUX)
    Y = torch.from_numpy(scene.Y).cuda()
    step = plan.capture(Y.shape[0], Y.shape[1], "approx")
    step.Y.copy_(Y)
    for _ in range(3):
        step.replay()
    torch.cuda.synchronize()
    lt = (ctypes.c_ulonglong * 16)()
    lib.srpb_lt_profile_read(ctypes.addressof(lt))
    step.replay()
    torch.cuda.synchronize()
    lib.srpb_lt_profile_read(ctypes.addressof(lt))
    tr = np.zeros((160, 64), dtype=np.uint64)
    lib.srpb_tc_trace_read(tr.ctypes.data)
    M = (1 << 64) - 1
    lt_start, lt_end = M - lt[10], lt[11]
    n = int((tr[:, 60] > 0).sum())
    k4_in = tr[:n, 60].astype(np.float64)
    k4_out = tr[:n, 61].astype(np.float64)
    t0 = float(lt_start)
    print(f"lattice   {0.0:7.2f} .. {(lt_end - t0) / 1e3:7.2f} us")
    print(f"K4 entries {(k4_in.min() - t0) / 1e3:7.2f} .. {(k4_in.max() - t0) / 1e3:7.2f} us, "
          f"exits {(k4_out.min() - t0) / 1e3:7.2f} .. {(k4_out.max() - t0) / 1e3:7.2f} us")
    print("(fix-up runs between the lattice end and the K4 work; K4 entries before the lattice "
          "end are PDL prologues)")


if __name__ == "__main__":
    main()
