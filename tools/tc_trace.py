#!/usr/bin/env python
"""Per-CTA item timeline of the K4 tcgen05 kernel (instrumentation build):
make prof && python tools/tc_trace.py.  Times in us from the first CTA entry:
per item P = producer starts, R = first stage ready at the MMA, M = last MMA
issued, D = drain starts (accumulator full), W = item written."""
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

import bench  # noqa: E402
from paper_2012_09499_b200.plan import SrpPlan  # noqa: E402


def main():
    scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=bench.N_AUX)
    Y = torch.from_numpy(scene.Y).cuda()
    for _ in range(3):
        plan.run(Y, "approx")
    torch.cuda.synchronize()
    buf = np.zeros((160, 64), dtype=np.uint64)
    lib.srpb_tc_trace_read(buf.ctypes.data)
    n = int((buf[:, 60] > 0).sum())
    t0 = buf[:n, 60].min()
    rel = lambda v: (float(v) - float(t0)) / 1e3
    ends = [rel(buf[c, 61]) for c in range(n)]
    print(f"{n} CTAs, span {max(ends):.1f} us, exit range {min(ends):.1f}..{max(ends):.1f}")
    for c in [int(x) for x in (sys.argv[1:] or [0, 1, 40, 41, 100, 101])]:
        row = [f"CTA {c:3d} in {rel(buf[c, 60]):5.1f}"]
        for it in range(12):
            ev = buf[c, it * 5: it * 5 + 5]
            if ev[0] == 0 and ev[1] == 0:
                continue
            row.append(f"[{it}: " + " ".join(f"{k}{rel(v):.1f}" if v else f"{k}-"
                                             for k, v in zip("PRMDW", ev)) + "]")
        row.append(f"out {rel(buf[c, 61]):5.1f}")
        print("  ".join(row))


if __name__ == "__main__":
    main()
