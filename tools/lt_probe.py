#!/usr/bin/env python
"""Phase breakdown of the tensor-core lattice kernel (instrumentation build:
make prof && python tools/lt_probe.py [--c4 F]).  Cycles summed over CTAs / warps."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_09499_b200 import _native  # noqa: E402

lib = _native.load(os.path.join(ROOT, "paper_2012_09499_b200", "libsrpb_prof.so"))
lib.srpb_lt_profile_read.argtypes = [ctypes.c_void_p]

import bench  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

NAMES = {0: "setup", 2: "mma_done(epi view)", 3: "generator loop (per gen warp)",
         4: "gen wait Y (per gen warp)", 5: "epi wait acc (per epi warp)",
         6: "cluster_sync wait", 7: "rank0 output + end", 8: "lifetime"}


def main():
    from paper_2012_09499_b200 import scenes

    if len(sys.argv) > 1 and sys.argv[1] == "--c4":
        from lattice_time import c4_setup
        plan, Y = c4_setup(int(sys.argv[2]) if len(sys.argv) > 2 else 320)
    else:
        scene = scenes.make_c2()
        plan = bench.build_plan(scene, 4, torch.device("cuda", 0), weights="stored")
        Y = torch.from_numpy(scene.Y).cuda()
    for _ in range(2):
        plan.lattice_from_spectra(Y, split="f16")
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 16)()
    lib.srpb_lt_profile_read(ctypes.addressof(buf))
    plan.lattice_from_spectra(Y, split="f16")
    torch.cuda.synchronize()
    lib.srpb_lt_profile_read(ctypes.addressof(buf))
    c = list(buf)
    n = max(c[9], 1)
    per = {0: n, 2: 4 * n, 3: 16 * n, 4: 16 * n, 5: 4 * n, 6: n, 7: n, 8: n}
    M = (1 << 64) - 1
    print(f"{n} CTAs; span {(c[11] - (M - c[10])) / 1e3:.1f} us, starts spread "
          f"{(c[12] - (M - c[10])) / 1e3:.1f} us")
    for i, name in NAMES.items():
        print(f"  {name:34s} {c[i] / per[i]:10.0f} cycles")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(5):
        plan.lattice_from_spectra(Y, split="f16")
    ev[1].record()
    ev[1].synchronize()
    print(f"  event time per launch (instrumented build): {ev[0].elapsed_time(ev[1]) / 5 * 1e3:.1f} us")


if __name__ == "__main__":
    main()
