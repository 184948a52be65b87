#!/usr/bin/env python
"""On-the-fly K4 (C4 shapes: P=496, L=301, N_aux 2, 2246 K blocks per
tile) rel-L2 vs the oracle for several TMEM drain periods (K blocks per
accumulator group: the tensor core's fp32 accumulation drifts with the
chain length, each group is folded into round-to-nearest totals).
8 frames of the seeded C4 scene x 2048 seeded candidates.

  python tools/otf_kbg_accuracy.py [kbg ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_09499_b200 import scenes  # noqa: E402
from test_scale_parity_gpu import device_plan, oracle_approx  # noqa: E402
from helpers import rel_l2  # noqa: E402


def main():
    kbgs = [int(a) for a in sys.argv[1:]] or [10, 16, 24, 32]
    scene = scenes.make_c4(num_frames=8)
    idx = np.sort(np.random.default_rng(44).choice(scene.grid.shape[0], 2048, replace=False))
    ref = oracle_approx(scene, range(8), idx, 2)
    Y = torch.from_numpy(scene.Y).cuda()
    for k in kbgs:
        plan = device_plan(scene, 2, weights="onthefly", grid=scene.grid[idx],
                           interp_kb_per_group=k, conventional=False)
        maps, am = plan.run(Y, "approx")
        maps = maps.cpu().numpy().astype(np.float64)
        errs = [rel_l2(maps[f], ref[f]) for f in range(8)]
        bias = [float(np.sum(maps[f] * ref[f]) / np.sum(ref[f] * ref[f]) - 1.0) for f in range(8)]
        same = int(np.sum(am.cpu().numpy() == ref.argmax(axis=1)))
        print(f"kbg={k:3d}: rel-L2 worst {max(errs):.3e} mean {np.mean(errs):.3e}  "
              f"scale bias {np.mean(bias):+.2e}  argmax equal {same}/8", flush=True)


if __name__ == "__main__":
    main()
