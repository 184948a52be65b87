#!/usr/bin/env python
"""Per-frame latency of the reference-named drop-ins on C2 (the bench's
``C2_dropin_api`` line) and, with ``--profile``, a cProfile of the per-frame
loop (host overhead dominates: the GPU work of one frame is ~50 us)."""
import cProfile
import json
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    print(json.dumps(bench.dropin_line(dev)))
    if "--profile" not in sys.argv:
        return
    import paper_2012_09499_b200 as B
    from paper_2012_09499_b200 import scenes

    sc = scenes.make_c2(num_frames=64)
    arr = B.MicArray(sc.mic_pos, speed_of_sound=bench.C_SOUND)
    grid = B.build_tdoa_table(arr, B.CandidateGrid("near_field", sc.grid))
    table = B.precompute_sinc_table(grid, arr.pairs, bench.T, 4)
    freqs = bench.omega_of(sc.frame_length)
    frames = [B.SpectralFrame(sc.Y[f], freqs, frame_index=f) for f in range(64)]

    def per_frame():
        for fr in frames:
            cross = B.cross_spectrum(fr, arr.pairs)
            lat = B.build_gcc_lattice(cross, bench.T, 4)
            B.argmax_candidate(B.srp_approx(lat, table))

    per_frame()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        per_frame()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(22)


if __name__ == "__main__":
    main()
