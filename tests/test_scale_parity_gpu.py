"""GPU parity at the benchmarked shapes (BASELINE configs at their stated
sizes, or large stated subsets of them) against the pinned oracle.

Each case runs the product kernels the bench times -- the tensor-core
lattice, the paired tcgen05 K4 with several work items per CTA pair (stored
weights, or weights generated in TMEM for C4), the tcgen05 K2 -- and
compares per-frame maps (rel-L2 <= 1e-5, BASELINE north_star) and argmax
(identical) with the oracle's fp64 restatement of the reference
(``oracle/srp_oracle.py``, pinned by ``tests/golden``).  Inputs are the
complex64 spectra upcast to complex128 for the oracle, so only compute
error is measured.
"""

import numpy as np
import pytest
import torch

from paper_2012_09499_b200 import scenes
from paper_2012_09499_b200.plan import SrpPlan
from oracle import srp_oracle as O
from helpers import assert_maps_match

pytestmark = pytest.mark.gpu
T = 1.0 / 16000.0
C = 343.0


def _pairs(mic_pos):
    pairs = O.canonical_pairs(mic_pos.shape[0])
    pm = np.array([m for m, _ in pairs], np.int32)
    pmp = np.array([mp for _, mp in pairs], np.int32)
    bounds = np.array([np.linalg.norm(mic_pos[m] - mic_pos[mp]) / C for m, mp in pairs])
    return pairs, pm, pmp, bounds


def oracle_approx(scene, frames, cand_idx, n_aux, chunk=512):
    """Reference approximate maps [len(frames), len(cand_idx)] (srp.py:201-347),
    sinc table built per candidate chunk (the dense C4 table is 345 GB)."""
    pairs, pm, pmp, bounds = _pairs(scene.mic_pos)
    omega = O.bin_frequencies(16000.0, scene.frame_length)
    rows = []
    for f in frames:
        psi, _ = O.cross_spectrum(scene.Y[f].astype(np.complex128), pm, pmp)
        rows.append(O.gcc_lattice(psi, omega, bounds, T, n_aux)[1])
    out = np.zeros((len(frames), len(cand_idx)))
    for lo in range(0, len(cand_idx), chunk):
        tdoa = O.tdoa_table_nearfield(scene.mic_pos, scene.grid[cand_idx[lo:lo + chunk]], pairs, C)
        _, w = O.sinc_table(tdoa, bounds, T, n_aux)
        for i in range(len(frames)):
            out[i, lo:lo + chunk] = O.approx_map(w, rows[i])
    return out


def oracle_conventional(scene, frames, cand_idx):
    pairs, pm, pmp, _ = _pairs(scene.mic_pos)
    omega = O.bin_frequencies(16000.0, scene.frame_length)
    psi = np.stack([O.cross_spectrum(scene.Y[f].astype(np.complex128), pm, pmp)[0]
                    for f in frames])
    tdoa = O.tdoa_table_nearfield(scene.mic_pos, scene.grid[cand_idx], pairs, C)
    return O.conventional_frames(psi, omega, tdoa, candidate_chunk=4096)


def device_plan(scene, n_aux, weights="auto", grid=None, **kw):
    return SrpPlan.from_geometry(scene.mic_pos, scene.grid if grid is None else grid,
                                 O.bin_frequencies(16000.0, scene.frame_length),
                                 speed_of_sound=C, sample_period=T, n_aux=n_aux,
                                 weights=weights, **kw)


def test_full_c2_approx_all_frames_vs_oracle():
    """C2 at its full size (F=311, J=50k, N_aux=4): the bench's approximate
    step (tensor-core lattice -> floor fix-up -> paired K4 with the multi-item
    ring, stored weights) against the oracle for every frame and candidate;
    conventional (K1 split -> tcgen05 K2) for three frames at full J."""
    scene = scenes.make_c2()
    plan = device_plan(scene, 4, weights="stored")
    Y = torch.from_numpy(scene.Y).cuda()
    cap = plan.capture(Y.shape[0], Y.shape[1], "approx")
    maps, am = cap.replay(Y)
    torch.cuda.synchronize()
    ref = oracle_approx(scene, range(311), np.arange(plan.J), 4, chunk=50000)
    worst = assert_maps_match(maps.cpu().numpy(), ref, am.cpu().numpy(), what="C2 approx")
    assert worst <= 1e-5
    sel = [0, 155, 310]
    mc, ac = plan.run(Y, "conventional")
    refc = oracle_conventional(scene, sel, np.arange(plan.J))
    assert_maps_match(mc[sel].cpu().numpy(), refc, ac[sel].cpu().numpy(), what="C2 conv")


@pytest.mark.parametrize("n_aux", list(range(9)))
def test_c3_candidate_chunk_every_n_aux_vs_oracle(n_aux):
    """C3 (P=120, Kb=1024): a 20k-candidate chunk of the 500k grid, 8 frames,
    every N_aux of the sweep (0..8), product path (tensor-core lattice where
    it fits, paired K4 with stored weights); conventional at N_aux 0."""
    scene = scenes.make_c3(num_frames=8)
    idx = np.sort(np.random.default_rng(30 + n_aux).choice(scene.grid.shape[0], 20000,
                                                          replace=False))
    plan = device_plan(scene, n_aux, weights="stored", grid=scene.grid[idx])
    Y = torch.from_numpy(scene.Y).cuda()
    maps, am = plan.run(Y, "approx")
    ref = oracle_approx(scene, range(8), idx, n_aux)
    assert_maps_match(maps.cpu().numpy(), ref, am.cpu().numpy(), what=f"C3 approx n_aux={n_aux}")
    if n_aux == 0:
        # conventional: 2 frames x every 4th candidate vs the oracle (the fp64
        # phase matrix of all 20k x 120 pairs x 1024 bins costs ~10 s a frame);
        # argmax over the compared subset, fused argmax = argmax of the maps
        mc, ac = plan.run(Y, "conventional")
        sel = np.arange(0, 20000, 4)
        refc = oracle_conventional(scene, [0, 7], idx[sel])
        sub = mc[[0, 7]][:, torch.as_tensor(sel, device=mc.device)].cpu().numpy()
        assert_maps_match(sub, refc, np.argmax(sub, axis=1), what="C3 conv")
        assert torch.equal(ac.long(), torch.argmax(mc, dim=1))


def test_c4_onthefly_tensor_core_vs_oracle():
    """C4 (M=32, P=496, L=301): weights generated in TMEM by the paired
    on-the-fly K4 (the headline kernel) over a 20,480-candidate subset and
    200 frames (two frame tiles: several items per CTA pair), 8 of them
    compared with the oracle; conventional on 8 frames x 4096 candidates."""
    scene = scenes.make_c4(num_frames=200)
    idx = np.sort(np.random.default_rng(41).choice(scene.grid.shape[0], 20480, replace=False))
    plan = device_plan(scene, 2, weights="onthefly", grid=scene.grid[idx])
    assert plan.weight_mode == "onthefly"
    Y = torch.from_numpy(scene.Y).cuda()
    maps, am = plan.run(Y, "approx")
    frames = [0, 1, 57, 99, 100, 150, 198, 199]
    # the oracle's sinc table costs 143,692 weights per candidate: every 3rd
    # candidate (all 128-candidate tiles, all items) is compared, the argmax
    # over the compared subset, and the fused argmax of every frame must be
    # the argmax of its stored map over all 20,480
    sel = np.arange(0, 20480, 3)
    ref = oracle_approx(scene, frames, idx[sel], 2)
    sub = maps[frames][:, torch.as_tensor(sel, device=maps.device)].cpu().numpy()
    assert_maps_match(sub, ref, np.argmax(sub, axis=1), what="C4 approx (on the fly)")
    assert torch.equal(am.long(), torch.argmax(maps, dim=1))
    sub = np.arange(0, 20480, 5)[:4096]
    cplan = device_plan(scene, 2, grid=scene.grid[idx[sub]])
    mc, ac = cplan.run(Y[:8].contiguous(), "conventional")
    refc = oracle_conventional(scene, range(8), idx[sub])
    assert_maps_match(mc.cpu().numpy(), refc, ac.cpu().numpy(), what="C4 conv")


@pytest.mark.parametrize("batch", [1, 256])
def test_c5_batches_full_grid_vs_oracle(batch):
    """C5 (J=200k, N_aux=4) at batch 1 and 256 on the full grid: both paths;
    the oracle checks every frame at batch 1 and 8 frames at batch 256."""
    scene = scenes.make_c5(batch)
    plan = device_plan(scene, 4, weights="stored")
    Y = torch.from_numpy(scene.Y).cuda()
    frames = list(range(batch)) if batch == 1 else [0, 1, 63, 64, 127, 128, 254, 255]
    cand = np.arange(plan.J)
    maps, am = plan.run(Y, "approx")
    ref = oracle_approx(scene, frames, cand, 4, chunk=50000)
    assert_maps_match(maps[frames].cpu().numpy(), ref, am[frames].cpu().numpy(),
                      what=f"C5 approx batch {batch}")
    mc, ac = plan.run(Y, "conventional")
    fr = frames[:2]
    sel = np.arange(0, plan.J, 5)   # every 5th candidate (the fp64 phases cost ~8 s a frame)
    refc = oracle_conventional(scene, fr, sel)
    sub = mc[fr][:, torch.as_tensor(sel, device=mc.device)].cpu().numpy()
    assert_maps_match(sub, refc, np.argmax(sub, axis=1), what=f"C5 conv batch {batch}")
    assert torch.equal(ac.long(), torch.argmax(mc, dim=1))


def test_c5_large_batch_argmax_only_vs_oracle():
    """The mode of C5's 65536 batch (maps never materialised, only the fused
    in-kernel argmax leaves the kernels) at 2,048 frames on the full 200k
    grid: the argmax of sampled frames equals the oracle's over all
    candidates, and the whole batch equals the maps path's argmax."""
    batch = 2048
    scene = scenes.make_c5(batch)
    plan = device_plan(scene, 4, weights="stored")
    Y = torch.from_numpy(scene.Y).cuda()
    cand = np.arange(plan.J)
    frames = [0, 1023, 1024, 2047]
    for path in ("approx", "conventional"):
        none, am = plan.run(Y, path, maps=False)
        assert none is None and am.shape == (batch,)
        maps, am_maps = plan.run(Y, path)
        assert torch.equal(am, am_maps) and torch.equal(am.long(), torch.argmax(maps, dim=1))
        if path == "approx":
            ref = oracle_approx(scene, frames, cand, 4, chunk=50000)
            assert_maps_match(maps[frames].cpu().numpy(), ref, am[frames].cpu().numpy(),
                              what=f"C5 approx argmax-only batch {batch}")
        else:
            sel = np.arange(0, plan.J, 5)
            ref = oracle_conventional(scene, frames[:1], sel)
            sub = maps[frames[:1]][:, torch.as_tensor(sel, device=maps.device)].cpu().numpy()
            assert_maps_match(sub, ref, np.argmax(sub, axis=1),
                              what=f"C5 conventional argmax-only batch {batch}")
        del maps
