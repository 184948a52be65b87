"""Edge shapes of the two-team tcgen05 generator kernels (K2 steering
phases, on-the-fly K4 sinc weights): teams take alternate K blocks, so the
cases that matter are tiles with very few K blocks (fewer than the fold
window, a single block), odd K-block counts per pair (the phase generator
strides across pair boundaries) and many work items per CTA pair (the
accumulator ping-pong wraps across items).  Checked against the pinned
oracle (and, for K4, bit for bit against the stored-weight kernel)."""

import numpy as np
import pytest
import torch

from oracle import srp_oracle as O
from paper_2012_09499_b200.plan import SrpPlan
from helpers import REL_L2_TOL, assert_maps_match, rel_l2

pytestmark = pytest.mark.gpu
T = 1.0 / 16000.0
C = 343.0


def _geometry(mic_pos, points):
    pairs = O.canonical_pairs(mic_pos.shape[0])
    pm = np.array([m for m, _ in pairs], np.int32)
    pmp = np.array([mp for _, mp in pairs], np.int32)
    bounds = np.array([np.linalg.norm(mic_pos[m] - mic_pos[mp]) / C for m, mp in pairs])
    tdoa = O.tdoa_table_nearfield(mic_pos, points, pairs, C)
    return pairs, pm, pmp, bounds, tdoa


def _spectra(rng, F, M, Kb):
    return (rng.standard_normal((F, M, Kb)) + 1j * rng.standard_normal((F, M, Kb))).astype(
        np.complex64)


@pytest.mark.parametrize("n_aux", [0, 1])
def test_onthefly_short_lattice_many_items(n_aux):
    """3 microphones 2 cm apart: every pair's lattice has 3 (+2 N_aux)
    samples, so a tile is a single 64-column K block -- far below the fold
    window -- while 150k candidates give each CTA pair ~8 work items."""
    rng = np.random.default_rng(7 + n_aux)
    mic = np.array([[0.0, 0.0, 1.5], [0.02, 0.0, 1.5], [0.0, 0.02, 1.5]])
    pts = rng.uniform([-2.0, -2.0, 0.0], [2.0, 2.0, 2.5], size=(150_000, 3))
    pairs, pm, pmp, bounds, tdoa = _geometry(mic, pts)
    omega = O.bin_frequencies(16000.0, 1024)
    Y = _spectra(rng, 40, 3, omega.size)
    st = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=T, n_aux=n_aux, weights="stored",
                 backend="tc")
    ot = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=T, n_aux=n_aux,
                 weights="onthefly", backend="tc")
    assert ot.W is None and ot.T_pad <= 64  # one K block per tile
    Yd = torch.from_numpy(Y).cuda()
    m1, a1 = st.run(Yd, "approx")
    m2, a2 = ot.run(Yd, "approx")
    torch.cuda.synchronize()
    assert torch.equal(m1, m2) and torch.equal(a1, a2)
    # oracle on every frame, a seeded candidate subset (+ each frame's argmax)
    sel = np.unique(np.concatenate([rng.choice(pts.shape[0], 3000, replace=False),
                                    a2.cpu().numpy()]))
    _, w = O.sinc_table(tdoa[sel], bounds, T, n_aux)
    ref = np.stack([O.approx_map(w, O.gcc_lattice(
        O.cross_spectrum(Y[f].astype(np.complex128), pm, pmp)[0], omega, bounds, T, n_aux)[1])
        for f in range(Y.shape[0])])
    got = m2.cpu().numpy()[:, sel].astype(np.float64)
    for f in range(ref.shape[0]):
        assert rel_l2(got[f], ref[f]) <= REL_L2_TOL, f
        # a 2 cm array barely separates candidates: many are equal to fp32
        # rounding, so the argmax is checked up to such near-ties
        ga = int(np.searchsorted(sel, int(a2[f])))
        assert ref[f].max() - ref[f][ga] <= 1e-6 * np.abs(ref[f]).max(), f


@pytest.mark.parametrize("kb", [32, 96, 160])
def test_conventional_teams_odd_blocks_per_pair(kb):
    """K2 with 1, 3 and 5 K blocks per pair (Kb = 32, 96, 160 harmonic
    bins): the two generator teams' blocks straddle pair boundaries in both
    parities; 12 work items per CTA pair."""
    rng = np.random.default_rng(kb)
    M = 6
    mic = rng.uniform(0.0, 1.0, size=(M, 3)) * np.array([4.0, 3.0, 2.5])
    pts = rng.uniform(0.0, 1.0, size=(60_000, 3)) * np.array([4.0, 3.0, 2.5])
    pairs, pm, pmp, bounds, tdoa = _geometry(mic, pts)
    omega = O.bin_frequencies(16000.0, 1024)[:kb]
    Y = _spectra(rng, 24, M, kb)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=T, n_aux=2, backend="tc")
    maps, am = plan.run(torch.from_numpy(Y).cuda(), "conventional")
    torch.cuda.synchronize()
    psi = np.stack([O.cross_spectrum(Y[f].astype(np.complex128), pm, pmp)[0]
                    for f in range(Y.shape[0])])
    sel = np.unique(np.concatenate([rng.choice(pts.shape[0], 4000, replace=False),
                                    am.cpu().numpy()]))
    ref = O.conventional_frames(psi, omega, tdoa[sel])
    got = maps.cpu().numpy()[:, sel]
    assert_maps_match(got, ref, np.searchsorted(sel, am.cpu().numpy()),
                      what=f"conventional Kb={kb}")


@pytest.mark.parametrize("F", [1, 2, 3, 4])
def test_conventional_few_frames_vs_oracle(F):
    """Few-frame conventional batches (C5 batch 1 ..) take the per-candidate
    phase-recurrence kernel (conventional.cu conventional_few_kernel): maps
    and argmax vs the oracle, and vs the tensor-core K2 on the same psi."""
    rng = np.random.default_rng(100 + F)
    ang = 2 * np.pi * np.arange(8) / 8
    mic = np.stack([0.1 * np.cos(ang), 0.1 * np.sin(ang), np.full(8, 1.2)], axis=1)
    pts = rng.uniform([-2.5, -2.5, 0.0], [2.5, 2.5, 2.5], size=(40_000, 3))
    pairs, pm, pmp, bounds, tdoa = _geometry(mic, pts)
    omega = O.bin_frequencies(16000.0, 1024)
    Y = _spectra(rng, F, 8, omega.size)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega)
    maps, am = plan.run(torch.from_numpy(Y).cuda(), "conventional")
    torch.cuda.synchronize()
    psi = np.stack([O.cross_spectrum(Y[f].astype(np.complex128), pm, pmp)[0] for f in range(F)])
    sel = np.unique(np.concatenate([rng.choice(pts.shape[0], 4000, replace=False),
                                    am.cpu().numpy()]))
    ref = O.conventional_frames(psi, omega, tdoa[sel])
    assert_maps_match(maps.cpu().numpy()[:, sel], ref, np.searchsorted(sel, am.cpu().numpy()),
                      what=f"few-frame conventional F={F}")
    tc = SrpPlan(tdoa, pm, pmp, bounds, omega, backend="tc")
    m2, a2 = tc.run(torch.from_numpy(Y).cuda(), "conventional")
    assert rel_l2(maps.cpu().numpy(), m2.cpu().numpy()) <= 1e-5
    assert torch.equal(am.cpu(), a2.cpu())


def _xi16(plan, Y):
    hi, lo = plan.lattice_from_spectra(Y, split="f16")
    return ((hi.double() + lo.double()) / plan.xi_scale16).cpu().numpy()


@pytest.mark.parametrize("room,M", [((6.0, 5.0, 3.0), 12), ((0.9, 0.8, 0.5), 6)])
def test_lattice_tensor_core_multipass(room, M):
    """Tensor-core lattice with more than 64 lag slots (2L + 1 = 781 in a
    6x5x3 m room: 13 passes of 64 slots; ~2 passes for the small room):
    vs the SIMT lattice (3e-6) and the reference lattice (1e-5), pad columns
    zero, bitwise repeatable, and speculative-floor edge frames redone by
    the fix-up kernel after all passes (including a tiny channel power the
    in-place per-channel normalisation of later passes cannot take)."""
    rng = np.random.default_rng(M)
    mic = rng.uniform(0.0, 1.0, size=(M, 3)) * np.array(room)
    pts = rng.uniform(0.0, 1.0, size=(64, 3)) * np.array(room)
    pairs, pm, pmp, bounds, tdoa = _geometry(mic, pts)
    omega = O.bin_frequencies(16000.0, 1024)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=T, n_aux=2)
    assert plan.lattice_tc and 2 * plan.L + 1 > 64
    from paper_2012_09499_b200 import _native as NN
    assert NN.query("srpb_lattice_tc_supported", M, plan.P, plan.Kb, plan.L, plan.T_pad)
    Y = _spectra(rng, 21, M, omega.size)
    Y[2, 1, 7] = 1e-13 + 0j     # floor edge cases (the fix-up redoes the frame)
    Y[3, 0, 3] = 1e-20 + 1e-20j
    Y[4] = 0
    # a channel power below 1e-30 whose pair products stay above it: later
    # passes normalise channels in place, so pass 0 must flag the frame
    Y[5, :, 9] *= 1e3
    Y[5, 2, 9] = 1e-16 + 0j
    Yd = torch.from_numpy(Y).cuda()
    tc = _xi16(plan, Yd)
    assert np.array_equal(tc, _xi16(plan, Yd))
    plan.lattice_tc = False
    simt = _xi16(plan, Yd)
    plan.lattice_tc = True
    total = plan.total_samples
    assert np.all(tc[:, total:] == 0.0)
    for f in range(Y.shape[0]):
        if f == 4:
            assert np.all(tc[f] == 0.0)
            continue
        assert rel_l2(tc[f, :total], simt[f, :total]) <= 3e-6, f
    for f in (0, 2, 3, 5, 20):
        psi = O.cross_spectrum(Y[f].astype(np.complex128), pm, pmp)[0]
        ref = np.concatenate(O.gcc_lattice(psi, omega, bounds, T, 2)[1])
        assert rel_l2(tc[f, :total], ref) <= REL_L2_TOL, f


_SINGLE_CTA_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + '/tests')
from test_team_edges_gpu import _geometry, _spectra, T
from oracle import srp_oracle as O
from paper_2012_09499_b200.plan import SrpPlan
rng = np.random.default_rng(5)
mic = rng.uniform(0.0, 1.0, size=(10, 3)) * np.array([6.0, 5.0, 3.0])
pts = rng.uniform(0.0, 1.0, size=(40_000, 3)) * np.array([6.0, 5.0, 3.0])
pairs, pm, pmp, bounds, tdoa = _geometry(mic, pts)
omega = O.bin_frequencies(16000.0, 1024)
Y = torch.from_numpy(_spectra(rng, 40, 10, omega.size)).cuda()
out = {}
for w in ("onthefly", "stored"):
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=T, n_aux=2, weights=w)
    m, a = plan.run(Y, "approx")
    out[w] = (m.cpu().numpy(), a.cpu().numpy())
m, a = plan.run(Y, "conventional")
out["conv"] = (m.cpu().numpy(), a.cpu().numpy())
np.savez(sys.argv[2], **{k + "_m": v[0] for k, v in out.items()}, **{k + "_a": v[1] for k, v in out.items()})
"""


def test_single_cta_and_paired_kernels_agree_bitwise(tmp_path):
    """The CTA-pair (cta_group::2, default) and single-CTA variants of the
    generator kernels (K2, on-the-fly K4) and of the stored-weight K4 give
    bitwise identical maps and argmax (same per-element accumulation order);
    the switches are read once per process, so each variant runs in its own."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for name, env in (("pair", {}), ("single", {"SRPB_OTF_PAIR": "0", "SRPB_TC_PAIR": "0"})):
        path = tmp_path / f"{name}.npz"
        e = dict(os.environ, **env)
        subprocess.run([sys.executable, "-c", _SINGLE_CTA_SCRIPT, root, str(path)], env=e,
                       check=True, timeout=600)
        with np.load(path) as z:
            res[name] = {k: z[k] for k in z.files}
    for k in res["pair"]:
        assert np.array_equal(res["pair"][k], res["single"][k]), k
    assert np.array_equal(res["pair"]["onthefly_m"], res["pair"]["stored_m"])
