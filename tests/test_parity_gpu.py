"""GPU parity: the CUDA path (through libsrpb.so's C ABI) vs the reference.

Golden vectors come from running the unmodified reference
(``tests/golden/make_golden.py``); larger seeded cases compare against the
pinned oracle.  Tolerance (BASELINE.json north_star): per-frame relative L2
map error <= 1e-5 for the fp32 path, identical argmax.
"""

import numpy as np
import pytest
import torch

import paper_2012_09499_b200 as B
from paper_2012_09499_b200 import scenes
from paper_2012_09499_b200.plan import SrpPlan
from oracle import srp_oracle as O
from conftest import load_golden
from helpers import REL_L2_TOL, assert_maps_match, rel_l2

pytestmark = pytest.mark.gpu
T = 1.0 / 16000.0


def plan_from_golden(g, n_aux=None, weights="auto", backend="auto"):
    return SrpPlan(g["tdoa"], g["pair_m"], g["pair_mp"], g["bounds"], g["omega"],
                   sample_period=None if n_aux is None else T, n_aux=n_aux, weights=weights,
                   backend=backend)


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x)).cuda()


# --------------------------------------------------------------------- K0
def _rel_rows(a, b):
    """max over (frame, channel) of the rel-L2 error of a row of bins"""
    num = np.linalg.norm((a - b).reshape(-1, a.shape[-1]), axis=1)
    den = np.maximum(np.linalg.norm(b.reshape(-1, b.shape[-1]), axis=1), 1e-30)
    return float(np.max(num / den))


def test_stft_matches_reference():
    """Device STFT (FFT path: N = 64 ... 2048, both windows, several hops)
    against the reference's stft_analyze outputs."""
    g = load_golden("stft")
    for tag in "abcd":
        n, hop, win = (int(v) for v in g[f"cfg_{tag}"])
        spec = B.FrameSpec(16000.0, n, hop, "sqrt_hann" if win == 0 else "rectangular")
        frames = B.stft_analyze(g["x"], spec)
        Y = np.stack([fr.spectra for fr in frames])
        assert Y.shape == g[f"Y_{tag}"].shape, tag
        assert _rel_rows(Y, g[f"Y_{tag}"]) < 2e-6, tag
        np.testing.assert_allclose(frames[0].bin_frequencies, g[f"freqs_{tag}"])
        assert frames[3].frame_index == 3


def test_stft_non_power_of_two_frames_vs_oracle():
    """Even, non-power-of-two frame lengths take the direct-DFT kernel."""
    x = np.random.default_rng(5).standard_normal((2, 9000)).astype(np.float32)
    for n, hop, win in ((300, 150, "sqrt_hann"), (2, 1, "rectangular"), (1000, 333, "sqrt_hann"),
                        (256, 77, "sqrt_hann"), (4096, 1001, "rectangular")):  # FFT, odd hops
        Y = B.stft_frames(x, B.FrameSpec(16000.0, n, hop, win)).cpu().numpy()
        ref = O.stft(x.astype(float), n, hop, win)
        assert Y.shape == ref.shape and _rel_rows(Y, ref) < 2e-6, n


def test_run_audio_matches_spectra_path():
    """K0 -> K1a/K1b/K3 -> K4 from audio equals run() on the reference STFT
    of the same audio (to the fp32 tolerance), and the drop-in errors match."""
    g = load_golden("c1")
    x = np.random.default_rng(11).standard_normal((4, 16000)).astype(np.float32)
    plan = plan_from_golden(g, 2, weights="stored", backend="tc")
    maps_a, am_a = plan.run_audio(dev(x), 512)
    Y = O.stft(x.astype(float), 512).astype(np.complex64)
    maps_b, am_b = plan.run(dev(Y), "approx")
    assert_maps_match(maps_a.cpu().numpy(), maps_b.cpu().numpy(), am_a.cpu().numpy(),
                      what="run_audio")
    cap = plan.capture(None, 4, "approx", audio=(x.shape[1], 512, None, "sqrt_hann"))
    m_c, a_c = cap.replay(dev(x))
    assert torch.equal(m_c, maps_a) and torch.equal(a_c, am_a)
    runner = B.ChunkedRunner(plan, maps_a.shape[0], 4, "approx", chunks=2,
                             audio=(512, None, "sqrt_hann"))
    xh = torch.from_numpy(x).pin_memory()
    mh = torch.empty(tuple(maps_a.shape), dtype=torch.float32).pin_memory()
    ah = torch.empty(maps_a.shape[0], dtype=torch.int32).pin_memory()
    runner.run(xh, mh, ah)
    torch.cuda.synchronize()
    assert torch.equal(mh, maps_a.cpu()) and torch.equal(ah, am_a.cpu())
    with pytest.raises(ValueError, match="shorter than one frame"):
        plan.stft(dev(x[:, :100]), 512)
    with pytest.raises(ValueError, match="bins"):
        plan.stft(dev(x), 1024)


# --------------------------------------------------------------------- K1
@pytest.mark.parametrize("name", ["c1", "c2_subset", "random_small", "on_lattice"])
def test_gcc_phat_matches_reference(name):
    g = load_golden(name)
    plan = plan_from_golden(g)
    psi, floors = plan.cross_spectra(dev(g["Y"]))
    psi = psi.cpu().numpy()
    assert np.max(np.abs(psi - g["psi"])) < 2e-6
    np.testing.assert_allclose(floors.cpu().numpy(), g["floors"], rtol=1e-12)


def test_gcc_phat_edge_cases():
    g = load_golden("cross_edges")
    pm, pmp = g["pair_m"], g["pair_mp"]
    from paper_2012_09499_b200.spectral import gcc_phat_batch

    for key in ("rand", "scaled", "zero_bin"):
        psi, fl = gcc_phat_batch(dev(g[f"y_{key}"][None]), pm, pmp)
        assert np.max(np.abs(psi[0].cpu().numpy() - g[f"psi_{key}"])) < 2e-6
        assert fl.item() == pytest.approx(float(g[f"floor_{key}"]), rel=1e-12)
    psi, _ = gcc_phat_batch(dev(g["y_zero_bin"][None]), pm, pmp)
    assert torch.all(psi[0, :, 10] == 0)
    raw, fl = gcc_phat_batch(dev(g["y_rand"][None]), pm, pmp, weighting="identity")
    np.testing.assert_allclose(raw[0].cpu().numpy(), g["raw_rand"], rtol=1e-6, atol=1e-6)
    psi, fl = gcc_phat_batch(dev(np.zeros((1, 4, 64), np.complex64)), pm, pmp)
    assert torch.all(psi == 0) and fl.item() == 0.0
    tiny = np.full((1, 2, 64), 1e-8 + 0j, dtype=np.complex64)
    psi, fl = gcc_phat_batch(dev(tiny), [1], [0], phat_floor=1.0)
    np.testing.assert_allclose(psi[0].cpu().numpy(), g["psi_tiny_floor1"], rtol=1e-5)
    assert fl.item() == 1.0


# --------------------------------------------------------------------- K2
@pytest.mark.parametrize("backend", ["simt", "tc"])
@pytest.mark.parametrize("name", ["c1", "c2_subset", "random_small", "on_lattice"])
def test_conventional_matches_reference(name, backend):
    g = load_golden(name)
    if backend == "tc" and g["omega"].size % 16:
        pytest.skip("tensor-core conventional kernel needs Kb % 16 == 0")
    plan = plan_from_golden(g, backend=backend)
    maps, am = plan.conventional(dev(g["psi"].astype(np.complex64)))
    assert_maps_match(maps.cpu().numpy(), g["conv"], am.cpu().numpy(), what=name)
    if name in ("c1", "c2_subset"):  # real-source scenes: argmax must be identical
        assert list(am.cpu().numpy()) == list(g["argmax_conv"])


def test_conventional_nonharmonic_bins():
    g = load_golden("nonharmonic")
    plan = SrpPlan(g["tdoa"], g["pair_m"], g["pair_mp"], g["bounds"], g["omega"])
    assert not plan.harmonic
    maps, am = plan.conventional(dev(g["psi"].astype(np.complex64)))
    assert_maps_match(maps.cpu().numpy(), g["conv"], am.cpu().numpy(), what="nonharmonic")


# --------------------------------------------------------------------- K3
@pytest.mark.parametrize("name", ["c1", "c2_subset", "random_small", "on_lattice"])
def test_lattice_matches_reference(name):
    g = load_golden(name)
    psi = dev(g["psi"].astype(np.complex64))
    for n_aux in g["n_aux"]:
        plan = plan_from_golden(g, int(n_aux))
        assert list(plan.half_counts) == list(g[f"half_counts_{n_aux}"])
        xi = plan.lattice(psi).cpu().numpy()
        total = plan.total_samples
        assert np.all(xi[:, total:] == 0.0)
        for f in range(xi.shape[0]):
            assert rel_l2(xi[f, :total], g[f"lattice_{n_aux}"][f]) <= REL_L2_TOL


@pytest.mark.parametrize("name", ["c1", "c2_subset", "random_small", "on_lattice"])
def test_lattice_from_spectra_fused(name):
    """K1b fused into K3: identical to K1 -> K3 (same per-bin psi rounding,
    same accumulation order) and to the reference lattice; the tf32 split
    outputs equal srpb_tf32_split of Xi bitwise."""
    g = load_golden(name)
    Y = dev(g["Y"])
    for n_aux in g["n_aux"]:
        plan = plan_from_golden(g, int(n_aux))
        for kw in ({}, {"weighting": "identity"}, {"phat_floor": 1e-3}):
            two_step = plan.lattice(plan.cross_spectra(Y, **kw)[0])
            fused = plan.lattice_from_spectra(Y, **kw)
            assert torch.equal(fused, two_step), (name, n_aux, kw)
            hi, lo = plan.lattice_from_spectra(Y, split=True, **kw)
            h2, l2 = plan.split_tf32(fused)
            assert torch.equal(hi, h2) and torch.equal(lo, l2)
        xi = plan.lattice_from_spectra(Y).cpu().numpy()
        total = plan.total_samples
        assert np.all(xi[:, total:] == 0.0)
        for f in range(xi.shape[0]):
            assert rel_l2(xi[f, :total], g[f"lattice_{n_aux}"][f]) <= REL_L2_TOL


def test_speculative_floor_fixup_frames():
    """The relative PHAT floor is applied speculatively inside the fused
    lattice; frames where a bin falls below the floor (powers in range),
    where powers leave the fast range, or that are all zero must still match
    the exact two-step path (fp64 floor in K1) and the oracle."""
    g = load_golden("random_small")
    Y = g["Y"].astype(np.complex64).copy()          # [3, 5, 64]
    Y = np.concatenate([Y, Y[:1], Y[:1]])            # 5 frames
    Y[0, 1, 7] = 1e-13 + 0j                          # |raw| tiny but powers in range
    Y[0, 2, 7] = 1e-12 + 0j
    Y[1, 0, 3] = 1e-20 + 1e-20j                      # power out of the fast range
    Y[3] = 0                                         # all-zero frame
    Y[4, :, 5] = 0                                   # exact-zero bin
    plan = plan_from_golden(g, 3)
    Yd = dev(Y)
    fused = plan.lattice_from_spectra(Yd).cpu().numpy()
    exact = plan.lattice(plan.cross_spectra(Yd)[0]).cpu().numpy()
    total = plan.total_samples
    for f in range(Y.shape[0]):
        ref = np.concatenate(O.gcc_lattice(O.cross_spectrum(Y[f].astype(complex), g["pair_m"],
                                                            g["pair_mp"])[0],
                                           g["omega"], g["bounds"], T, 3)[1])
        if f == 3:
            assert np.all(fused[f] == 0.0) and np.all(ref == 0.0)
            continue
        assert rel_l2(fused[f, :total], ref) <= REL_L2_TOL, f
        assert rel_l2(fused[f, :total], exact[f, :total]) <= REL_L2_TOL, f
    assert np.array_equal(fused[2], exact[2])  # an untouched frame: bitwise the exact path


def _xi16(plan, Y):
    hi, lo = plan.lattice_from_spectra(Y, split="f16")
    return ((hi.double() + lo.double()) / plan.xi_scale16).cpu().numpy()


@pytest.mark.parametrize("name", ["c1", "c2_subset", "random_small", "on_lattice"])
def test_lattice_tensor_core_matches_simt_and_reference(name):
    """K1b + K3 as one tcgen05 GEMM over (frame, pair) rows (PHAT, fp16
    split output) vs the SIMT fused lattice and the reference lattice;
    pad columns zero; bitwise repeatable."""
    g = load_golden(name)
    Y = dev(g["Y"])
    for n_aux in g["n_aux"]:
        plan = plan_from_golden(g, int(n_aux))
        assert plan.lattice_tc, (name, plan.Kb, plan.L)
        from paper_2012_09499_b200 import _native as NN
        served = NN.query("srpb_lattice_tc_supported", Y.shape[1], plan.P, plan.Kb, plan.L,
                          plan.T_pad)
        assert served or name == "random_small", name  # random_small: N = 64, 14-frame tiles
        tc = _xi16(plan, Y)
        assert np.array_equal(tc, _xi16(plan, Y))
        plan.lattice_tc = False
        simt = _xi16(plan, Y)
        plan.lattice_tc = True
        total = plan.total_samples
        assert np.all(tc[:, total:] == 0.0)
        for f in range(tc.shape[0]):
            assert rel_l2(tc[f, :total], simt[f, :total]) <= 3e-6, (name, n_aux, f)
            assert rel_l2(tc[f, :total], g[f"lattice_{n_aux}"][f]) <= REL_L2_TOL


def test_lattice_tensor_core_fixup_frames_and_ragged_rows():
    """Speculative-floor edge frames through the tensor-core lattice (the
    fix-up pass redoes them exactly), F x P not a multiple of the 128-row
    tile, odd bin-block count per CTA half."""
    g = load_golden("random_small")
    Y = g["Y"].astype(np.complex64).copy()          # [3, 5, 64]
    Y = np.concatenate([Y, Y[:1], Y[:1]] + [Y] * 4)  # 17 frames x 10 pairs = 170 rows
    Y[0, 1, 7] = 1e-13 + 0j
    Y[0, 2, 7] = 1e-12 + 0j
    Y[1, 0, 3] = 1e-20 + 1e-20j
    Y[3] = 0
    Y[4, :, 5] = 0
    plan = plan_from_golden(g, 3)
    assert plan.lattice_tc
    Yd = dev(Y)
    tc = _xi16(plan, Yd)
    total = plan.total_samples
    for f in range(Y.shape[0]):
        ref = np.concatenate(O.gcc_lattice(O.cross_spectrum(Y[f].astype(complex), g["pair_m"],
                                                            g["pair_mp"])[0],
                                           g["omega"], g["bounds"], T, 3)[1])
        if f == 3:
            assert np.all(tc[f] == 0.0) and np.all(ref == 0.0)
            continue
        assert rel_l2(tc[f, :total], ref) <= REL_L2_TOL, f
    # 3 bin blocks (Kb = 96): CTA halves of 2 and 1 blocks
    rng = np.random.default_rng(3)
    omega = np.arange(96) * (2 * np.pi * 16000.0 / 192.0)
    pairs = O.canonical_pairs(4)
    pm = np.array([a for a, _ in pairs], np.int32)
    pmp = np.array([b for _, b in pairs], np.int32)
    bounds = np.full(len(pairs), 5e-4)
    tdoa = rng.uniform(-1, 1, (9, len(pairs))) * bounds
    p2 = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=T, n_aux=2)
    assert p2.lattice_tc
    Y2 = (rng.standard_normal((40, 4, 96)) + 1j * rng.standard_normal((40, 4, 96))).astype(
        np.complex64)
    xi = _xi16(p2, dev(Y2))
    for f in (0, 21, 39):
        psi = O.cross_spectrum(Y2[f].astype(complex), pm, pmp)[0]
        ref = np.concatenate(O.gcc_lattice(psi, omega, bounds, T, 2)[1])
        assert rel_l2(xi[f, : p2.total_samples], ref) <= REL_L2_TOL


def test_lattice_from_spectra_odd_bins_and_ragged_tiles():
    """Odd Kb (partial bin chunk), F not a multiple of the 64-frame tile,
    reach > 32 lags (several lag tiles) vs the oracle."""
    rng = np.random.default_rng(7)
    M, Kb, F = 5, 77, 70
    pairs = O.canonical_pairs(M)
    pm = np.array([m for m, _ in pairs], np.int32)
    pmp = np.array([mp for _, mp in pairs], np.int32)
    bounds = rng.uniform(1e-3, 3e-3, len(pairs))  # up to 48 samples -> T_p up to 101
    omega = np.arange(1, Kb + 1) * (2 * np.pi * 16000.0 / 200.0)
    tdoa = rng.uniform(-1, 1, (9, len(pairs))) * bounds
    Y = (rng.standard_normal((F, M, Kb)) + 1j * rng.standard_normal((F, M, Kb))).astype(np.complex64)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=T, n_aux=3)
    xi = plan.lattice_from_spectra(dev(Y)).cpu().numpy()
    for f in (0, 37, 69):
        psi = O.cross_spectrum(Y[f].astype(complex), pm, pmp)[0]
        ref = np.concatenate(O.gcc_lattice(psi, omega, bounds, T, 3)[1])
        assert rel_l2(xi[f, : plan.total_samples], ref) <= REL_L2_TOL
    assert np.all(xi[:, plan.total_samples:] == 0.0)


# --------------------------------------------------------------------- W
def test_sinc_table_matches_reference():
    g = load_golden("random_small")
    plan = plan_from_golden(g, 1, weights="stored")
    W = plan.W.cpu().numpy()
    ref = g["sinc_w_1"]
    assert np.max(np.abs(W[:, : ref.shape[1]] - ref)) < 1e-6
    assert np.all(W[:, ref.shape[1]:] == 0.0)


def test_sinc_table_exact_indicator_rows():
    g = load_golden("sinc_integer")
    plan = SrpPlan(g["tdoa"], [1], [0], g["bounds"], np.array([0.0, 1.0]), sample_period=T,
                   n_aux=0, weights="stored")
    W = plan.W.cpu().numpy()[:, : g["weights"].shape[1]]
    assert np.array_equal(W, g["weights"].astype(np.float32))


# --------------------------------------------------------------------- K4
@pytest.mark.parametrize("weights", ["stored-simt", "stored-tc", "onthefly"])
@pytest.mark.parametrize("name", ["c1", "c2_subset", "random_small", "on_lattice"])
def test_approx_matches_reference(name, weights):
    g = load_golden(name)
    psi = dev(g["psi"].astype(np.complex64))
    w, backend = (weights.split("-") + ["simt"])[:2]
    for n_aux in g["n_aux"]:
        plan = plan_from_golden(g, int(n_aux), weights=w, backend=backend)
        maps, am = plan.approx(plan.lattice(psi))
        assert_maps_match(maps.cpu().numpy(), g[f"approx_{n_aux}"], am.cpu().numpy(),
                          what=f"{name} n_aux={n_aux} {weights}")
        if name in ("c1", "c2_subset"):
            assert list(am.cpu().numpy()) == list(g[f"argmax_approx_{n_aux}"])


def test_approx_exact_on_lattice():
    """Acceptance criterion 4: on-lattice TDOAs reconstruct the exact map."""
    g = load_golden("on_lattice")
    psi = dev(g["psi"].astype(np.complex64))
    plan = plan_from_golden(g, 0)
    maps, _ = plan.approx(plan.lattice(psi))
    conv, _ = plan_from_golden(g).conventional(psi)
    for f in range(maps.shape[0]):
        assert rel_l2(maps[f].cpu().numpy(), conv[f].cpu().numpy()) <= REL_L2_TOL


# ------------------------------------------------------- end to end (Y -> maps)
@pytest.mark.parametrize("path", ["conventional", "approx"])
def test_end_to_end_from_stft(path):
    g = load_golden("c1")
    plan = plan_from_golden(g, 2)
    maps, am = plan.run(dev(g["Y"]), path=path)
    ref = g["conv"] if path == "conventional" else g["approx_2"]
    refam = g["argmax_conv"] if path == "conventional" else g["argmax_approx_2"]
    assert_maps_match(maps.cpu().numpy(), ref, am.cpu().numpy(), what=path)
    assert list(am.cpu().numpy()) == list(refam)


@pytest.mark.parametrize("precision", ["auto", "tf32"])
@pytest.mark.parametrize("name", ["c1", "c2_subset", "random_small", "on_lattice"])
def test_run_tensor_core_precisions(name, precision):
    """Y -> maps through the tensor-core engine in 3xFP16 (PHAT-bounded
    operands, default) and 3xTF32, both paths, vs the reference."""
    g = load_golden(name)
    Y = dev(g["Y"])
    if g["omega"].size % 32:
        pytest.skip("3xFP16 conventional kernel needs Kb % 32 == 0")
    for n_aux in g["n_aux"]:
        plan = SrpPlan(g["tdoa"], g["pair_m"], g["pair_mp"], g["bounds"], g["omega"],
                       sample_period=T, n_aux=int(n_aux), weights="stored", backend="tc",
                       precision=precision)
        maps, am = plan.run(Y, "approx")
        assert_maps_match(maps.cpu().numpy(), g[f"approx_{n_aux}"], am.cpu().numpy(),
                          what=f"{name} n_aux={n_aux} {precision} approx")
        if name in ("c1", "c2_subset"):
            assert list(am.cpu().numpy()) == list(g[f"argmax_approx_{n_aux}"])
    maps, am = plan.run(Y, "conventional")
    assert_maps_match(maps.cpu().numpy(), g["conv"], am.cpu().numpy(),
                      what=f"{name} {precision} conventional")
    if name in ("c1", "c2_subset"):
        assert list(am.cpu().numpy()) == list(g["argmax_conv"])


@pytest.mark.parametrize("name", ["c1", "c2_subset", "random_small", "on_lattice"])
def test_tc16_onthefly_weights_bitwise_equal_stored(name):
    """K4 with the sinc weights generated in tensor memory equals the
    stored-W 3xFP16 kernel bit for bit (same weight arithmetic and split),
    and both match the reference."""
    g = load_golden(name)
    Y = dev(g["Y"])
    for n_aux in g["n_aux"]:
        st = plan_from_golden(g, int(n_aux), weights="stored", backend="tc")
        ot = plan_from_golden(g, int(n_aux), weights="onthefly", backend="tc")
        assert ot.W is None
        m1, a1 = st.run(Y, "approx")
        m2, a2 = ot.run(Y, "approx")
        assert torch.equal(m1, m2) and torch.equal(a1, a2), (name, n_aux)
        assert_maps_match(m2.cpu().numpy(), g[f"approx_{n_aux}"], a2.cpu().numpy(),
                          what=f"{name} onthefly-tc16")


def test_captured_step_and_chunked_runner_match_eager():
    """CUDA-graph replay (CapturedStep) and the 3-stream chunked host
    pipeline give bitwise the same maps/argmax as the eager plan.run."""
    g = load_golden("c2_subset")
    Y = np.concatenate([g["Y"]] * 40)  # 120 frames: 3 chunks of >= 32
    plan = plan_from_golden(g, 4, weights="stored", backend="tc")
    for path in ("approx", "conventional"):
        ref_maps, ref_am = plan.run(dev(Y), path)
        cap = plan.capture(Y.shape[0], Y.shape[1], path)
        m, a = cap.replay(dev(Y))
        assert cap.launches >= 2
        assert torch.equal(m, ref_maps) and torch.equal(a, ref_am)
        m2, a2 = cap.replay()  # replays are repeatable
        assert torch.equal(m2, ref_maps) and torch.equal(a2, ref_am)
        runner = B.ChunkedRunner(plan, Y.shape[0], Y.shape[1], path, chunks=3)
        assert len(runner.bounds) == 3
        Yh = torch.from_numpy(Y).pin_memory()
        mh = torch.empty(tuple(ref_maps.shape), dtype=torch.float32).pin_memory()
        ah = torch.empty(Y.shape[0], dtype=torch.int32).pin_memory()
        for _ in range(2):  # back-to-back calls reuse the static buffers safely
            runner.run(Yh, mh, ah)
        torch.cuda.synchronize()
        assert torch.equal(mh, ref_maps.cpu()) and torch.equal(ah, ref_am.cpu())


def test_graph_replay_after_launches_of_other_widths():
    """A captured step replays unchanged after eager launches of the same
    kernels with other frame counts (other tile widths, stage counts and
    dynamic shared memory sizes)."""
    g = load_golden("c2_subset")
    Y = np.concatenate([g["Y"]] * 60)  # 180 frames: two frame tiles
    plan = plan_from_golden(g, 4, weights="stored", backend="tc")
    for path in ("approx", "conventional"):
        ref_maps, ref_am = plan.run(dev(Y), path)
        cap = plan.capture(Y.shape[0], Y.shape[1], path)
        for f in (1, 7, 33):
            plan.run(dev(Y[:f]), path)
        m, a = cap.replay(dev(Y))
        torch.cuda.synchronize()
        assert torch.equal(m, ref_maps) and torch.equal(a, ref_am)


def test_argmax_only_mode_matches_maps_mode():
    g = load_golden("c2_subset")
    plan = plan_from_golden(g, 4)
    Y = dev(g["Y"])
    m1, a1 = plan.run(Y, "approx", maps=True)
    m0, a0 = plan.run(Y, "approx", maps=False)
    assert m0 is None and torch.equal(a0, a1)
    assert torch.equal(B.standalone_argmax(m1), a1)


# -------------------------------------------- larger seeded shapes vs oracle
def _oracle_case(scene, J, F, n_aux, weights="auto"):
    pairs = O.canonical_pairs(scene.mic_pos.shape[0])
    pm = np.array([m for m, _ in pairs], np.int32)
    pmp = np.array([mp for _, mp in pairs], np.int32)
    c = scene.speed_of_sound
    bounds = np.array([np.linalg.norm(scene.mic_pos[m] - scene.mic_pos[mp]) / c for m, mp in pairs])
    grid = scene.grid[np.linspace(0, scene.grid.shape[0] - 1, J).astype(int)]
    tdoa = O.tdoa_table_nearfield(scene.mic_pos, grid, pairs, c)
    omega = O.bin_frequencies(16000.0, scene.frame_length)
    Y = scene.Y[:F]
    psi = np.stack([O.cross_spectrum(Y[f].astype(complex), pm, pmp)[0] for f in range(F)])
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=T, n_aux=n_aux, weights=weights)
    return plan, psi, omega, tdoa, bounds, Y


@pytest.mark.parametrize("backend", ["simt", "tc"])
@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_config_shapes_vs_oracle(cfg, backend):
    """Full-K contractions (all pairs, all bins) of every config on a
    candidate/frame subset: accumulation error over C3/C4's long K."""
    if cfg == "c2":
        scene, J, F, n_aux, w = scenes.make_c2(num_frames=6), 3000, 6, 4, "stored"
    elif cfg == "c3":
        scene, J, F, n_aux, w = scenes.make_c3(num_frames=3), 800, 3, 8, "stored"
    else:
        scene, J, F, n_aux, w = scenes.make_c4(num_frames=2), 300, 2, 2, (
            "onthefly" if backend == "simt" else "stored")
    plan, psi, omega, tdoa, bounds, Y = _oracle_case(scene, J, F, n_aux, w)
    plan.backend = backend
    psi_g, _ = plan.cross_spectra(dev(Y))
    assert np.max(np.abs(psi_g.cpu().numpy() - psi)) < 2e-6
    conv_ref = O.conventional_frames(psi, omega, tdoa, candidate_chunk=512)
    conv, am = plan.conventional(psi_g)
    assert_maps_match(conv.cpu().numpy(), conv_ref, am.cpu().numpy(), what=f"{cfg} conv")
    _, wts = O.sinc_table(tdoa, bounds, T, n_aux)
    approx_ref = np.stack([O.approx_map(wts, O.gcc_lattice(psi[f], omega, bounds, T, n_aux)[1])
                           for f in range(F)])
    maps, am = plan.approx(plan.lattice(psi_g))
    assert_maps_match(maps.cpu().numpy(), approx_ref, am.cpu().numpy(), what=f"{cfg} approx")
    maps, am = plan.run(dev(Y), "approx")  # fused K1b/K3 front end
    assert_maps_match(maps.cpu().numpy(), approx_ref, am.cpu().numpy(), what=f"{cfg} run")


# --------------------------------------------- device geometry (plan build)
def test_plan_from_geometry_matches_host_table():
    """TDOAs + phase/sinc splits computed on the device equal the host path
    (reference operation order, fp64): identical splits, identical maps."""
    scene = scenes.make_c2(num_frames=4)
    pts = scene.grid[::7]
    arr = B.MicArray(scene.mic_pos, speed_of_sound=343.0)
    grid = B.build_tdoa_table(arr, B.CandidateGrid("near_field", pts))
    pm = np.array([p.index_m for p in arr.pairs], np.int32)
    pmp = np.array([p.index_m_prime for p in arr.pairs], np.int32)
    bounds = np.array([p.tdoa_bound for p in arr.pairs])
    omega = O.bin_frequencies(16000.0, 1024)
    host = SrpPlan(grid.tdoa_table, pm, pmp, bounds, omega, sample_period=T, n_aux=4,
                   weights="stored")
    devp = SrpPlan.from_geometry(scene.mic_pos, pts, omega, speed_of_sound=343.0,
                                 sample_period=T, n_aux=4, weights="stored")
    for name in ("conv_ti", "conv_tf", "sx_i", "sx_f"):
        a, b = getattr(host, name), getattr(devp, name)
        mism = int((a != b).sum().item())
        assert mism <= a.numel() // 100000, (name, mism)  # exact up to rare rounding ties
    Y = dev(scene.Y)
    for path in ("approx", "conventional"):
        m1, a1 = host.run(Y, path)
        m2, a2 = devp.run(Y, path)
        assert_maps_match(m2.cpu().numpy(), m1.cpu().numpy(), a2.cpu().numpy(), what=path)
    # far field (unit directions) against the host table
    dirs = np.random.default_rng(2).standard_normal((500, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    gf = B.build_tdoa_table(arr, B.CandidateGrid("far_field", dirs))
    pf = SrpPlan.from_geometry(scene.mic_pos, dirs, omega, speed_of_sound=343.0, far_field=True)
    hf = SrpPlan(gf.tdoa_table, pm, pmp, bounds, omega)
    assert int((pf.conv_ti != hf.conv_ti).sum().item()) <= 2
    assert float((pf.conv_tf - hf.conv_tf).abs().max().item()) < 1e-6
    # a point outside the physical bound raises like the reference
    with pytest.raises(AssertionError, match="exceeded"):
        SrpPlan.from_geometry(scene.mic_pos, dirs * 2.0, omega, speed_of_sound=343.0,
                              far_field=True)


# ------------------------------------ size-independent properties at full C2
def test_full_c2_frame_sharding_and_determinism():
    """BASELINE config C2 at full size (J=50k, F=311): maps are independent
    of how frames are batched (the sharding invariant), bitwise repeatable,
    and the fused argmax equals the standalone K5 over the stored maps."""
    scene = scenes.make_c2()
    pairs = O.canonical_pairs(8)
    pm = np.array([m for m, _ in pairs], np.int32)
    pmp = np.array([mp for _, mp in pairs], np.int32)
    bounds = np.array([np.linalg.norm(scene.mic_pos[m] - scene.mic_pos[mp]) / 343.0
                       for m, mp in pairs])
    tdoa = O.tdoa_table_nearfield(scene.mic_pos, scene.grid, pairs, 343.0)
    omega = O.bin_frequencies(16000.0, 1024)
    # one kernel for every shard (auto would send a < 32-frame shard to SIMT)
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=T, n_aux=4, backend="tc")
    Y = dev(scene.Y)
    assert Y.shape == (311, 8, 512) and plan.J == 50000
    for path in ("approx", "conventional"):
        full, am = plan.run(Y, path)
        again, am2 = plan.run(Y, path)
        assert torch.equal(full, again) and torch.equal(am, am2)
        parts = [plan.run(Y[lo:lo + 100].contiguous(), path) for lo in range(0, 311, 100)]
        assert torch.equal(torch.cat([p[0] for p in parts]), full)
        assert torch.equal(torch.cat([p[1] for p in parts]), am)
        assert torch.equal(B.standalone_argmax(full), am)
    # spot-check two frames against the oracle at full J
    sel = [0, 200]
    psi = np.stack([O.cross_spectrum(scene.Y[f].astype(complex), pm, pmp)[0] for f in sel])
    conv_ref = O.conventional_frames(psi, omega, tdoa, candidate_chunk=4096)
    conv, _ = plan.run(Y, "conventional")
    for i, f in enumerate(sel):
        assert rel_l2(conv[f].cpu().numpy(), conv_ref[i]) <= REL_L2_TOL
        assert int(np.argmax(conv_ref[i])) == int(torch.argmax(conv[f]).item())


@pytest.mark.parametrize("path", ["approx", "conventional"])
def test_candidate_sharding_batch1(path):
    """C5-style batch 1: the candidate-range plans two ranks
    would hold reproduce the full plan's maps bitwise, and their packed keys
    reduce (MAX, as the all-reduce does) to the full plan's argmax."""
    from paper_2012_09499_b200 import distributed as D
    scene = scenes.make_c2(num_frames=3)
    pairs = O.canonical_pairs(8)
    pm = np.array([a for a, _ in pairs], np.int32)
    pmp = np.array([b for _, b in pairs], np.int32)
    bounds = np.array([np.linalg.norm(scene.mic_pos[a] - scene.mic_pos[b]) / 343.0
                       for a, b in pairs])
    tdoa = O.tdoa_table_nearfield(scene.mic_pos, scene.grid, pairs, 343.0)
    omega = O.bin_frequencies(16000.0, 1024)
    J = tdoa.shape[0]
    full = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=T, n_aux=4)
    for F in (1, 3):
        Y = dev(scene.Y[:F])
        m_full, a_full = full.run(Y, path)
        maps, keys = [], []
        for lo, hi in D.candidate_ranges(J, 2):
            p = SrpPlan(tdoa[lo:hi], pm, pmp, bounds, omega, sample_period=T, n_aux=4)
            m, a = D.run_candidate_sharded(p, Y, lo, J, path)  # no process group: local
            assert int(a.min()) >= lo and int(a.max()) < hi
            maps.append(m)
            keys.append(D.keys_to_signed(D.keys_from_maps(m, a.long() - lo, lo)))
        assert torch.equal(torch.cat(maps, dim=1), m_full)
        red = D.keys_from_signed(torch.maximum(keys[0], keys[1]))
        assert torch.equal(D.keys_index(red).to(torch.int32), a_full)


def test_lattice_tensor_core_in_kernel_fixup():
    """The speculative-floor fix-up run inside the tensor-core lattice (the
    CTA completing a frame tests it and redoes it exactly) equals the
    separate fix-up kernel bitwise, leaves its frame counters zero, and
    matches the oracle on edge frames."""
    g = load_golden("c2_subset")
    Y = g["Y"].astype(np.complex64)                  # [3, 8, 512]
    Y = np.concatenate([Y] * 4)                      # 12 frames x 28 pairs: 3 row tiles
    Y[0, 1, 7] = 1e-13 + 0j                          # |raw| below the floor, powers in range
    Y[0, 2, 7] = 1e-12 + 0j
    Y[1, 0, 3] = 1e-20 + 1e-20j                      # power out of the fast range
    Y[2] = 0                                         # all-zero frame
    Y[3, :, 5] = 0                                   # exact-zero bin
    Y[9, 4, 100] = 1e-14 + 0j                        # a frame straddling two row tiles
    n_aux = int(g["n_aux"][-1])
    plan = plan_from_golden(g, n_aux)
    from paper_2012_09499_b200 import _native as NN
    assert NN.query("srpb_lattice_tc_supported", Y.shape[1], plan.P, plan.Kb, plan.L, plan.T_pad)
    Yd = dev(Y)
    plan.lattice_fixup_fused = True
    fused = _xi16(plan, Yd)
    assert np.array_equal(fused, _xi16(plan, Yd))
    assert int(plan._frame_counters(Y.shape[0]).abs().sum().item()) == 0
    plan.lattice_fixup_fused = False
    sep = _xi16(plan, Yd)
    plan.lattice_fixup_fused = True
    assert np.array_equal(fused, sep)
    total = plan.total_samples
    for f in range(Y.shape[0]):
        ref = np.concatenate(O.gcc_lattice(O.cross_spectrum(Y[f].astype(complex), g["pair_m"],
                                                            g["pair_mp"])[0],
                                           g["omega"], g["bounds"], T, n_aux)[1])
        if f == 2:
            assert np.all(fused[f] == 0.0) and np.all(ref == 0.0)
            continue
        assert rel_l2(fused[f, :total], ref) <= REL_L2_TOL, f


@pytest.mark.parametrize("kbg", [1, 4])
def test_conventional_generator_short_drain_periods_full_width(kbg):
    """K2's phase generators fold accumulator chunks while generating; drain
    periods shorter than a group's chunk count must not stall the ring
    (the launcher widens them): full-width frame tiles (F = 311 -> N = 160),
    tf32 and fp16 operand splits, vs the oracle on a candidate subset."""
    scene = scenes.make_c2()
    pairs = O.canonical_pairs(8)
    pm = np.array([a for a, _ in pairs], np.int32)
    pmp = np.array([b for _, b in pairs], np.int32)
    bounds = np.array([np.linalg.norm(scene.mic_pos[a] - scene.mic_pos[b]) / 343.0
                       for a, b in pairs])
    tdoa = O.tdoa_table_nearfield(scene.mic_pos, scene.grid[::25], pairs, 343.0)  # J = 2000
    omega = O.bin_frequencies(16000.0, 1024)
    Y = dev(scene.Y)
    ref = None
    for precision in ("auto", "tf32"):
        plan = SrpPlan(tdoa, pm, pmp, bounds, omega, backend="tc", precision=precision,
                       kb_per_group=kbg)
        maps, am = plan.run(Y, "conventional")
        m = maps.cpu().numpy()
        if ref is None:
            sel = [0, 155, 310]
            psi = np.stack([O.cross_spectrum(scene.Y[f].astype(complex), pm, pmp)[0] for f in sel])
            ref = O.conventional_frames(psi, omega, tdoa)
        for i, f in enumerate(sel):
            assert rel_l2(m[f], ref[i]) <= REL_L2_TOL, (precision, kbg, f)


def test_conventional_fused_split_equals_two_step():
    """run(..., "conventional") has K1 write the fp16 operand split directly
    (srpb_gcc_phat_split16); it must equal psi -> srpb_f16_split -> K2 bit
    for bit, and the launch count drops by the split pass."""
    from paper_2012_09499_b200 import _native as NN
    g = load_golden("c2_subset")
    plan = plan_from_golden(g, 4, backend="tc")
    Y = dev(np.concatenate([g["Y"]] * 12).astype(np.complex64))  # 36 frames: tensor-core K2
    n0 = NN.launch_count()
    m1, a1 = plan.run(Y, "conventional")
    fused = NN.launch_count() - n0
    psi, _ = plan.cross_spectra(Y)
    n0 = NN.launch_count()
    m2, a2 = plan.conventional(psi, _bounded=True)  # PHAT psi: the 3xFP16 K2 as well
    two = NN.launch_count() - n0
    assert torch.equal(m1, m2) and torch.equal(a1, a2)
    # K1's frame-resident single pass (floor, psi16) + K2 vs split + K2 (after K1)
    assert fused == 2 and two == 2


def test_concurrent_steps_of_one_plan_own_their_kernel_state():
    """Two captured steps of the same plan and frame count, replayed
    concurrently on two streams, and eager calls on a third: each owns its
    argmax keys and item cursor (ADVICE: shared per-F state let concurrent
    grids advance one cursor), so every result equals the serial one."""
    g = load_golden("c2_subset")
    Y = dev(np.concatenate([g["Y"]] * 12).astype(np.complex64))  # 36 frames
    plan = plan_from_golden(g, 4, weights="stored", backend="tc")
    for path in ("approx", "conventional"):
        ref_m, ref_a = plan.run(Y, path)
        c1 = plan.capture(Y.shape[0], Y.shape[1], path)
        c2 = plan.capture(Y.shape[0], Y.shape[1], path)
        c1.Y.copy_(Y)
        c2.Y.copy_(Y)
        torch.cuda.synchronize()
        s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        eager = []
        for _ in range(4):
            with torch.cuda.stream(s1):
                c1.replay()
            with torch.cuda.stream(s2):
                c2.replay()
            with torch.cuda.stream(s3):
                eager.append(plan.run(Y, path))
        torch.cuda.synchronize()
        for m, a in [(c1.maps, c1.argmax), (c2.maps, c2.argmax)] + eager:
            assert torch.equal(m, ref_m) and torch.equal(a, ref_a), path


def test_dropin_argmax_only_and_small_bin_tables():
    """srp_approx_frames(..., maps=False) returns argmax-only maps equal to the
    full maps' argmax; a sinc table built without bin frequencies takes the
    fp16 prescale from the lattice's own bins (no overflow for Kb < 512)."""
    g = load_golden("random_small")
    arr = B.MicArray(g["mic_pos"], speed_of_sound=float(g["speed_of_sound"]))
    grid = B.build_tdoa_table(arr, B.CandidateGrid("near_field", g["grid"]))
    freqs = g["omega"]
    frames = [B.SpectralFrame(g["Y"][f].astype(complex), freqs, frame_index=f)
              for f in range(g["Y"].shape[0])]
    crosses = B.cross_spectrum_frames(frames, arr.pairs)
    lats = B.build_gcc_lattice_frames(crosses, T, 1)
    table = B.precompute_sinc_table(grid, arr.pairs, T, 1)  # Kb-agnostic table plan
    full = B.srp_approx_frames(lats, table)
    am = B.srp_approx_frames(lats, table, maps=False)
    got = np.stack([m.values for m in full])
    assert_maps_match(got, g["approx_1"], [B.argmax_candidate(m) for m in full],
                      what="drop-in approx (64 bins)")
    for mf, ma in zip(full, am):
        assert B.argmax_candidate(ma) == B.argmax_candidate(mf) == int(np.argmax(mf.values))
        with pytest.raises(ValueError, match="maps=False"):
            _ = ma.values
