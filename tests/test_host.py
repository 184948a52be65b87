"""CPU tests of the host side: the C ABI library (loads, exports every symbol
of include/srpb.h, rejects invalid arguments before any launch), the plan's
layout arithmetic, the geometry/host constants, the closed-form counters and
the drop-in API's validation errors (same types/messages as the reference).
No kernel runs here."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2012_09499_b200 as B
from paper_2012_09499_b200 import _native, scenes
from paper_2012_09499_b200.plan import is_harmonic, lattice_layout, split_rint
from oracle import srp_oracle as O

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
T = 1.0 / 16000.0


def header_symbols():
    src = open(os.path.join(ROOT, "include", "srpb.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(srpb_\w+)\s*\(", src, re.M)))


# ----------------------------------------------------------------- C ABI
def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_native.lib_path())
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.exported_symbols())


def test_abi_version_and_error_reporting_without_gpu():
    lib = _native.load()
    assert lib.srpb_abi_version() == 13
    # invalid arguments are rejected on the host before any CUDA call
    with pytest.raises(ValueError, match="bad shape"):
        _native.call("srpb_gcc_phat", None, -1, 4, 64, None, None, 6, 0, 1e-12, -1.0, None, None,
                     None)
    with pytest.raises(ValueError, match="unknown weighting"):
        _native.call("srpb_gcc_phat", None, 1, 4, 64, None, None, 6, 7, 1e-12, -1.0, None, None,
                     None)
    with pytest.raises(ValueError, match="multiple of 32"):
        _native.call("srpb_interp", None, None, 1, 10, 33, None, None, None)
    with pytest.raises(ValueError, match="multiple of 16"):
        _native.call("srpb_conventional_tc", None, None, 1, 6, 40, 80, None, None, 10, None, None,
                     4, None)
    with pytest.raises(ValueError, match="maps and/or keys"):
        _native.call("srpb_conventional", None, 0, 6, 64, 128, None, None, 10, None, None, None)
    assert b"maps and/or keys" in lib.srpb_last_error()


# --------------------------------------------------------- plan arithmetic
@pytest.mark.parametrize("n_aux", [0, 1, 2, 4, 8])
def test_lattice_layout_matches_reference_counts(n_aux):
    g = np.load(os.path.join(ROOT, "tests", "golden", "c2_subset.npz"))
    halves, reach, off, total, t_pad = lattice_layout(g["bounds"], T, n_aux)
    assert list(halves) == list(O.lattice_half_counts(g["bounds"], T))
    assert list(reach) == [h + n_aux for h in halves]
    assert off[0] == 0 and off[-1] == total == sum(2 * (h + n_aux) + 1 for h in halves)
    assert t_pad % 32 == 0 and t_pad - 32 < total <= t_pad
    if n_aux in (0, 2, 4):
        assert total == {0: 372, 2: 484, 4: 596}[n_aux]  # BASELINE.md sizes for C2


def test_lattice_layout_validation():
    with pytest.raises(ValueError, match="sample_period"):
        lattice_layout([1e-4], 0.0, 1)
    with pytest.raises(ValueError, match="n_aux"):
        lattice_layout([1e-4], T, -1)


def test_split_rint_reconstructs():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-400, 400, 10000), np.arange(-5, 6, dtype=float),
                        np.array([0.5, -0.5, 2.5, 1e-17])])
    i, f = split_rint(x)
    assert np.all(np.abs(f) <= 0.5)
    assert np.allclose(i + f.astype(float), x, atol=1e-5)
    assert np.all(f[np.isin(x, np.arange(-5, 6))] == 0.0)  # exact nodes stay exact


def test_harmonic_detection_matches_reference_rule():
    assert is_harmonic(O.bin_frequencies(16000.0, 1024))
    assert not is_harmonic(np.array([0.0]))
    assert not is_harmonic(np.sort(np.random.default_rng(1).uniform(0, 1e4, 32)))
    assert not is_harmonic(O.bin_frequencies(16000.0, 1024) + 1.0)


# ------------------------------------------------------------- geometry
def test_geometry_pairs_and_tdoa_table_match_oracle():
    arr = B.circular_array(6, 0.1, center=(2.9, 3.4, 3.3), speed_of_sound=340.0)
    assert [(p.index_m, p.index_m_prime) for p in arr.pairs] == O.canonical_pairs(6)
    dists = sorted(round(p.distance, 12) for p in arr.pairs)
    expected = sorted([0.1] * 6 + [round(0.1 * math.sqrt(3.0), 12)] * 6 + [0.2] * 3)
    np.testing.assert_allclose(dists, expected, rtol=1e-12)
    pts = np.random.default_rng(3).uniform(0, 5, (50, 3))
    grid = B.build_tdoa_table(arr, B.CandidateGrid("near_field", pts))
    ref = O.tdoa_table_nearfield(arr.positions, pts, O.canonical_pairs(6), 340.0)
    np.testing.assert_allclose(grid.tdoa_table, ref, rtol=0, atol=1e-18)
    for p_idx, p in enumerate(arr.pairs):
        assert B.tdoa_nearfield(arr, p, pts[3]) == pytest.approx(grid.tdoa_table[3, p_idx], abs=1e-18)


def test_geometry_validation():
    with pytest.raises(ValueError):
        B.MicPair(1, 1, 0.1, 1e-4)
    with pytest.raises(ValueError, match="coincident"):
        B.MicArray([[0, 0, 0], [0, 0, 0]])
    with pytest.raises(ValueError, match="unit"):
        B.CandidateGrid("far_field", [[1.0, 1.0, 0.0]])
    with pytest.raises(ValueError, match="TDOA table"):
        B.CandidateGrid("near_field", [[1.0, 1.0, 0.0]]).require_table()


# ------------------------------------------- counters / complexity report
def test_complexity_report_acceptance_criterion_1():
    """tests/test_acceptance.py:66-89 of the reference."""
    arr = B.circular_array(6, 0.1, speed_of_sound=340.0)
    for n_aux in (0, 1, 2, 4, 8):
        rep = B.complexity_report(8101, 1024, arr.pairs, T, n_aux)
        assert rep.avg_samples_per_pair == 14.2 + 2.0 * n_aux
    rep = B.complexity_report(8101, 1024, arr.pairs, T, 2)
    assert rep.mults_conventional == 124_431_360
    assert rep.mults_sampling == 279_552
    assert rep.mults_interpolation == 2_211_573
    assert abs(rep.ratio_sampling - 2.25e-3) <= 0.01 * 2.25e-3
    assert abs(rep.ratio_interpolation - 1.78e-2) <= 0.01 * 1.78e-2
    d = rep.as_dict()
    assert d["half_counts"] == list(rep.half_counts)
    with pytest.raises(ValueError):
        B.complexity_report(0, 8, arr.pairs, T, 0)


def test_mult_counter_and_srpmap():
    a = B.MultCounter(complex_mults=3, real_mults=5)
    a.merge(B.MultCounter(complex_mults=10, real_mults=1))
    assert (a.complex_mults, a.real_mults) == (13, 6)
    a.reset()
    assert (a.complex_mults, a.real_mults) == (0, 0)
    m = B.SrpMap(np.array([1.0, 3.0, 3.0, 2.0]), "conventional")
    assert m.num_candidates == 4 and m.values.dtype == np.float64
    with pytest.raises(ValueError):
        B.SrpMap(np.zeros((2, 2)), "conventional")


# ------------------------------------------- drop-in validation (no GPU)
def test_dropin_validation_errors_precede_device_work():
    arr = B.circular_array(4, 0.1)
    freqs = 2 * np.pi * np.arange(64) * 16000.0 / 128.0
    frame = B.SpectralFrame(np.ones((2, 64), complex), freqs)
    with pytest.raises(ValueError, match="out of range"):
        B.cross_spectrum(frame, arr.pairs)
    with pytest.raises(ValueError, match="weighting"):
        B.cross_spectrum(frame, arr.pairs[:1], weighting="scot")
    with pytest.raises(ValueError):
        B.cross_spectrum(frame, ())
    with pytest.raises(ValueError):
        B.CrossSpectra(np.zeros((2, 8), complex), np.arange(8.0), arr.pairs, "phat")
    cross = B.CrossSpectra(np.ones((6, 64), complex), freqs, arr.pairs, "phat")
    with pytest.raises(ValueError, match="n_aux"):
        B.build_gcc_lattice(cross, T, -1)
    with pytest.raises(ValueError, match="sample_period"):
        B.lattice_half_counts(arr.pairs, 0.0)
    pts = np.random.default_rng(0).uniform(-1, 1, (5, 3))
    grid = B.build_tdoa_table(arr, B.CandidateGrid("near_field", pts))
    with pytest.raises(ValueError, match="pair columns"):
        B.precompute_sinc_table(grid, arr.pairs[:3], T, 1)
    with pytest.raises(ValueError, match="n_aux"):
        B.precompute_sinc_table(grid, arr.pairs, T, -2)
    lat = B.GccLattice(T, 1, B.lattice_half_counts(arr.pairs, T),
                       [np.zeros(2 * (h + 1) + 1) for h in B.lattice_half_counts(arr.pairs, T)])
    tab = B.SincTable(T, 2, B.lattice_half_counts(arr.pairs, T))
    with pytest.raises(ValueError, match="n_aux"):
        B.srp_approx(lat, tab)
    with pytest.raises(ValueError, match="spacing"):
        B.srp_approx(lat, B.SincTable(T / 2, 1, B.lattice_half_counts(arr.pairs, T)))
    with pytest.raises(ValueError):
        B.GccLattice(T, 0, (3,), [np.zeros(5)])
    bad = B.CrossSpectra(np.ones((3, 64), complex), freqs, arr.pairs[:3], "phat")
    with pytest.raises(ValueError, match="pairs"):
        B.srp_conventional_frames([bad], grid)


def test_spectral_framing_matches_reference_rules():
    spec = B.FrameSpec(16000.0, 1024)
    assert spec.hop_length == 512 and spec.num_bins == 512
    np.testing.assert_allclose(spec.bin_frequencies(), O.bin_frequencies(16000.0, 1024))
    assert spec.num_frames(160000) == 311
    with pytest.raises(ValueError):
        B.FrameSpec(16000.0, 1023)
    with pytest.raises(ValueError):
        spec.num_frames(100)
    win = spec.window_samples()
    n = np.arange(1024)
    np.testing.assert_allclose(win, np.sqrt(0.5 - 0.5 * np.cos(2 * np.pi * n / 1024)))
    # the STFT itself runs on the device (K0): tests/test_parity_gpu.py


# ----------------------------------------------------------- scenes
def test_scene_shapes_match_baseline_configs():
    c1 = scenes.make_c1()
    assert c1.Y.shape == (61, 4, 256) and c1.grid.shape == (1681, 3)
    c2 = scenes.make_c2(num_frames=4)
    assert c2.Y.shape == (4, 8, 512) and c2.grid.shape[0] == 50000
    assert scenes.box_grid(100, 100, 50, (10, 10, 5)).shape[0] == 500000
    assert scenes.box_grid(120, 100, 50, (6, 5, 3)).shape[0] == 600000
    c5 = scenes.make_c5(2, grid_limit=10)
    assert c5.Y.shape == (2, 8, 512) and c5.Y.dtype == np.complex64
    # seeded: identical on regeneration
    assert np.array_equal(scenes.make_c1(num_frames=2).Y, scenes.make_c1(num_frames=2).Y)


def test_chunk_bounds():
    from paper_2012_09499_b200.pipeline import chunk_bounds

    assert chunk_bounds(311, 4) == [(0, 78), (78, 156), (156, 234), (234, 311)]
    assert chunk_bounds(40, 4) == [(0, 40)]  # chunks keep >= 32 frames
    assert chunk_bounds(100, 3) == [(0, 34), (34, 67), (67, 100)]
    b = chunk_bounds(1000, 7)
    assert b[0][0] == 0 and b[-1][1] == 1000 and all(x[1] == y[0] for x, y in zip(b, b[1:]))
    # explicit chunk sizes (the C4 bench: tile multiples + a short last chunk)
    assert chunk_bounds(4096, sizes=[1280, 1280, 1280, 256]) == [
        (0, 1280), (1280, 2560), (2560, 3840), (3840, 4096)]
    assert chunk_bounds(1000, sizes=[300, 300]) == [(0, 300), (300, 1000)]  # remainder joins
    assert chunk_bounds(500, sizes=[300, 300, 300]) == [(0, 300), (300, 500)]  # clipped


def test_srpmap_argmax_only_and_lazy_argmax():
    """SrpMap without materialised values (maps=False drop-ins) reports its
    argmax and refuses .values; the fused argmax is fetched lazily from the
    shared device rows (no per-call host sync)."""
    import numpy as np
    import pytest

    from paper_2012_09499_b200.spectral import _DeviceRows
    from paper_2012_09499_b200.srp import SrpMap, argmax_candidate

    class FakeTensor:  # the host copy is all _DeviceRows touches here
        def __init__(self, a):
            self.a = a

        def cpu(self):
            return self

        def numpy(self):
            return self.a

    rows = _DeviceRows(FakeTensor(np.array([5, 1, 7])), np.int64)
    m = SrpMap(None, "approximated", frame_index=2, _argmax=(rows, 2), _num=50)
    assert argmax_candidate(m) == 7 and m.num_candidates == 50
    with pytest.raises(ValueError, match="maps=False"):
        _ = m.values
    with pytest.raises(ValueError):
        SrpMap(None, "x")  # neither values nor argmax


def test_harness_install_rebinds_and_restores():
    """harness.installed swaps exactly the hot-path names a harness module
    binds, and restores the originals."""
    import types
    import paper_2012_09499_b200 as B
    from paper_2012_09499_b200 import harness as H

    def stub(*a, **k):
        raise NotImplementedError

    ns = types.SimpleNamespace(cross_spectrum=stub, srp_approx=stub, argmax_candidate=stub,
                               approximation_error_db=stub, unrelated=stub)
    table = H.drop_ins()
    assert set(table) == set(H.SWAPPED_NAMES)
    assert table["srp_oracle"] is B.srp_oracle
    assert table["approximation_error_db"] is B.approximation_error_db
    with H.installed(ns):
        assert ns.cross_spectrum is B.cross_spectrum
        assert ns.srp_approx is B.srp_approx
        assert ns.argmax_candidate is B.argmax_candidate
        assert ns.unrelated is stub
        assert not hasattr(ns, "srp_oracle")  # only names the module already binds
    assert ns.cross_spectrum is stub and ns.srp_approx is stub
    restore = H.install(ns)
    assert ns.approximation_error_db is B.approximation_error_db
    restore()
    assert ns.approximation_error_db is stub


def test_tensor_core_lattice_shape_rules_without_gpu():
    """Host-side shape rules of the tensor-core lattice (no launch): lag
    slots rounded to 16; long lattices (C4: 2L + 1 = 603) are served in passes,
    C2/C3 in one; beyond 1024 slots or with Kb % 32 != 0 the SIMT lattice
    serves the call."""
    _native.load()
    q = _native.query
    assert q("srpb_lattice_tc_cols", 301) == 608 and q("srpb_lattice_tc_cols", 9) == 32
    # C4: 32 mics, 496 pairs, Kb 512, L = 301 (N_aux 2 included), T_pad 143712
    assert q("srpb_lattice_tc_supported", 32, 496, 512, 301, 143712) == 1
    # C2: 8 mics, 28 pairs, L = 13; C3: 16 mics, 120 pairs, Kb 1024, L = 23
    assert q("srpb_lattice_tc_supported", 8, 28, 512, 13, 640) == 1
    assert q("srpb_lattice_tc_supported", 16, 120, 1024, 23, 3392) == 1
    assert q("srpb_lattice_tc_supported", 32, 496, 512, 600, 600000) == 0  # > 1024 slots
    assert q("srpb_lattice_tc_supported", 8, 28, 520, 13, 640) == 0       # Kb % 32 != 0


# ------------------------------------------------------- bench.py host logic
def test_bench_step_roofline_bounds_and_fractions():
    """Per-sweep-line roofline of bench.py: tensor floor = algorithmic flops /
    (bf16 peak / 3), HBM floor = weight table + spectra + maps / HBM peak."""
    import types

    import bench

    peaks = {"hbm_gbs": 6500.0, "bf16_tflops": 1600.0, "bf16_tflops_sustained": 1400.0}
    c5 = types.SimpleNamespace(J=200000, total_samples=596, T_pad=608, weight_mode="stored",
                               P=28, Kb=512, M=8)
    r = bench.step_roofline(0.115, c5, 1, "approx", peaks)["roofline"]
    assert r["bound"] == "hbm"          # batch 1 streams the weight table once
    nbytes = 4 * 200000 * 608 + 8 * 8 * 512 + 4 * 200000
    assert math.isclose(r["hbm_gbs"], nbytes / 0.115e-3 / 1e9, rel_tol=1e-12)
    assert math.isclose(r["frac"], r["hbm_frac"]) and 0 < r["frac"] < 1
    r = bench.step_roofline(2.6, c5, 4096, "approx", peaks)["roofline"]
    assert r["bound"] == "tensor"
    assert math.isclose(r["tensor_tflops"], 2 * 596 * 4096 * 200000 / 2.6e-3 / 1e12, rel_tol=1e-12)
    assert math.isclose(r["peaks"]["tflops_3xfp16"], 1600.0 / 3)   # short step: burst peak
    r = bench.step_roofline(1750.0, c5, 65536, "conventional", peaks, maps=False)["roofline"]
    assert math.isclose(r["peaks"]["tflops_3xfp16"], 1400.0 / 3)   # long step: sustained peak
    assert math.isclose(r["tensor_tflops"], 4 * 28 * 512 * 65536 * 200000 / 1.75 / 1e12,
                        rel_tol=1e-12)


def test_bench_reference_arm_uses_installed_reference_when_present():
    import bench

    assert bench.cpu_kind() in ("reference", "port")
    assert (bench.cpu_kind() == "reference") == os.path.isfile(
        os.path.join(bench.REF_DIR, "srpfast", "srp.py"))
