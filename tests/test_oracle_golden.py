"""Pin the CPU oracle to the reference's own outputs (CPU, no GPU).

``tests/golden/*.npz`` were written by running the unmodified reference
(``tests/golden/make_golden.py``).  The oracle must reproduce them to fp64
rounding before it may judge the CUDA path.
"""

import numpy as np
import pytest

from oracle import srp_oracle as O
from conftest import load_golden

RTOL = 1e-10


def rel_err(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name", ["c1", "c2_subset", "random_small", "on_lattice"])
def test_oracle_matches_reference_paths(name):
    g = load_golden(name)
    Y = g["Y"].astype(np.complex128)
    T = 1.0 / 16000.0
    psis = []
    for f in range(Y.shape[0]):
        psi, floor = O.cross_spectrum(Y[f], g["pair_m"], g["pair_mp"])
        assert rel_err(psi, g["psi"][f]) < 1e-13
        assert floor == pytest.approx(float(g["floors"][f]), rel=1e-12)
        psis.append(psi)
    psi = np.stack(psis)
    conv = O.conventional_frames(psi, g["omega"], g["tdoa"])
    assert rel_err(conv, g["conv"]) < RTOL
    assert [O.argmax(c) for c in conv] == list(g["argmax_conv"])
    for n_aux in g["n_aux"]:
        halves, w = O.sinc_table(g["tdoa"], g["bounds"], T, int(n_aux))
        assert list(halves) == list(g[f"half_counts_{n_aux}"])
        for f in range(psi.shape[0]):
            h2, rows = O.gcc_lattice(psi[f], g["omega"], g["bounds"], T, int(n_aux))
            assert rel_err(np.concatenate(rows), g[f"lattice_{n_aux}"][f]) < RTOL
            approx = O.approx_map(w, rows)
            assert rel_err(approx, g[f"approx_{n_aux}"][f]) < RTOL
            assert O.argmax(approx) == int(g[f"argmax_approx_{n_aux}"][f])


def test_oracle_sinc_weights_match_reference():
    g = load_golden("random_small")
    _, w = O.sinc_table(g["tdoa"], g["bounds"], 1.0 / 16000.0, 1)
    np.testing.assert_allclose(np.concatenate(w, axis=1), g["sinc_w_1"], atol=1e-15, rtol=0)


def test_oracle_sinc_exact_indicator():
    g = load_golden("sinc_integer")
    _, w = O.sinc_table(g["tdoa"], g["bounds"], 1.0 / 16000.0, 0)
    assert np.array_equal(w[0], g["weights"])


def test_oracle_cross_edges():
    g = load_golden("cross_edges")
    pm, pmp = g["pair_m"], g["pair_mp"]
    for key in ("rand", "scaled", "zero_bin"):
        psi, floor = O.cross_spectrum(g[f"y_{key}"].astype(complex), pm, pmp)
        assert rel_err(psi, g[f"psi_{key}"]) < 1e-13
        assert floor == pytest.approx(float(g[f"floor_{key}"]), rel=1e-12)
    raw, floor = O.cross_spectrum(g["y_rand"].astype(complex), pm, pmp, weighting="identity")
    assert rel_err(raw, g["raw_rand"]) < 1e-14 and floor == 0.0
    psi, floor = O.cross_spectrum(np.zeros((4, 64), complex), pm, pmp)
    assert np.all(psi == 0) and floor == float(g["floor_all_zero"])
    psi, floor = O.cross_spectrum(np.full((2, 64), 1e-8 + 0j), [1], [0], phat_floor=1.0)
    np.testing.assert_allclose(psi, g["psi_tiny_floor1"], rtol=1e-14)


def test_oracle_nonharmonic_bins():
    g = load_golden("nonharmonic")
    conv = O.conventional_frames(g["psi"], g["omega"], g["tdoa"])
    assert rel_err(conv, g["conv"]) < 1e-12


def test_oracle_closed_form_counts():
    """Acceptance criterion 1 (tests/test_acceptance.py:66-89): M=6 circle,
    r=0.1 m, c=340, J=8101, K=1024, N_aux=2."""
    ang = 2 * np.pi * np.arange(6) / 6
    pos = np.stack([0.1 * np.cos(ang), 0.1 * np.sin(ang), np.zeros(6)], axis=1)
    pairs = O.canonical_pairs(6)
    bounds = [float(np.linalg.norm(pos[m] - pos[mp])) / 340.0 for m, mp in pairs]
    halves = O.lattice_half_counts(bounds, 1.0 / 16000.0)
    rep = O.complexity(8101, 1024, halves, 2)
    assert rep["mults_conventional"] == 124_431_360
    assert rep["mults_sampling"] == 279_552
    assert rep["mults_interpolation"] == 2_211_573
    assert rep["avg_samples_per_pair"] == pytest.approx(14.2 + 4.0)


def test_oracle_stft_matches_reference():
    g = load_golden("stft")
    for tag in "abcd":
        n, hop, win = (int(v) for v in g[f"cfg_{tag}"])
        Y = O.stft(g["x"], n, hop, "sqrt_hann" if win == 0 else "rectangular")
        assert Y.shape == g[f"Y_{tag}"].shape
        assert rel_err(Y, g[f"Y_{tag}"]) < 1e-13
        np.testing.assert_allclose(O.bin_frequencies(16000.0, n), g[f"freqs_{tag}"], rtol=1e-15)
