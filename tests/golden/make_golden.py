"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

It imports the unmodified reference package ``srpfast`` and records its
outputs for seeded inputs as ``tests/golden/*.npz``.  The committed fixtures
pin both the oracle (``tests/test_oracle_golden.py``, CPU) and the CUDA path
(``tests/test_parity_gpu.py``, GPU).  Inputs are stored as complex64 and
handed to the reference upcast to complex128, so fixtures compare compute
error only.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import srpfast  # noqa: E402  (the reference, from PYTHONPATH)
from srpfast.geometry import CandidateGrid, MicArray, build_tdoa_table, circular_array  # noqa: E402
from srpfast.spectral import (  # noqa: E402
    CrossSpectra,
    FrameSpec,
    SpectralFrame,
    cross_spectrum,
    stft_analyze,
)
from srpfast.srp import (  # noqa: E402
    argmax_candidate,
    build_gcc_lattice,
    lattice_half_counts,
    precompute_sinc_table,
    srp_approx,
    srp_conventional_frames,
)

from paper_2012_09499_b200 import scenes  # noqa: E402  (input synthesis only)

FS = 16000.0
T = 1.0 / FS


def harmonic(num_bins, frame_length):
    return 2.0 * np.pi * np.arange(num_bins) * FS / frame_length


def pair_rows(pairs):
    return (
        np.array([p.index_m for p in pairs], dtype=np.int32),
        np.array([p.index_m_prime for p in pairs], dtype=np.int32),
        np.array([p.distance for p in pairs]),
        np.array([p.tdoa_bound for p in pairs]),
    )


def run_paths(Y64, array, grid, omega, n_aux_list, weighting="phat"):
    """Reference outputs for frames Y64 (F, M, K) complex64."""
    frames = [
        SpectralFrame(spectra=Y64[f].astype(np.complex128), bin_frequencies=omega, frame_index=f)
        for f in range(Y64.shape[0])
    ]
    crosses = [cross_spectrum(fr, array.pairs, weighting=weighting) for fr in frames]
    out = {
        "psi": np.stack([c.values for c in crosses]),
        "floors": np.array([c.phat_floor for c in crosses]),
    }
    conv = srp_conventional_frames(crosses, grid)
    out["conv"] = np.stack([m.values for m in conv])
    out["argmax_conv"] = np.array([argmax_candidate(m) for m in conv], dtype=np.int64)
    for n_aux in n_aux_list:
        table = precompute_sinc_table(grid, array.pairs, T, n_aux)
        lats = [build_gcc_lattice(c, T, n_aux) for c in crosses]
        approx = [srp_approx(l, table) for l in lats]
        out[f"lattice_{n_aux}"] = np.stack([np.concatenate(l.samples) for l in lats])
        out[f"half_counts_{n_aux}"] = np.array(lats[0].half_counts, dtype=np.int64)
        out[f"approx_{n_aux}"] = np.stack([m.values for m in approx])
        out[f"argmax_approx_{n_aux}"] = np.array(
            [argmax_candidate(m) for m in approx], dtype=np.int64
        )
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def scene_case(name, scene, num_frames, n_aux_list, grid_limit=None):
    array = MicArray(scene.mic_pos, speed_of_sound=scene.speed_of_sound)
    pts = scene.grid if grid_limit is None else scene.grid[:grid_limit]
    grid = build_tdoa_table(array, CandidateGrid(mode="near_field", entries=pts))
    Y = scene.Y[:num_frames]
    omega = harmonic(scene.num_bins, scene.frame_length)
    res = run_paths(Y, array, grid, omega, n_aux_list)
    pm, pmp, dist, bounds = pair_rows(array.pairs)
    save(
        name,
        Y=Y, mic_pos=scene.mic_pos, grid=pts, tdoa=grid.tdoa_table, omega=omega,
        pair_m=pm, pair_mp=pmp, distance=dist, bounds=bounds,
        n_aux=np.array(n_aux_list), frame_length=np.array(scene.frame_length),
        speed_of_sound=np.array(scene.speed_of_sound), **res,
    )


def random_small():
    """Random 5-mic array / 30 candidates / 64 bins (tests/test_srp.py style)."""
    rng = np.random.default_rng(20240)
    array = MicArray(rng.normal(size=(5, 3)) * 0.2)
    pts = rng.uniform(-3.0, 3.0, size=(30, 3))
    grid = build_tdoa_table(array, CandidateGrid(mode="near_field", entries=pts))
    Y = scenes.random_frames(rng, 3, 5, 64)
    omega = harmonic(64, 128)
    res = run_paths(Y, array, grid, omega, (0, 1, 3))
    table = precompute_sinc_table(grid, array.pairs, T, 1)
    pm, pmp, dist, bounds = pair_rows(array.pairs)
    save(
        "random_small.npz",
        Y=Y, mic_pos=array.positions, grid=pts, tdoa=grid.tdoa_table, omega=omega,
        pair_m=pm, pair_mp=pmp, distance=dist, bounds=bounds, n_aux=np.array([0, 1, 3]),
        frame_length=np.array(128), speed_of_sound=np.array(340.0),
        sinc_w_1=np.concatenate(table.weights, axis=1), **res,
    )


def on_lattice():
    """TDOAs on lattice multiples: approx == conventional (acceptance 4)."""
    rng = np.random.default_rng(4)
    array = circular_array(6, 0.1, speed_of_sound=340.0)
    halves = lattice_half_counts(array.pairs, T)
    mult = np.stack([rng.integers(-h, h + 1, size=40) for h in halves], axis=1)
    grid = CandidateGrid(
        mode="near_field", entries=rng.uniform(-1.0, 1.0, size=(40, 3)), tdoa_table=mult * T
    )
    Y = scenes.random_frames(rng, 2, 6, 1024)
    omega = harmonic(1024, 2048)
    res = run_paths(Y, array, grid, omega, (0, 2))
    pm, pmp, dist, bounds = pair_rows(array.pairs)
    save(
        "on_lattice.npz",
        Y=Y, mic_pos=array.positions, tdoa=grid.tdoa_table, multiples=mult, omega=omega,
        pair_m=pm, pair_mp=pmp, distance=dist, bounds=bounds, n_aux=np.array([0, 2]),
        frame_length=np.array(2048), speed_of_sound=np.array(340.0), **res,
    )


def cross_edges():
    """GCC-PHAT edge cases of tests/test_spectral.py:136-221."""
    rng = np.random.default_rng(7)
    array = circular_array(4, 0.1)
    omega = harmonic(64, 128)
    pm, pmp, _, _ = pair_rows(array.pairs)
    out = {"pair_m": pm, "pair_mp": pmp, "omega": omega}

    def cs(y, pairs=array.pairs, **kw):
        c = cross_spectrum(SpectralFrame(spectra=y, bin_frequencies=omega), pairs, **kw)
        return c.values, c.phat_floor

    y = (rng.normal(size=(4, 64)) + 1j * rng.normal(size=(4, 64))).astype(np.complex64)
    out["y_rand"] = y
    out["psi_rand"], out["floor_rand"] = cs(y.astype(np.complex128))
    out["raw_rand"], out["floor_identity"] = cs(y.astype(np.complex128), weighting="identity")
    y_scaled = (1e4 * y.astype(np.complex128)).astype(np.complex64)
    out["y_scaled"] = y_scaled
    out["psi_scaled"], out["floor_scaled"] = cs(y_scaled.astype(np.complex128))
    yz = y.copy()
    yz[:, 10] = 0.0
    out["y_zero_bin"] = yz
    out["psi_zero_bin"], out["floor_zero_bin"] = cs(yz.astype(np.complex128))
    out["psi_all_zero"], out["floor_all_zero"] = cs(np.zeros((4, 64), dtype=complex))
    tiny = np.full((2, 64), 1e-8 + 0j)
    pairs2 = circular_array(2, 0.05).pairs
    out["psi_tiny_floor1"], out["floor_tiny_floor1"] = cs(tiny, pairs=pairs2, phat_floor=1.0)
    save("cross_edges.npz", **out)


def sinc_integer():
    """Exact indicator rows at integer TDOAs (tests/test_srp.py:153-167)."""
    array = circular_array(2, 0.2, speed_of_sound=340.0)
    tdoas = np.array([[3.0 * T], [-2.0 * T], [0.0]])
    grid = CandidateGrid(
        mode="near_field", entries=np.zeros((3, 3)) + [1.0, 0.0, 0.0], tdoa_table=tdoas
    )
    table = precompute_sinc_table(grid, array.pairs, T, 0)
    _, _, _, bounds = pair_rows(array.pairs)
    save("sinc_integer.npz", tdoa=tdoas, bounds=bounds, weights=table.weights[0],
         half_counts=np.array(table.half_counts))


def nonharmonic():
    """Irregular bins: the reference's dense-exp phase path (srp.py:366-367)."""
    rng = np.random.default_rng(48)
    array = MicArray(rng.normal(size=(4, 3)) * 0.2)
    pts = rng.uniform(-2.0, 2.0, size=(25, 3))
    grid = build_tdoa_table(array, CandidateGrid(mode="near_field", entries=pts))
    omega = np.sort(rng.uniform(0, 5e4, size=48))
    Y = scenes.random_frames(rng, 2, 4, 48)
    frames = [SpectralFrame(spectra=Y[f].astype(complex), bin_frequencies=omega) for f in range(2)]
    crosses = [cross_spectrum(fr, array.pairs) for fr in frames]
    conv = srp_conventional_frames(crosses, grid)
    pm, pmp, dist, bounds = pair_rows(array.pairs)
    save(
        "nonharmonic.npz", Y=Y, omega=omega, tdoa=grid.tdoa_table, pair_m=pm, pair_mp=pmp,
        bounds=bounds, psi=np.stack([c.values for c in crosses]),
        conv=np.stack([m.values for m in conv]),
    )


def stft_cases():
    """Reference STFT (spectral.stft_analyze) of seeded float32 audio: several
    frame lengths, hops and both windows; trailing samples dropped."""
    rng = np.random.default_rng(20240611)
    x = rng.standard_normal((3, 6000)).astype(np.float32)
    x[1] *= 1e-3  # a quiet channel
    x[2, 2500:2600] = 0.0  # a silent stretch
    cases = {}
    for tag, (n, hop, win) in {"a": (512, None, "sqrt_hann"), "b": (256, 100, "rectangular"),
                               "c": (2048, 512, "sqrt_hann"), "d": (64, 64, "sqrt_hann")}.items():
        spec = FrameSpec(FS, n, hop, win)
        frames = stft_analyze(x.astype(np.float64), spec)
        cases[f"Y_{tag}"] = np.stack([fr.spectra for fr in frames])  # [F, M, Kb] complex128
        cases[f"cfg_{tag}"] = np.array([n, spec.hop_length, 0 if win == "sqrt_hann" else 1])
        cases[f"freqs_{tag}"] = frames[0].bin_frequencies
    save("stft.npz", x=x, **cases)


def main():
    print("reference srpfast", srpfast.__version__, "from", os.path.dirname(srpfast.__file__))
    stft_cases()
    scene_case("c1.npz", scenes.make_c1(num_frames=8), 8, (2,))
    scene_case("c2_subset.npz", scenes.make_c2(num_frames=3), 3, (0, 2, 4), grid_limit=3000)
    random_small()
    on_lattice()
    cross_edges()
    sinc_integer()
    nonharmonic()


if __name__ == "__main__":
    main()
