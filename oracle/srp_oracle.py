"""CPU oracle for the SRP-map hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm (``srpfast``,
arXiv 2012.09499) for exactly the path the B200 build accelerates:
GCC-PHAT cross-spectra -> {conventional SRP | lattice IDFT + sinc
interpolation} -> per-frame argmax.  It exists to CHECK the CUDA path and to
time the reference's CPU algorithm beside it.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it; the product package
``paper_2012_09499_b200`` never does (it fails loudly without its CUDA
library instead of falling back here).

Parity pin: every function below is checked against golden vectors produced
by running the reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/srpfast`` in the build container and writes
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` asserts agreement to
fp64 rounding).  All arithmetic is fp64 / complex128 like the reference
(``spectral.py:119,163``; ``srp.py:97``; ``geometry.py:288``).

The per-pair loops, the geometric phase recurrence and the complex GEMMs are
kept in the reference's order of operations on purpose: ``bench.py --impl
reference`` times this port as the reference's CPU implementation, so it
must cost what the reference costs (``srp.py:420-424``: one J x K phase
matrix and one zgemm per pair).
"""

from __future__ import annotations

import math

import numpy as np

#: adaptive PHAT floor factor, ``spectral.py:31-32``
PHAT_FLOOR_REL = 1e-12


# --------------------------------------------------------------------------
# spectral.py
# --------------------------------------------------------------------------
def cross_spectrum(spectra, pair_m, pair_mp, weighting="phat", phat_floor=None):
    """Weighted cross-spectra of one frame (``spectral.py:218-285``).

    ``spectra`` is (M, K) complex; ``pair_m``/``pair_mp`` the canonical pair
    index rows (``index_m > index_m_prime``, ``geometry.py:141-176``).
    Returns ``(psi (P, K) complex128, applied_floor float)``.
    """
    y = np.asarray(spectra, dtype=np.complex128)
    pm = np.asarray(pair_m, dtype=np.int64)
    pmp = np.asarray(pair_mp, dtype=np.int64)
    if weighting not in ("phat", "identity"):
        raise ValueError(f"unknown weighting {weighting!r}")
    if pm.size == 0:
        raise ValueError("pairs must be non-empty")
    if int(pm.max()) >= y.shape[0]:
        raise ValueError(
            f"pair index {int(pm.max())} out of range for {y.shape[0]} channels"
        )
    # spectral.py:258 -- raw product y_m * conj(y_m')
    raw = y[pm] * np.conj(y[pmp])
    if weighting == "identity":  # spectral.py:259-267
        return raw, 0.0
    mag = np.abs(raw)
    if phat_floor is None:  # spectral.py:269-271: 1e-12 * RMS |raw| over (P, K)
        floor = PHAT_FLOOR_REL * float(np.sqrt(np.mean(mag ** 2)))
    else:  # spectral.py:272-275
        if not (phat_floor > 0 and math.isfinite(phat_floor)):
            raise ValueError(f"phat_floor must be positive, got {phat_floor}")
        floor = float(phat_floor)
    # spectral.py:276-277 -- exact-zero products stay exactly zero
    out = np.zeros_like(raw)
    nz = mag > 0.0
    out[nz] = raw[nz] / np.maximum(mag[nz], floor)
    return out, floor


def stft(signals, frame_length, hop_length=None, window="sqrt_hann"):
    """Framed, windowed one-sided spectra [F, M, K] complex128
    (``spectral.stft_analyze`` ``spectral.py:185-215``; window
    ``FrameSpec.window_samples`` ``:85-90``; frame count ``num_frames``
    ``:92-99``).  Frame f covers samples [f hop, f hop + N); DC kept, Nyquist
    dropped; trailing samples that do not fill a frame are dropped."""
    x = np.atleast_2d(np.asarray(signals, dtype=float))
    n = int(frame_length)
    hop = n // 2 if hop_length is None else int(hop_length)
    if window == "rectangular":
        w = np.ones(n)
    else:
        w = np.sqrt(0.5 - 0.5 * np.cos(2.0 * np.pi * np.arange(n) / n))
    num = (x.shape[1] - n) // hop + 1
    out = np.empty((num, x.shape[0], n // 2), dtype=np.complex128)
    for f in range(num):
        out[f] = np.fft.rfft(x[:, f * hop: f * hop + n] * w[None, :], axis=1)[:, : n // 2]
    return out


def bin_frequencies(sample_rate, frame_length):
    """``w_k = 2 pi k fs / N`` for ``k < N/2`` (``spectral.py:80-83``)."""
    k = np.arange(frame_length // 2)
    return 2.0 * np.pi * k * sample_rate / frame_length


# --------------------------------------------------------------------------
# srp.py
# --------------------------------------------------------------------------
def lattice_half_counts(tdoa_bounds, sample_period):
    """``N_p = floor(bound_p / T)`` (``srp.py:123-134``)."""
    if not (sample_period > 0 and math.isfinite(sample_period)):
        raise ValueError(f"sample_period must be positive, got {sample_period}")
    return tuple(int(math.floor(b / sample_period)) for b in tdoa_bounds)


def lattice_offsets(half_count, n_aux):
    """Integer lags ``-(N_p+n_aux) .. N_p+n_aux`` (``srp.py:137-140``)."""
    r = int(half_count) + int(n_aux)
    return np.arange(-r, r + 1)


def gcc_at_lag(psi_row, omega, lag):
    """``2 Re sum_k psi_k e^{j w_k lag}`` (``srp.py:112-120``)."""
    return 2.0 * float(np.dot(psi_row, np.exp(1j * np.asarray(omega) * lag)).real)


def phase_matrix(tau, omega):
    """``e^{j w_k tau_j}`` as (J, K) (``srp.py:350-373``).

    Harmonic bins (``w_0 = 0``, constant spacing to rtol 1e-12) use the
    reference's geometric recurrence column by column; others the dense exp.
    """
    tau = np.asarray(tau, dtype=float)
    omega = np.asarray(omega, dtype=float)
    kc = omega.size
    harmonic = (
        kc >= 2
        and omega[0] == 0.0
        and omega[1] > 0.0
        and np.allclose(np.diff(omega), omega[1], rtol=1e-12, atol=0.0)
    )
    if not harmonic:
        return np.exp(1j * np.multiply.outer(tau, omega))
    out = np.empty((tau.size, kc), dtype=np.complex128)
    out[:, 0] = 1.0
    step = np.exp(1j * omega[1] * tau)
    for k in range(1, kc):
        np.multiply(out[:, k - 1], step, out=out[:, k])
    return out


def conventional_frames(psi, omega, tdoa_table, candidate_chunk=None):
    """Exact maps for F frames (``srp.py:391-429``).

    ``psi`` is (F, P, K) complex, ``tdoa_table`` (J, P) seconds.  Returns
    (F, J) fp64: ``sum_p 2 Re(phases_p @ psi_p)`` accumulated pair by pair
    (``srp.py:420-424``).  ``candidate_chunk`` bounds the (J, K) complex128
    temporary for large grids (the reference allocates it whole); the
    per-candidate arithmetic is unchanged by chunking.
    """
    psi = np.asarray(psi, dtype=np.complex128)
    table = np.asarray(tdoa_table, dtype=float)
    n_frames, n_pairs, _ = psi.shape
    if table.shape[1] != n_pairs:
        raise ValueError(f"frame has {n_pairs} pairs, grid table has {table.shape[1]}")
    n_cand = table.shape[0]
    chunk = n_cand if candidate_chunk is None else int(candidate_chunk)
    stacked = np.transpose(psi, (1, 2, 0))  # (P, K, F) as srp.py:419
    out = np.zeros((n_cand, n_frames))
    for lo in range(0, n_cand, chunk):
        hi = min(n_cand, lo + chunk)
        acc = np.zeros((hi - lo, n_frames))
        for p in range(n_pairs):
            ph = phase_matrix(table[lo:hi, p], omega)
            acc += 2.0 * (ph @ stacked[p]).real
        out[lo:hi] = acc
    return out.T.copy()


def gcc_lattice(psi, omega, tdoa_bounds, sample_period, n_aux):
    """Lattice samples of one frame (``srp.py:201-247``).

    Returns ``(half_counts, rows)``; row ``p`` holds ``2 Re(e^{j w nT} @
    psi_p)`` at ``n = -(N_p+n_aux) .. N_p+n_aux`` (index 0 = most negative).
    """
    if n_aux < 0 or int(n_aux) != n_aux:
        raise ValueError(f"n_aux must be a non-negative integer, got {n_aux}")
    halves = lattice_half_counts(tdoa_bounds, sample_period)
    omega = np.asarray(omega, dtype=float)
    rows = []
    for p, n_p in enumerate(halves):
        lags = lattice_offsets(n_p, n_aux) * sample_period
        ph = np.exp(1j * np.multiply.outer(lags, omega))
        rows.append(2.0 * (ph @ psi[p]).real)
    return halves, rows


def sinc_kernel(x):
    """``np.sinc`` snapped to exact 0/1 at integers (``srp.py:250-261``)."""
    x = np.asarray(x, dtype=float)
    out = np.sinc(x)
    node = x == np.rint(x)
    out[node] = 0.0
    out[node & (x == 0.0)] = 1.0
    return out


def sinc_table(tdoa_table, tdoa_bounds, sample_period, n_aux):
    """Per-pair (J, T_p) weights ``sinc(tau/T - n)`` (``srp.py:287-317``)."""
    if n_aux < 0 or int(n_aux) != n_aux:
        raise ValueError(f"n_aux must be a non-negative integer, got {n_aux}")
    table = np.asarray(tdoa_table, dtype=float)
    if table.shape[1] != len(tdoa_bounds):
        raise ValueError(
            f"grid table has {table.shape[1]} pair columns, expected {len(tdoa_bounds)}"
        )
    halves = lattice_half_counts(tdoa_bounds, sample_period)
    weights = []
    for p, n_p in enumerate(halves):
        offs = lattice_offsets(n_p, n_aux)
        x = table[:, p] / sample_period
        weights.append(sinc_kernel(x[:, None] - offs[None, :]))
    return halves, weights


def approx_map(weights, rows):
    """``sum_p W_p @ xi_p`` accumulated pair by pair (``srp.py:340-344``)."""
    values = np.zeros(weights[0].shape[0])
    for w, row in zip(weights, rows):
        values += w @ row
    return values


def argmax(values):
    """Lowest index among maxima (``srp.py:107-109``)."""
    return int(np.argmax(np.asarray(values)))


def complexity(num_candidates, num_bins, half_counts, n_aux):
    """Closed-form per-frame counts (``srp.py:573-619``)."""
    counts = [2 * (h + int(n_aux)) + 1 for h in half_counts]
    total = sum(counts)
    avg = 2.0 / len(half_counts) * sum(half_counts) + 2.0 * n_aux + 1.0
    return {
        "total_samples": total,
        "avg_samples_per_pair": avg,
        "mults_conventional": num_candidates * len(half_counts) * num_bins,
        "mults_sampling": total * num_bins,
        "mults_interpolation": total * num_candidates,
    }


# --------------------------------------------------------------------------
# geometry.py (host constants feeding the path)
# --------------------------------------------------------------------------
def canonical_pairs(num_mics):
    """(index_m, index_m_prime) in ``itertools.combinations`` order
    (``geometry.py:141-176``)."""
    out = []
    for mp in range(num_mics):
        for m in range(mp + 1, num_mics):
            out.append((m, mp))
    return out


def tdoa_table_nearfield(mic_pos, points, pairs, c):
    """``(|p_m - q| - |p_m' - q|) / c`` per candidate and pair
    (``geometry.py:383-389``)."""
    pos = np.asarray(mic_pos, dtype=float)
    q = np.asarray(points, dtype=float)
    dist = np.linalg.norm(q[:, None, :] - pos[None, :, :], axis=2)
    cols = [(dist[:, m] - dist[:, mp]) / c for (m, mp) in pairs]
    return np.stack(cols, axis=1)
