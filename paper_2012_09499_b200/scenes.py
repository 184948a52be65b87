"""Seeded synthetic scenes for the five BASELINE.json configurations.

Host-side input synthesis only (the reference renders scenes on the host
too, ``simulate.py``); nothing here is on the hot path.  The reference
publishes no dataset for this path, so seeded synthetic signals with the
configs' shapes stand in.  Seeds follow
``SeedSequence([config_id, scene_index, stream])``.

Every scene is rendered per STFT frame in the frequency domain: the source's
windowed frame spectrum ``S_f(k)`` (periodic sqrt-Hann, ``spectral.py:85-90``)
is delayed per microphone by the phase ramp ``e^{-j w_k r_m / c}`` and
attenuated by ``1 / r_m`` ("frame-wise static delay"), then independent
sensor noise -- and for C2 a diffuse field of plane waves -- is added at
the configured SNR.  One-sided bins ``k < N/2`` (Nyquist dropped,
``spectral.py:70-73``).  Output ``Y`` is ``[F, M, N/2]`` complex64.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

C_SOUND = 343.0  # c = 343 m/s for every config
FS = 16000.0


@dataclass
class Scene:
    name: str
    mic_pos: np.ndarray          # (M, 3) fp64
    grid: np.ndarray             # (J, 3) fp64 candidate positions (near field)
    Y: np.ndarray                # (F, M, Kb) complex64 STFT frames
    frame_length: int
    sample_rate: float = FS
    speed_of_sound: float = C_SOUND
    n_aux: tuple = (2,)
    sources: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))

    @property
    def num_frames(self):
        return self.Y.shape[0]

    @property
    def num_bins(self):
        return self.Y.shape[2]


def _rng(config_id, scene_index, stream):
    return np.random.default_rng(np.random.SeedSequence([config_id, scene_index, stream]))


def sqrt_hann(n):
    k = np.arange(n)
    return np.sqrt(0.5 - 0.5 * np.cos(2.0 * np.pi * k / n))


def frame_spectra(signal, frame_length, hop, num_frames=None):
    """Windowed one-sided frame spectra of a 1-D signal, ``(F, N/2)``."""
    n = frame_length
    f_total = (signal.size - n) // hop + 1
    if num_frames is not None:
        f_total = min(f_total, num_frames)
    idx = np.arange(n)[None, :] + hop * np.arange(f_total)[:, None]
    frames = signal[idx] * sqrt_hann(n)[None, :]
    return np.fft.rfft(frames, axis=1)[:, : n // 2]


def box_grid(nx, ny, nz, extent, origin=(0.0, 0.0, 0.0)):
    """Cell-centred candidate grid over ``extent`` metres, x-major order."""
    ex, ey, ez = extent
    ox, oy, oz = origin
    xs = ox + (np.arange(nx) + 0.5) * ex / nx
    ys = oy + (np.arange(ny) + 0.5) * ey / ny
    zs = oz + (np.arange(nz) + 0.5) * ez / nz
    g = np.stack(np.meshgrid(xs, ys, zs, indexing="ij"), axis=-1)
    return g.reshape(-1, 3)


def uca(num_mics, radius, center):
    ang = 2.0 * np.pi * np.arange(num_mics) / num_mics
    c = np.asarray(center, dtype=float)
    return np.stack(
        [c[0] + radius * np.cos(ang), c[1] + radius * np.sin(ang), np.full(num_mics, c[2])],
        axis=1,
    )


def _render(rng, mic_pos, src_positions, src_gains, src_spectra, omega, c):
    """Sum of point sources: ``g / r_m * S_f(k) * e^{-j w_k r_m / c}``."""
    F, Kb = src_spectra[0].shape
    M = mic_pos.shape[0]
    Y = np.zeros((F, M, Kb), dtype=np.complex128)
    for pos, gain, S in zip(src_positions, src_gains, src_spectra):
        r = np.linalg.norm(mic_pos - pos[None, :], axis=1)  # (M,)
        ramp = np.exp(-1j * np.outer(r / c, omega)) * (gain / r)[:, None]  # (M, Kb)
        Y += S[:, None, :] * ramp[None, :, :]
    return Y


def _add_noise(rng, Y, snr_db, frame_length):
    """Independent white sensor noise at ``snr_db`` relative to mean power."""
    p_sig = float(np.mean(np.abs(Y) ** 2))
    F, M, Kb = Y.shape
    noise_t = rng.standard_normal((F * M, frame_length))
    N = np.fft.rfft(noise_t * sqrt_hann(frame_length)[None, :], axis=1)[:, :Kb]
    N = N.reshape(F, M, Kb)
    p_n = float(np.mean(np.abs(N) ** 2))
    scale = np.sqrt(p_sig / (p_n * 10.0 ** (snr_db / 10.0)))
    return Y + scale * N


def _diffuse(rng, mic_pos, F, Kb, frame_length, omega, c, directions=32):
    """Diffuse field: independent white plane waves from random directions."""
    u = rng.standard_normal((directions, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    out = np.zeros((F, mic_pos.shape[0], Kb), dtype=np.complex128)
    win = sqrt_hann(frame_length)
    for d in range(directions):
        w = rng.standard_normal((F, frame_length)) * win[None, :]
        S = np.fft.rfft(w, axis=1)[:, :Kb]
        delay = mic_pos @ u[d] / c
        out += S[:, None, :] * np.exp(-1j * np.outer(delay, omega))[None, :, :]
    return out


def _omega(frame_length, fs=FS):
    return 2.0 * np.pi * np.arange(frame_length // 2) * fs / frame_length


def make_c1(scene_index=0, num_frames=None):
    """C1 (configs[0]): M=4 square 0.2 m at z=1.5, source in z=0 plane,
    1 s white noise, 10 dB SNR, N=512 hop 256, 41x41 grid, N_aux=2."""
    rng = _rng(1, scene_index, 0)
    mic = np.array(
        [[0.1, 0.1, 1.5], [-0.1, 0.1, 1.5], [-0.1, -0.1, 1.5], [0.1, -0.1, 1.5]]
    )
    n = 512
    src = np.array([rng.uniform(-2, 2), rng.uniform(-2, 2), 0.0])
    x = rng.standard_normal(int(FS))
    S = frame_spectra(x, n, n // 2, num_frames)
    omega = _omega(n)
    Y = _render(rng, mic, [src], [1.0], [S], omega, C_SOUND)
    Y = _add_noise(rng, Y, 10.0, n)
    g = np.linspace(-2.0, 2.0, 41)
    gx, gy = np.meshgrid(g, g, indexing="ij")
    grid = np.stack([gx.ravel(), gy.ravel(), np.zeros(gx.size)], axis=1)
    return Scene("C1", mic, grid, Y.astype(np.complex64), n, n_aux=(2,),
                 sources=src[None, :])


def make_c2(scene_index=0, num_frames=None, grid_limit=None):
    """C2 (configs[1]): UCA M=8 r=0.1 m, 10 s white source + 6 image
    sources (gains U(0.2,0.6)), diffuse noise at 5 dB, N=1024 hop 512,
    50x50x20 grid over 5x5x2 m, N_aux in {0,2,4}."""
    rng = _rng(2, scene_index, 0)
    center = np.array([2.5, 2.5, 1.0])
    mic = uca(8, 0.1, center)
    n = 1024
    box = np.array([5.0, 5.0, 2.0])
    src = rng.uniform(0.2, 1.0, size=3) * box
    images = rng.uniform(0.0, 1.0, size=(6, 3)) * box * np.array([3, 3, 3]) - box
    gains = [1.0] + list(rng.uniform(0.2, 0.6, size=6))
    x = rng.standard_normal(int(10 * FS))
    S = frame_spectra(x, n, n // 2, num_frames)
    omega = _omega(n)
    Y = _render(rng, mic, [src] + list(images), gains, [S] * 7, omega, C_SOUND)
    p_sig = float(np.mean(np.abs(Y) ** 2))
    D = _diffuse(rng, mic, Y.shape[0], Y.shape[2], n, omega, C_SOUND)
    D *= np.sqrt(p_sig / (float(np.mean(np.abs(D) ** 2)) * 10.0 ** 0.5))
    Y = Y + D
    grid = box_grid(50, 50, 20, box)
    if grid_limit is not None:
        grid = grid[:grid_limit]
    return Scene("C2", mic, grid, Y.astype(np.complex64), n, n_aux=(0, 2, 4),
                 sources=src[None, :])


def make_c3(scene_index=0, num_frames=None, grid_limit=None):
    """C3 (configs[2]): two stacked 8-mic rings r=0.15 m 0.1 m apart,
    60 s white source moving at 0.5 m/s (reflecting), 0 dB SNR, N=2048
    hop 1024, 100x100x50 grid over 10x10x5 m, N_aux 0..8."""
    rng = _rng(3, scene_index, 0)
    box = np.array([10.0, 10.0, 5.0])
    c0 = np.array([5.0, 5.0, 1.5])
    mic = np.concatenate([uca(8, 0.15, c0), uca(8, 0.15, c0 + [0, 0, 0.1])])
    n = 2048
    hop = n // 2
    x = rng.standard_normal(int(60 * FS))
    S = frame_spectra(x, n, hop, num_frames)
    F = S.shape[0]
    p0 = rng.uniform(0.1, 0.9, size=3) * box
    v = rng.standard_normal(3)
    v *= 0.5 / np.linalg.norm(v)
    omega = _omega(n)
    Y = np.zeros((F, 16, n // 2), dtype=np.complex128)
    pos = p0.copy()
    dt = hop / FS
    for f in range(F):
        Y[f] = _render(rng, mic, [pos], [1.0], [S[f:f + 1]], omega, C_SOUND)[0]
        pos = pos + v * dt
        for a in range(3):  # reflect at the walls
            if pos[a] < 0 or pos[a] > box[a]:
                v[a] = -v[a]
                pos[a] = min(max(pos[a], 0.0), box[a])
    Y = _add_noise(rng, Y, 0.0, n)
    grid = box_grid(100, 100, 50, box)
    if grid_limit is not None:
        grid = grid[:grid_limit]
    return Scene("C3", mic, grid, Y.astype(np.complex64), n, n_aux=tuple(range(9)),
                 sources=p0[None, :])


def make_c4(scene_index=0, num_frames=4096, grid_limit=None):
    """C4 (configs[3]): M=32 uniform random mics in a 6x5x3 m room, 2 equal
    power white sources, 10 dB SNR, N=1024 hop 512, 4096 frames,
    120x100x50 grid."""
    rng = _rng(4, scene_index, 0)
    box = np.array([6.0, 5.0, 3.0])
    mic = rng.uniform(0.0, 1.0, size=(32, 3)) * box
    n = 1024
    srcs = rng.uniform(0.1, 0.9, size=(2, 3)) * box
    length = (num_frames - 1) * (n // 2) + n
    omega = _omega(n)
    specs = [frame_spectra(rng.standard_normal(length), n, n // 2) for _ in range(2)]
    Y = _render(rng, mic, list(srcs), [1.0, 1.0], specs, omega, C_SOUND)
    Y = _add_noise(rng, Y, 10.0, n)
    grid = box_grid(120, 100, 50, box)
    if grid_limit is not None:
        grid = grid[:grid_limit]
    return Scene("C4", mic, grid, Y.astype(np.complex64), n, n_aux=(2,), sources=srcs)


def _c5_block(rng, batch, mic, box, n, omega):
    """``batch`` independent seeded white-noise scenes (one frame each):
    a random source in the box, 1/r gain, delay phase ramp, 10 dB white
    sensor noise (vectorised over the batch)."""
    srcs = rng.uniform(0.1, 0.9, size=(batch, 3)) * box
    win = sqrt_hann(n)
    S = np.fft.rfft(rng.standard_normal((batch, n)) * win[None, :], axis=1)[:, : n // 2]
    r = np.linalg.norm(mic[None, :, :] - srcs[:, None, :], axis=2)  # (B, M)
    Y = (S[:, None, :] * np.exp(-1j * r[:, :, None] / C_SOUND * omega[None, None, :])
         / r[:, :, None])
    return _add_noise(rng, Y, 10.0, n), srcs


def make_c5(batch, scene_index=0, grid_limit=None):
    """C5 (configs[4]): UCA M=8 r=0.1 m, N=1024, 100x100x20 grid (200k)
    over 5x5x2 m, ``batch`` frames of independent seeded white-noise
    scenes at 10 dB, N_aux=4.  Batches above 4096 are rendered in blocks of
    4096 scenes with their own seeds ``[5, scene_index, batch, block]``
    (bounded host memory at 65536)."""
    box = np.array([5.0, 5.0, 2.0])
    mic = uca(8, 0.1, [2.5, 2.5, 1.0])
    n = 1024
    omega = _omega(n)
    if batch <= 4096:
        Y, srcs = _c5_block(_rng(5, scene_index, batch), batch, mic, box, n, omega)
        Y = Y.astype(np.complex64)
    else:
        Y = np.empty((batch, 8, n // 2), dtype=np.complex64)
        srcs = np.empty((batch, 3))
        for b, lo in enumerate(range(0, batch, 4096)):
            hi = min(batch, lo + 4096)
            rng = np.random.default_rng(np.random.SeedSequence([5, scene_index, batch, b]))
            yb, sb = _c5_block(rng, hi - lo, mic, box, n, omega)
            Y[lo:hi] = yb
            srcs[lo:hi] = sb
    grid = box_grid(100, 100, 20, box)
    if grid_limit is not None:
        grid = grid[:grid_limit]
    return Scene("C5", mic, grid, Y, n, n_aux=(4,), sources=srcs)


def random_frames(rng, num_frames, num_mics, num_bins):
    """Unit-variance complex Gaussian spectra (the reference tests' fake
    ``SpectralFrame``s, ``tests/test_srp.py:34-41``)."""
    y = rng.standard_normal((num_frames, num_mics, num_bins)) + 1j * rng.standard_normal(
        (num_frames, num_mics, num_bins)
    )
    return y.astype(np.complex64)
