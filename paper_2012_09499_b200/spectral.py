"""Drop-in for ``srpfast.spectral`` on the B200 path.

``cross_spectrum`` (``pkg/src/srpfast/spectral.py:218-285``) keeps the
reference's signature, validation messages and return type; the arithmetic
runs in the K1 kernel (``csrc/gcc_phat.cu``) through ``libsrpb.so``.
``CrossSpectra`` and ``SpectralFrame`` accept numpy arrays like the
reference, and additionally carry device-resident tensors so a chain
``cross_spectrum -> build_gcc_lattice -> srp_approx`` never round-trips
through the host; ``.values`` materialises complex128 numpy on first access.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .plan import DEFAULT_PHAT_FLOOR_REL

WINDOWS = ("sqrt_hann", "rectangular")
WEIGHTINGS = ("phat", "identity")

__all__ = [
    "FrameSpec",
    "SpectralFrame",
    "CrossSpectra",
    "stft_analyze",
    "cross_spectrum",
    "cross_spectrum_frames",
    "DEFAULT_PHAT_FLOOR_REL",
]


class FrameSpec:
    """STFT framing parameters (``spectral.py:35-99``)."""

    def __init__(self, sample_rate, frame_length, hop_length=None, window="sqrt_hann"):
        if not (sample_rate > 0 and math.isfinite(sample_rate)):
            raise ValueError(f"sample_rate must be positive, got {sample_rate}")
        if frame_length < 2 or frame_length % 2 != 0:
            raise ValueError(f"frame_length must be an even integer >= 2, got {frame_length}")
        hop = frame_length // 2 if hop_length is None else hop_length
        if hop < 1:
            raise ValueError(f"hop_length must be >= 1, got {hop}")
        if window not in WINDOWS:
            raise ValueError(f"window must be one of {WINDOWS}, got {window!r}")
        self.sample_rate = float(sample_rate)
        self.frame_length = int(frame_length)
        self.hop_length = int(hop)
        self.window = window

    @property
    def num_bins(self) -> int:
        return self.frame_length // 2

    @property
    def sample_period(self) -> float:
        return 1.0 / self.sample_rate

    def bin_frequencies(self) -> np.ndarray:
        k = np.arange(self.num_bins)
        return 2.0 * np.pi * k * self.sample_rate / self.frame_length

    def window_samples(self) -> np.ndarray:
        if self.window == "rectangular":
            return np.ones(self.frame_length)
        n = np.arange(self.frame_length)
        return np.sqrt(0.5 - 0.5 * np.cos(2.0 * np.pi * n / self.frame_length))

    def num_frames(self, num_samples: int) -> int:
        if num_samples < self.frame_length:
            raise ValueError(
                f"signal of {num_samples} samples is shorter than one frame ({self.frame_length})"
            )
        return (num_samples - self.frame_length) // self.hop_length + 1


def _as_freqs(freqs, n):
    freqs = np.asarray(freqs, dtype=float)
    if freqs.shape != (n,):
        raise ValueError("bin_frequencies length must match spectra columns")
    return freqs


class SpectralFrame:
    """One-sided spectra (M, K) of one frame (``spectral.py:102-134``).

    ``spectra`` may be a numpy array (kept as complex128, like the
    reference) or a complex64 CUDA tensor (kept on the device).
    """

    def __init__(self, spectra, bin_frequencies, frame_index=0):
        if isinstance(spectra, torch.Tensor):
            if spectra.dim() != 2:
                raise ValueError(f"spectra must be 2-D (M, K), got {tuple(spectra.shape)}")
            self._dev = spectra.to(torch.complex64).contiguous()
            self._host = None
            shape = tuple(spectra.shape)
        else:
            s = np.asarray(spectra, dtype=complex)
            if s.ndim != 2:
                raise ValueError(f"spectra must be 2-D (M, K), got {s.shape}")
            self._host, self._dev = s, None
            shape = s.shape
        self.bin_frequencies = _as_freqs(bin_frequencies, shape[1])
        self.frame_index = frame_index
        self._shape = shape

    @property
    def spectra(self) -> np.ndarray:
        if self._host is None:
            self._host = self._dev.cpu().numpy().astype(np.complex128)
        return self._host

    def device_spectra(self, device=None) -> torch.Tensor:
        dev = N.require_cuda(device)
        if self._dev is None or self._dev.device != dev:
            src = self._host if self._dev is None else self._dev.cpu().numpy()
            self._dev = torch.as_tensor(np.ascontiguousarray(src, dtype=np.complex64), device=dev)
        return self._dev

    num_channels = property(lambda self: self._shape[0])
    num_bins = property(lambda self: self._shape[1])


class _DeviceRows:
    """A [F, ...] device tensor whose host copy is fetched once, on demand."""

    def __init__(self, tensor: torch.Tensor, host_dtype):
        self.tensor = tensor
        self.host_dtype = host_dtype
        self._host = None

    def host(self) -> np.ndarray:
        if self._host is None:
            self._host = self.tensor.cpu().numpy().astype(self.host_dtype)
        return self._host


class CrossSpectra:
    """Weighted pairwise cross-spectra of one frame (``spectral.py:137-182``)."""

    def __init__(self, values, bin_frequencies, pairs, weighting, phat_floor=0.0,
                 frame_index=0, _rows=None, _row=0, _floors=None):
        self.pairs = tuple(pairs)
        if _rows is not None:
            self._rows, self._row, self._host = _rows, _row, None
            shape = tuple(_rows.tensor.shape[1:])
        else:
            v = np.asarray(values, dtype=complex)
            if v.ndim != 2 or v.shape[0] != len(self.pairs):
                raise ValueError(f"values must have shape (P={len(self.pairs)}, K), got {v.shape}")
            self._rows, self._row, self._host = None, 0, v
            shape = v.shape
        self.bin_frequencies = _as_freqs(bin_frequencies, shape[1])
        if weighting not in WEIGHTINGS:
            raise ValueError(f"unknown weighting {weighting!r}")
        self.weighting = weighting
        # device-computed floors ([F] fp64 rows) are fetched when first read,
        # so building cross-spectra never waits for the device
        self._floors = _floors
        self._phat_floor = None if _floors is not None else float(phat_floor)
        self.frame_index = frame_index
        self._shape = shape

    @property
    def phat_floor(self) -> float:
        if self._phat_floor is None:
            self._phat_floor = float(self._floors.host()[self._row]) \
                if self.weighting == "phat" else 0.0
        return self._phat_floor

    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            self._host = self._rows.host()[self._row]
        return self._host

    def device_values(self, device=None) -> torch.Tensor:
        """[P, K] complex64 on the device (uploaded once if host-born)."""
        dev = N.require_cuda(device)
        if self._rows is not None and self._rows.tensor.device == dev:
            return self._rows.tensor[self._row]
        t = torch.as_tensor(np.ascontiguousarray(self.values, dtype=np.complex64), device=dev)
        self._rows = _DeviceRows(t[None], np.complex128)
        self._rows._host = self._host[None] if self._host is not None else None
        self._row = 0
        return t

    num_pairs = property(lambda self: self._shape[0])
    num_bins = property(lambda self: self._shape[1])


WINDOW_CODES = {"sqrt_hann": 0, "rectangular": 1}


def stft_frames(signals, spec: FrameSpec, device=None, out=None) -> torch.Tensor:
    """K0 on the device: ``signals`` (M, L) (numpy or CUDA tensor) ->
    Y [F, M, K] complex64 CUDA tensor, K = frame_length / 2 (framing, window
    and bins of ``spectral.stft_analyze`` ``spectral.py:185-215``)."""
    dev = N.require_cuda(device)
    if isinstance(signals, torch.Tensor):
        x = signals.to(device=dev, dtype=torch.float32)
        if x.dim() == 1:
            x = x[None, :]
    else:
        a = np.atleast_2d(np.asarray(signals, dtype=float))
        if a.ndim != 2:
            raise ValueError(f"signals must be (M, L), got {a.shape}")
        x = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=dev)
    if x.dim() != 2:
        raise ValueError(f"signals must be (M, L), got {tuple(x.shape)}")
    x = x.contiguous()
    M, L = x.shape
    F = spec.num_frames(L)  # raises for signals shorter than one frame
    Y = out if out is not None else torch.empty((F, M, spec.num_bins), dtype=torch.complex64,
                                                 device=dev)
    N.call("srpb_stft", N.ptr(x), M, L, spec.frame_length, spec.hop_length,
           WINDOW_CODES[spec.window], F, N.ptr(Y), N.stream_handle(dev))
    return Y


def stft_analyze(signals, spec: FrameSpec) -> list:
    """Window, frame and rFFT multichannel audio (``spectral.py:185-215``) on
    the device (K0); frames keep their spectra on the GPU (complex64) until
    ``.spectra`` is read."""
    Y = stft_frames(signals, spec)
    freqs = spec.bin_frequencies()
    return [SpectralFrame(Y[f], freqs, frame_index=f) for f in range(Y.shape[0])]


#: per-frame callers (the reference harness, experiment.py:460-484) pass the
#: same immutable pairs tuple every frame: its index rows (host, and per
#: device) are built once.  Keyed on identity, tuples only (a list may change).
_PAIR_ROWS: dict = {}


def _pair_entry(pairs):
    if isinstance(pairs, tuple):
        e = _PAIR_ROWS.get(id(pairs))
        if e is not None and e[0] is pairs:
            return e
    pm = np.array([p.index_m for p in pairs], dtype=np.int32)
    pmp = np.array([p.index_m_prime for p in pairs], dtype=np.int32)
    e = (pairs, pm, pmp, {})
    if isinstance(pairs, tuple):
        if len(_PAIR_ROWS) >= 16:
            _PAIR_ROWS.clear()
        _PAIR_ROWS[id(pairs)] = e   # holds `pairs`: the id cannot be reused
    return e


def _pair_rows(pairs):
    e = _pair_entry(pairs)
    return e[1], e[2]


def _pair_rows_device(pairs, dev):
    """(pair_m, pair_mp) int32 device tensors of ``pairs`` (cached per device)."""
    e = _pair_entry(pairs)
    t = e[3].get(str(dev))
    if t is None:
        t = (torch.as_tensor(e[1], device=dev), torch.as_tensor(e[2], device=dev))
        e[3][str(dev)] = t
    return t


def gcc_phat_batch(Y: torch.Tensor, pair_m, pair_mp, weighting="phat", phat_floor=None):
    """K1 over a device batch ``Y`` [F, M, K] complex64 -> (Psi, floors)."""
    if weighting not in WEIGHTINGS:
        raise ValueError(f"unknown weighting {weighting!r}")
    dev = N.require_cuda(Y.device)
    F, M, K = Y.shape
    abs_floor = -1.0
    if weighting == "phat" and phat_floor is not None:
        if not (phat_floor > 0 and math.isfinite(phat_floor)):
            raise ValueError(f"phat_floor must be positive, got {phat_floor}")
        abs_floor = float(phat_floor)
    if isinstance(pair_m, torch.Tensor):
        pm, pmp = pair_m, pair_mp
    else:
        pm = torch.as_tensor(np.asarray(pair_m, dtype=np.int32), device=dev)
        pmp = torch.as_tensor(np.asarray(pair_mp, dtype=np.int32), device=dev)
    P = pm.numel()
    psi = torch.empty((F, P, K), dtype=torch.complex64, device=dev)
    floors = torch.empty(F, dtype=torch.float64, device=dev)
    N.call("srpb_gcc_phat", N.ptr(Y.contiguous()), F, M, K, N.ptr(pm), N.ptr(pmp), P,
           0 if weighting == "phat" else 1, DEFAULT_PHAT_FLOOR_REL, abs_floor, N.ptr(psi),
           N.ptr(floors), N.stream_handle(dev))
    return psi, floors


def cross_spectrum_frames(frames, pairs, weighting="phat", phat_floor=None, device=None):
    """Batched :func:`cross_spectrum`: one K1 launch for all frames."""
    if weighting not in WEIGHTINGS:
        raise ValueError(f"unknown weighting {weighting!r}")
    if not pairs:
        raise ValueError("pairs must be non-empty")
    frames = [
        fr if isinstance(fr, SpectralFrame)
        else SpectralFrame(fr.spectra, fr.bin_frequencies, getattr(fr, "frame_index", 0))
        for fr in frames
    ]
    if not frames:
        return []
    pm, pmp = _pair_rows(pairs)
    for fr in frames:
        if int(pm.max()) >= fr.num_channels:
            raise ValueError(
                f"pair index {int(pm.max())} out of range for {fr.num_channels} channels"
            )
    if weighting == "phat" and phat_floor is not None:
        if not (phat_floor > 0 and math.isfinite(phat_floor)):
            raise ValueError(f"phat_floor must be positive, got {phat_floor}")
    shape = (frames[0].num_channels, frames[0].num_bins)
    if any((fr.num_channels, fr.num_bins) != shape for fr in frames):
        return [cross_spectrum(fr, pairs, weighting, phat_floor) for fr in frames]
    dev = N.require_cuda(device)
    Y = (frames[0].device_spectra(dev)[None] if len(frames) == 1   # per-frame callers: a view
         else torch.stack([fr.device_spectra(dev) for fr in frames]))
    psi, floors = gcc_phat_batch(Y, *_pair_rows_device(pairs, dev), weighting, phat_floor)
    rows = _DeviceRows(psi, np.complex128)
    frows = _DeviceRows(floors, np.float64)
    return [
        CrossSpectra(None, fr.bin_frequencies, pairs, weighting, frame_index=fr.frame_index,
                     _rows=rows, _row=i, _floors=frows)
        for i, fr in enumerate(frames)
    ]


def cross_spectrum(frame, pairs, weighting="phat", phat_floor=None) -> CrossSpectra:
    """Pairwise cross-spectra ``psi_p(k) = gamma y_m(k) conj(y_m'(k))``
    (``spectral.py:218-285``) computed by the K1 kernel."""
    if weighting not in WEIGHTINGS:
        raise ValueError(f"unknown weighting {weighting!r}")
    if not pairs:
        raise ValueError("pairs must be non-empty")
    return cross_spectrum_frames([frame], pairs, weighting, phat_floor)[0]
