"""Device-resident SRP plan: the batched entry point of the hot path.

One ``SrpPlan`` holds everything that depends only on geometry, bins and
lattice parameters, uploaded/built once (SURVEY.md 8(b) "plan object caching
device-resident geometry and W"):

* pair index rows (``geometry.py:141-176`` canonical order),
* the conventional steering split ``x = w_1 tau N / 2pi = i + f`` per
  (pair, candidate) -- harmonic bins, ``srp.py:360-373`` -- or the raw fp64
  ``tau``/``omega`` for non-harmonic bins (``srp.py:366-367``),
* lattice layout ``N_p = floor(bound/T)`` (``srp.py:123-134``), reach
  ``N_p + n_aux``, prefix offsets in ``np.concatenate`` order, the padded
  width ``T_pad`` (multiple of 32), and the twiddles ``e^{j w_k n T}``,
* the sinc split ``tau/T = i + f`` and, when it fits, the weight table
  ``W [J, T_pad]`` built on the device (``srp.py:287-317``); otherwise the
  interpolation kernel regenerates the weights on the fly.

All per-frame work goes through ``libsrpb.so``; nothing here computes maps.
"""

from __future__ import annotations

import functools
import math
import os
import threading

import numpy as np
import torch

from . import _native as N
from .geometry import TDOA_BOUND_SLACK

DEFAULT_PHAT_FLOOR_REL = 1e-12  # spectral.py:31-32
#: store W when it needs at most this many bytes (else generate on the fly)
DEFAULT_MAX_WEIGHT_BYTES = 48 << 30
#: conventional batches up to this many frames take the few-frame SIMT kernel
#: (conventional.cu conventional_few_kernel; kFewMaxFrames)
FEW_FRAMES = 4


def is_harmonic(omega: np.ndarray) -> bool:
    """The reference's test for the recurrence branch (``srp.py:359-365``)."""
    omega = np.asarray(omega, dtype=float)
    return bool(
        omega.size >= 2
        and omega[0] == 0.0
        and omega[1] > 0.0
        and np.allclose(np.diff(omega), omega[1], rtol=1e-12, atol=0.0)
    )


def split_rint(x: np.ndarray):
    """fp64 ``x`` -> (int64 rint(x), fp32 x - rint(x)), |fraction| <= 1/2."""
    i = np.rint(x)
    return i.astype(np.int64), (x - i).astype(np.float32)


def _on_plan_device(fn):
    """Run a plan method with the plan's GPU as the current device (the C
    entry points launch on the current device; a plan built for a
    non-current GPU would otherwise launch onto the wrong one)."""
    @functools.wraps(fn)
    def wrapper(self, *args, **kw):
        dev = getattr(self, "device", None)
        if dev is None or dev.index is None or dev.index == torch.cuda.current_device():
            return fn(self, *args, **kw)
        with N.on_device(dev):
            return fn(self, *args, **kw)
    return wrapper


def lattice_layout(tdoa_bounds, sample_period, n_aux):
    """Half counts, reach, prefix offsets, total and padded width."""
    if not (sample_period > 0 and math.isfinite(sample_period)):
        raise ValueError(f"sample_period must be positive, got {sample_period}")
    if n_aux < 0 or int(n_aux) != n_aux:
        raise ValueError(f"n_aux must be a non-negative integer, got {n_aux}")
    halves = tuple(int(math.floor(b / sample_period)) for b in tdoa_bounds)
    reach = np.array([h + int(n_aux) for h in halves], dtype=np.int32)
    counts = 2 * reach + 1
    off = np.zeros(len(halves) + 1, dtype=np.int32)
    off[1:] = np.cumsum(counts)
    total = int(off[-1])
    t_pad = max(32, (total + 31) // 32 * 32)
    return halves, reach, off, total, t_pad


class SrpPlan:
    """Geometry-dependent device state for conventional and approximate maps.

    Parameters
    ----------
    tdoa_table : (J, P) float64 seconds, canonical pair order
    pair_m, pair_mp : (P,) channel indices (``index_m``, ``index_m_prime``)
    tdoa_bounds : (P,) seconds (``MicPair.tdoa_bound``)
    bin_frequencies : (Kb,) rad/s
    sample_period, n_aux : lattice spacing and guard samples (approximate
        path); ``None`` builds the conventional path only
    weights : ``"auto"`` | ``"stored"`` | ``"onthefly"``
    precision : tensor-core operand split, ``"auto"`` (3xFP16 wherever the
        operand bounds are proven -- ``run`` with PHAT weighting -- else
        3xTF32) or ``"tf32"`` (always 3xTF32)
    """

    def __init__(self, *args, device=None, **kw):
        self.device = N.require_cuda(device)
        with N.on_device(self.device):
            self._init(*args, **kw)

    def _init(self, tdoa_table, pair_m, pair_mp, tdoa_bounds, bin_frequencies,
                 sample_period=None, n_aux=None, weights="auto",
                 max_weight_bytes=DEFAULT_MAX_WEIGHT_BYTES, conventional=True, backend="auto",
                 kb_per_group=4, interp_kb_per_group=None, precision="auto", _geometry=None):
        if precision not in ("auto", "tf32"):
            raise ValueError(f"precision must be auto|tf32, got {precision!r}")
        self.precision = precision
        if backend not in ("auto", "simt", "tc"):
            raise ValueError(f"backend must be auto|simt|tc, got {backend!r}")
        self.backend = backend
        # TMEM drain periods (32-column K blocks per accumulator group): the
        # tensor core's accumulation drifts toward zero over long chains, so
        # K2's long K (2 P Kb) folds every 4 blocks (48 MMA steps, ~6e-7);
        # K4's short K (C2: 19 blocks) folds every 10 (120 steps, ~1.5e-6).
        self.kb_per_group = int(kb_per_group)
        self.interp_kb_per_group = 10 if interp_kb_per_group is None else int(interp_kb_per_group)
        # 3xFP16 blocks hold 64 elements but the same 12 MMA accumulations as
        # a tf32 block, and the drift grows with accumulations.  Measured K2
        # rel-L2 vs the oracle at full C2 J / C4's K (tools/conv_kbg_accuracy.py):
        # period 4: 1.5e-6, 8: 3.4e-6, 16: 7.1e-6, 32: 1.1e-5 -> 8 keeps a 3x
        # margin under the 1e-5 tolerance and is ~6% faster than 4
        self.kb_per_group16 = 2 * self.kb_per_group
        # 3xFP16 K4 (stored and on-the-fly weights share it: their maps are
        # bitwise equal): the error is almost all a scale bias growing with
        # the period -- measured at C4 (P = 496, 2246 K blocks, 8 frames x 2048
        # candidates, tools/otf_kbg_accuracy.py): period 10: 2.1e-6, 16:
        # 3.1e-6, 24: 4.6e-6, 32: 6.1e-6; 16 keeps the 3x margin (on-the-fly
        # K4 at C4 shapes 1.5% faster than 10, fewer folds)
        self.interp_kb_per_group16 = (16 if interp_kb_per_group is None
                                      else self.interp_kb_per_group)
        self.W_hi = self.W_lo = None
        self.W16 = None
        omega = np.asarray(bin_frequencies, dtype=np.float64)
        self._geom = _geometry
        if _geometry is not None:  # TDOAs and splits computed on the device
            table = None
            self.J, self.P = int(_geometry["points"].shape[0]), len(pair_m)
            if self.J == 0:
                raise ValueError("the candidate grid is empty")
        else:
            table = np.asarray(tdoa_table, dtype=np.float64)
            if table.ndim != 2 or table.shape[0] == 0:
                raise ValueError(f"tdoa_table must have shape (J, P), got {table.shape}")
            self.J, self.P = table.shape
        self.Kb = omega.size
        if len(pair_m) != self.P or len(pair_mp) != self.P or len(tdoa_bounds) != self.P:
            raise ValueError(f"grid table has {self.P} pair columns, expected {len(pair_m)}")
        self.omega = omega
        self.bounds = np.asarray(tdoa_bounds, dtype=np.float64)
        dev = self.device
        self.pair_m = torch.as_tensor(np.asarray(pair_m, dtype=np.int32), device=dev)
        self.pair_mp = torch.as_tensor(np.asarray(pair_mp, dtype=np.int32), device=dev)
        self.M = int(max(np.max(pair_m), np.max(pair_mp))) + 1
        self.harmonic = is_harmonic(omega)
        self.period = 2 * self.Kb

        self._conv_ready = False
        if conventional:
            self._build_conventional(table)

        self.sample_period = None
        self.n_aux = None
        self.W = None
        if sample_period is not None:
            self._build_lattice(table, float(sample_period), int(n_aux) if n_aux is not None else 0,
                                weights, max_weight_bytes)

    # ------------------------------------------------------------------ build
    def _device_split(self, conv=False, sinc=False, tau=False):
        """srpb_tdoa_split from the plan's device geometry: returns the
        requested (conv_ti, conv_tf), (sx_i, sx_f), tau tensors."""
        g, dev = self._geom, self.device
        J, P = self.J, self.P
        out = {}
        if conv:
            out["conv"] = (torch.empty((P, J), dtype=torch.int32, device=dev),
                           torch.empty((P, J), dtype=torch.float32, device=dev))
        if sinc:
            out["sinc"] = (torch.empty((P, J), dtype=torch.int32, device=dev),
                           torch.empty((P, J), dtype=torch.float32, device=dev))
        if tau:
            out["tau"] = torch.empty((J, P), dtype=torch.float64, device=dev)
        viol = torch.zeros(1, dtype=torch.int32, device=dev)
        ci, cf = out.get("conv", (None, None))
        si, sf = out.get("sinc", (None, None))
        N.call("srpb_tdoa_split", N.ptr(g["pos"]), g["pos"].shape[0], N.ptr(g["points"]), J,
               N.ptr(self.pair_m), N.ptr(self.pair_mp), P, 1 if g["far_field"] else 0,
               float(g["c"]), float(self.omega[1]) if self.Kb > 1 else 0.0, self.period,
               float(getattr(self, "sample_period", None) or 0.0), N.ptr(g["bounds"]),
               TDOA_BOUND_SLACK,
               N.ptr(ci), N.ptr(cf), N.ptr(si), N.ptr(sf), N.ptr(out.get("tau")), N.ptr(viol),
               N.stream_handle(dev))
        if int(viol.item()) != 0:
            raise AssertionError("TDOA magnitude exceeded its physical bound")
        return out

    def _build_conventional(self, table):
        dev = self.device
        if self._geom is not None:
            if self.harmonic:
                self.conv_ti, self.conv_tf = self._device_split(conv=True)["conv"]
            else:
                self.omega_dev = torch.as_tensor(self.omega, device=dev)
                self.tau_dev = self._device_split(tau=True)["tau"]
            self._conv_ready = True
            return
        if self.harmonic:
            # x = w_1 tau N / 2pi: theta_k / 2pi = k x / N (srp.py:370-372)
            x = np.ascontiguousarray((self.omega[1] * table.T) * self.period / (2.0 * math.pi))
            i, f = split_rint(x)
            self.conv_ti = torch.as_tensor(
                np.ascontiguousarray(np.mod(i, self.period), dtype=np.int32), device=dev)
            self.conv_tf = torch.as_tensor(np.ascontiguousarray(f), device=dev)
        else:
            self.omega_dev = torch.as_tensor(self.omega, device=dev)
            self.tau_dev = torch.as_tensor(np.ascontiguousarray(table), device=dev)
        self._conv_ready = True

    def _build_lattice(self, table, T, n_aux, weights, max_weight_bytes):
        dev = self.device
        halves, reach, off, total, t_pad = lattice_layout(self.bounds, T, n_aux)
        self.sample_period, self.n_aux = T, n_aux
        self.half_counts, self.total_samples, self.T_pad = halves, total, t_pad
        self.reach_np, self.off_np = reach, off
        self.reach = torch.as_tensor(reach, device=dev)
        self.off = torch.as_tensor(off, device=dev)
        self.L = int(reach.max())
        self.omega_dev = torch.as_tensor(self.omega, device=dev)
        self.twiddles = torch.empty((self.Kb, (self.L + 16) // 16 * 16, 2), dtype=torch.float32,
                                    device=dev)
        s = N.stream_handle(dev)
        N.call("srpb_lattice_twiddles", N.ptr(self.omega_dev), self.Kb, T, self.L,
               N.ptr(self.twiddles), s)
        # tensor-core lattice (PHAT, fp16 split): B = [cos; -sin] rows per lag
        # slot, 3xFP16 (srpb_lattice_tc_twiddles); shapes it serves: Kb a
        # multiple of 32, 2L + 1 <= 1024 lag slots (passes of 64 slots beyond 64)
        self.tc_twiddles = None
        n_tc = (2 * self.L + 1 + 15) // 16 * 16
        if self.Kb % 32 == 0 and self.Kb >= 64 and n_tc <= 1024:
            self.tc_twiddles = tuple(torch.empty((n_tc, 2 * self.Kb), dtype=torch.float16,
                                                 device=dev) for _ in range(2))
            N.call("srpb_lattice_tc_twiddles", N.ptr(self.omega_dev), self.Kb, T, self.L,
                   N.ptr(self.tc_twiddles[0]), N.ptr(self.tc_twiddles[1]), s)
        self.lattice_tc = self.tc_twiddles is not None  # user toggle (A/B tests)
        # floor fix-up inside the tensor-core lattice (frame counters) or as
        # its own kernel: measured, the separate kernel overlapped by PDL is
        # ~2 us faster per C2 step (the in-kernel completion adds a fence +
        # atomics + flag test to every tile's tail); SRPB_FIXUP_FUSED=1 flips it
        self.lattice_fixup_fused = os.environ.get("SRPB_FIXUP_FUSED", "0") == "1"
        # sinc split x = tau / T (srp.py:310)
        if self._geom is not None:
            self.sx_i, self.sx_f = self._device_split(sinc=True)["sinc"]
        else:
            xs = np.ascontiguousarray(table.T) / T
            i, f = split_rint(xs)
            if np.any(np.abs(i) > 2**30):
                raise ValueError("tdoa / sample_period out of int32 range")
            self.sx_i = torch.as_tensor(np.ascontiguousarray(i, dtype=np.int32), device=dev)
            self.sx_f = torch.as_tensor(np.ascontiguousarray(f), device=dev)
        need = self.J * t_pad * 4
        if weights not in ("auto", "stored", "onthefly"):
            raise ValueError(f"weights must be auto|stored|onthefly, got {weights!r}")
        store = weights == "stored" or (weights == "auto" and need <= max_weight_bytes)
        if store:
            self.W = torch.empty((self.J, t_pad), dtype=torch.float32, device=dev)
            N.call("srpb_sinc_table", N.ptr(self.sx_i), N.ptr(self.sx_f), self.J, self.P,
                   N.ptr(self.off), N.ptr(self.reach), t_pad, N.ptr(self.W), s)
        self.weight_mode = "stored" if store else "onthefly"

    # ---------------------------------------------------------------- helpers
    _owner_tls = threading.local()

    def _state_owner(self):
        """Key of the launch context that owns the persistent kernel state:
        the CapturedStep being captured (its graph replays reuse the same
        pointers), else the current stream.  Two launches that could run
        concurrently never share a cursor / key buffer."""
        owner = getattr(SrpPlan._owner_tls, "owner", None)
        if owner is not None:
            return ("graph", owner)
        return ("stream", torch.cuda.current_stream(self.device).cuda_stream)

    def _argmax_state(self, F):
        """Persistent zeroed (keys [F], done counter + item cursor) for the
        tensor-core kernels' dynamic item scheduling and in-kernel argmax
        finish: the last CTA decodes the keys and resets all three, so no
        reset / decode launches are needed per call.  One set per (F, owner):
        kernels in flight on different streams or graphs never share one."""
        st = getattr(self, "_am_state", None)
        if st is None:
            st = self._am_state = {}
        key = (F, self._state_owner())
        if key not in st:
            # done counter [0] and the dynamic item cursor [1]
            st[key] = (torch.zeros(F, dtype=torch.int64, device=self.device),
                       torch.zeros(2, dtype=torch.int32, device=self.device))
        return st[key]

    def _frame_counters(self, F):
        """Persistent zeroed per-frame counters of the in-kernel floor fix-up
        (the kernel leaves them zero), one set per (F, owner)."""
        st = getattr(self, "_fc_state", None)
        if st is None:
            st = self._fc_state = {}
        key = (F, self._state_owner())
        if key not in st:
            st[key] = torch.zeros(F, dtype=torch.int32, device=self.device)
        return st[key]

    def _keys(self, F):
        keys = torch.empty(F, dtype=torch.int64, device=self.device)
        N.call("srpb_argmax_keys_reset", N.ptr(keys), F, N.stream_handle(self.device))
        return keys

    def keys_to_index(self, keys):
        idx = torch.empty(keys.numel(), dtype=torch.int32, device=self.device)
        N.call("srpb_keys_to_index", N.ptr(keys), keys.numel(), N.ptr(idx),
               N.stream_handle(self.device))
        return idx

    def _check_frames(self, t, shape_tail, dtype, name):
        if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.dtype != dtype or tuple(t.shape[1:]) != tuple(shape_tail) or not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous {dtype} [F, {shape_tail}], got "
                             f"{t.dtype} {tuple(t.shape)}")

    # -------------------------------------------------------------- hot path
    def _check_spectra(self, Y, weighting, phat_floor):
        """Validate ``Y`` [F, M, Kb] complex64 -> (F, weighting code, abs floor)."""
        if weighting not in ("phat", "identity"):
            raise ValueError(f"unknown weighting {weighting!r}")
        if Y.dim() != 3 or Y.shape[2] != self.Kb:
            raise ValueError(f"Y must be [F, M, {self.Kb}], got {tuple(Y.shape)}")
        if Y.shape[1] < self.M:
            raise ValueError(f"pair index {self.M - 1} out of range for {Y.shape[1]} channels")
        self._check_frames(Y, (Y.shape[1], self.Kb), torch.complex64, "Y")
        abs_floor = -1.0
        if weighting == "phat" and phat_floor is not None:
            if not (phat_floor > 0 and math.isfinite(phat_floor)):
                raise ValueError(f"phat_floor must be positive, got {phat_floor}")
            abs_floor = float(phat_floor)
        return Y.shape[0], (0 if weighting == "phat" else 1), abs_floor

    @_on_plan_device
    def cross_spectra(self, Y, weighting="phat", phat_floor=None, out=None):
        """K1: ``Y`` [F, M, Kb] complex64 -> (Psi [F, P, Kb] complex64,
        applied floors [F] float64)."""
        F, wcode, abs_floor = self._check_spectra(Y, weighting, phat_floor)
        psi = out if out is not None else torch.empty((F, self.P, self.Kb), dtype=torch.complex64,
                                                      device=self.device)
        floors = torch.empty(F, dtype=torch.float64, device=self.device)
        N.call("srpb_gcc_phat", N.ptr(Y), F, Y.shape[1], self.Kb, N.ptr(self.pair_m),
               N.ptr(self.pair_mp), self.P, wcode, DEFAULT_PHAT_FLOOR_REL, abs_floor, N.ptr(psi),
               N.ptr(floors), N.stream_handle(self.device))
        return psi, floors

    @_on_plan_device
    def lattice_from_spectra(self, Y, weighting="phat", phat_floor=None, split=False):
        """K1a + fused K1b/K3: ``Y`` [F, M, Kb] -> Xi [F, T_pad] fp32, or its
        tensor-core operand split (Xi_hi, Xi_lo): ``split=True`` / ``"tf32"``
        tf32 floats, ``"f16"`` fp16 of ``xi_scale16 * Xi`` (PHAT only).  The
        cross-spectra are formed inside the lattice kernel and never stored."""
        if self.sample_period is None:
            raise ValueError("plan was built without a lattice (sample_period)")
        F, wcode, abs_floor = self._check_spectra(Y, weighting, phat_floor)
        if split is True:
            split = "tf32"
        if split not in (False, "tf32", "f16"):
            raise ValueError(f"split must be False|'tf32'|'f16', got {split!r}")
        if split == "f16" and wcode != 0:
            raise ValueError("the fp16 split needs PHAT-bounded lattice samples")
        s = N.stream_handle(self.device)
        # PHAT with the relative floor: applied speculatively inside the
        # lattice call (no floor pass); an explicit floor needs no pass either
        floors = clean = None
        shape = (F, self.T_pad)
        scale = 0.0
        if split:
            dt = torch.float16 if split == "f16" else torch.float32
            outs = (None, torch.empty(shape, dtype=dt, device=self.device),
                    torch.empty(shape, dtype=dt, device=self.device))
            scale = self.xi_scale16 if split == "f16" else 0.0
        else:
            outs = (torch.empty(shape, dtype=torch.float32, device=self.device), None, None)
        spec = None
        if wcode == 0 and abs_floor <= 0:  # speculative floor statistics
            spec = torch.empty(3 * F * self.P, dtype=torch.float32, device=self.device)
        args = (N.ptr(Y), F, Y.shape[1], self.Kb, N.ptr(self.pair_m), N.ptr(self.pair_mp),
                self.P, wcode, N.ptr(floors), abs_floor, N.ptr(clean), N.ptr(self.twiddles),
                self.L, N.ptr(self.off), N.ptr(self.reach), self.T_pad,
                *(N.ptr(o) for o in outs), float(scale), DEFAULT_PHAT_FLOOR_REL, N.ptr(spec))
        # the tensor-core path also needs the tile's spectra and Xi rows to
        # fit its shared-memory ring: the C side decides, ask it
        if (split == "f16" and self.lattice_tc and spec is not None and N.query(
                "srpb_lattice_tc_supported", Y.shape[1], self.P, self.Kb, self.L, self.T_pad)):
            # K1b + K3 as one tensor-core GEMM over (frame, pair) rows; the
            # floor fix-up runs inside it (persistent zeroed frame counters)
            cnt = self._frame_counters(F) if self.lattice_fixup_fused else None
            self._main("srpb_lattice_from_spectra_tc", *args, N.ptr(self.tc_twiddles[0]),
                       N.ptr(self.tc_twiddles[1]), N.ptr(cnt), s)
            if cnt is not None:
                N.note_launches(-1)  # the fix-up ran inside the lattice kernel
        else:
            self._main("srpb_lattice_from_spectra", *args, s)
        return outs[1:] if split else outs[0]

    def _use_tc(self, F, kind):
        """Tensor-core kernels whenever the plan allows them (not a backend
        switch: both families are this library's sm_100a kernels).  Measured
        at C5 (J = 200k): even at F = 1 the tcgen05 kernels win (the steering
        phases / weights dominate and are shared by the frames of a tile), so
        the SIMT kernels serve only shapes the tensor-core path cannot take
        (Kb % 16 != 0, non-harmonic bins, tf32 without a stored W) -- and
        conventional batches of <= FEW_FRAMES frames with harmonic bins, which
        the per-candidate phase-recurrence kernel serves (C5 batch 1: 2.83 ms
        on the tensor cores, whose frame tile is 31/32 idle there)."""
        if self.backend == "simt":
            return False
        if kind == "conv":
            if self.backend != "tc" and self.harmonic and F <= FEW_FRAMES:
                return False
            ok = self.harmonic and self.Kb % 16 == 0
        elif kind == "interp16":  # 3xFP16 K4: stored W or weights generated in TMEM
            ok = True
        else:                     # 3xTF32 K4 needs the stored W
            ok = self.W is not None
        if self.backend == "tc" and not ok:
            raise ValueError(f"tensor-core {kind} path unavailable for this plan")
        return ok

    #: optional profiler hook: an object with before(name) / after(name)
    #: called around each main kernel launch (bench.py records CUDA events)
    kernel_timer = None

    def _main(self, name, *args):
        t = self.kernel_timer
        if t is not None:
            t.before(name)
        N.call(name, *args)
        if t is not None:
            t.after(name)

    def split_tf32(self, x):
        """(hi, lo) tf32 operand split of a float32/complex64 tensor."""
        xf = torch.view_as_real(x) if x.is_complex() else x
        hi = torch.empty(xf.shape, dtype=torch.float32, device=self.device)
        lo = torch.empty_like(hi)
        N.call("srpb_tf32_split", N.ptr(xf), xf.numel(), N.ptr(hi), N.ptr(lo),
               N.stream_handle(self.device))
        return hi, lo

    # 3xFP16 prescales (powers of two): |phase|, |W|, PHAT |psi| <= 1; PHAT
    # lattice samples |xi| <= 2 sum_k |psi_k| <= 2 Kb
    F16_UNIT_SCALE = 2.0 ** 14

    @property
    def xi_scale16(self):
        return self.f16_scale_for_bins(self.Kb)

    @staticmethod
    def f16_scale_for_bins(kb):
        """Power-of-two prescale keeping PHAT lattice samples (|xi| <= 2 kb)
        inside fp16's range."""
        return 2.0 ** math.floor(math.log2(60000.0 / (2.0 * max(int(kb), 1))))

    def split_f16(self, x, scale):
        """(hi, lo) fp16 split of scale * x (float32/complex64 tensor)."""
        xf = torch.view_as_real(x) if x.is_complex() else x
        hi = torch.empty(xf.shape, dtype=torch.float16, device=self.device)
        lo = torch.empty_like(hi)
        N.call("srpb_f16_split", N.ptr(xf), xf.numel(), float(scale), N.ptr(hi), N.ptr(lo),
               N.stream_handle(self.device))
        return hi, lo

    def _f16_ok(self, kind, bounded):
        """3xFP16 tensor-core path for this contraction?"""
        if self.precision != "auto" or not bounded:
            return False
        if kind == "conv":
            return self.harmonic and self.Kb % 32 == 0
        return True  # stored W, or weights generated in TMEM

    @_on_plan_device
    def conventional(self, psi, maps=True, maps_out=None, _bounded=False):
        """K2 (+ fused K5): Psi [F, P, Kb] -> (maps [F, J] fp32 | None,
        argmax [F] int32)."""
        if not self._conv_ready:
            raise ValueError("plan was built without the conventional path")
        self._check_frames(psi, (self.P, self.Kb), torch.complex64, "psi")
        F = psi.shape[0]
        out = None
        if maps:
            out = maps_out if maps_out is not None else torch.empty(
                (F, self.J), dtype=torch.float32, device=self.device)
        s = N.stream_handle(self.device)
        if self._use_tc(F, "conv") and self._f16_ok("conv", _bounded):
            hi, lo = self.split_f16(psi, self.F16_UNIT_SCALE)
            return self._conventional_tc16(hi, lo, F, maps, out)
        keys = self._keys(F)
        if self._use_tc(F, "conv"):
            hi, lo = self.split_tf32(psi)
            self._main("srpb_conventional_tc", N.ptr(hi), N.ptr(lo), F, self.P, self.Kb, self.period,
                   N.ptr(self.conv_ti), N.ptr(self.conv_tf), self.J, N.ptr(out), N.ptr(keys),
                   self.kb_per_group, s)
        elif self.harmonic:
            self._main("srpb_conventional", N.ptr(psi), F, self.P, self.Kb, self.period,
                   N.ptr(self.conv_ti), N.ptr(self.conv_tf), self.J, N.ptr(out), N.ptr(keys), s)
        else:
            self._main("srpb_conventional_general", N.ptr(psi), F, self.P, self.Kb,
                   N.ptr(self.omega_dev), N.ptr(self.tau_dev), self.J, N.ptr(out), N.ptr(keys), s)
        return out, self.keys_to_index(keys)

    def _conventional_tc16(self, hi, lo, F, maps=True, out=None):
        """K2 on the fp16 operand split of psi (x F16_UNIT_SCALE), argmax
        finished in-kernel."""
        if maps and out is None:
            out = torch.empty((F, self.J), dtype=torch.float32, device=self.device)
        keys, done = self._argmax_state(F)
        idx = torch.empty(F, dtype=torch.int32, device=self.device)
        self._main("srpb_conventional_tc16", N.ptr(hi), N.ptr(lo), self.F16_UNIT_SCALE, F,
                   self.P, self.Kb, self.period, N.ptr(self.conv_ti), N.ptr(self.conv_tf),
                   self.J, N.ptr(out if maps else None), N.ptr(keys), self.kb_per_group16,
                   N.ptr(idx), N.ptr(done), N.stream_handle(self.device))
        return (out if maps else None), idx

    @_on_plan_device
    def lattice(self, psi, out=None):
        """K3: Psi [F, P, Kb] -> Xi [F, T_pad] fp32 (pad columns zero)."""
        if self.sample_period is None:
            raise ValueError("plan was built without a lattice (sample_period)")
        self._check_frames(psi, (self.P, self.Kb), torch.complex64, "psi")
        F = psi.shape[0]
        xi = out if out is not None else torch.empty((F, self.T_pad), dtype=torch.float32,
                                                     device=self.device)
        self._main("srpb_lattice", N.ptr(psi), F, self.P, self.Kb, N.ptr(self.twiddles), self.L,
               N.ptr(self.off), N.ptr(self.reach), self.T_pad, N.ptr(xi),
               N.stream_handle(self.device))
        return xi

    @_on_plan_device
    def approx(self, xi, maps=True, maps_out=None, bounded=False):
        """K4 (+ fused K5): Xi [F, T_pad] -> (maps [F, J] | None, argmax [F]).
        ``bounded``: False, or the bin count Kb' of the PHAT cross-spectra the
        samples come from (|xi| <= 2 Kb'): then the 3xFP16 tensor-core kernel
        (argmax finished in-kernel) applies with a prescale for that bound."""
        if self.sample_period is None:
            raise ValueError("plan was built without a lattice (sample_period)")
        self._check_frames(xi, (self.T_pad,), torch.float32, "xi")
        F = xi.shape[0]
        out = None
        if maps:
            out = maps_out if maps_out is not None else torch.empty(
                (F, self.J), dtype=torch.float32, device=self.device)
        if bounded and self._f16_ok("interp", True) and self._use_tc(F, "interp16"):
            scale = self.f16_scale_for_bins(int(bounded))
            xh, xl = self.split_f16(xi, scale)
            return self._approx_tc16(xh, xl, out, xi_scale=scale)
        keys = self._keys(F)
        s = N.stream_handle(self.device)
        if self._use_tc(F, "interp"):
            return self._approx_tc(*self.split_tf32(xi), out, keys)
        elif self.W is not None:
            self._main("srpb_interp", N.ptr(self.W), N.ptr(xi), F, self.J, self.T_pad, N.ptr(out),
                   N.ptr(keys), s)
        else:
            self._main("srpb_interp_onthefly", N.ptr(self.sx_i), N.ptr(self.sx_f), self.P,
                   N.ptr(self.off), N.ptr(self.reach), N.ptr(xi), F, self.J, self.T_pad,
                   N.ptr(out), N.ptr(keys), s)
        return out, self.keys_to_index(keys)

    def _approx_tc16(self, xh, xl, out, xi_scale=None):
        """K4 in 3xFP16 from the fp16 split of xi_scale16 * Xi (weights from
        the stored W split, or generated in tensor memory when W is not
        stored); argmax finished in-kernel."""
        F = xh.shape[0]
        xs = self.xi_scale16 if xi_scale is None else xi_scale
        keys, done = self._argmax_state(F)
        idx = torch.empty(F, dtype=torch.int32, device=self.device)
        if self.W is None:
            self._main("srpb_interp_tc16_onthefly", N.ptr(self.sx_i), N.ptr(self.sx_f), self.P,
                       N.ptr(self.off), N.ptr(self.reach), N.ptr(xh), N.ptr(xl),
                       xs, F, self.J, self.T_pad, N.ptr(out), N.ptr(keys),
                       self.interp_kb_per_group16, N.ptr(idx), N.ptr(done),
                       N.stream_handle(self.device))
            return out, idx
        if self.W16 is None:
            self.W16 = self.split_f16(self.W, self.F16_UNIT_SCALE)
        self._main("srpb_interp_tc16", N.ptr(self.W16[0]), N.ptr(self.W16[1]),
                   self.F16_UNIT_SCALE, N.ptr(xh), N.ptr(xl), xs, F, self.J, self.T_pad,
                   N.ptr(out), N.ptr(keys), self.interp_kb_per_group16, N.ptr(idx), N.ptr(done),
                   N.stream_handle(self.device))
        return out, idx

    def _approx_tc(self, xh, xl, out, keys):
        if self.W_hi is None:
            self.W_hi, self.W_lo = self.split_tf32(self.W)
        self._main("srpb_interp_tc", N.ptr(self.W_hi), N.ptr(self.W_lo), N.ptr(xh), N.ptr(xl),
                   xh.shape[0], self.J, self.T_pad, N.ptr(out), N.ptr(keys),
                   self.interp_kb_per_group, N.stream_handle(self.device))
        return out, self.keys_to_index(keys)

    @_on_plan_device
    def argmax(self, maps):
        """K5 standalone over stored maps [F, J] fp32."""
        if maps.dim() != 2 or maps.dtype != torch.float32 or not maps.is_contiguous():
            raise ValueError("maps must be contiguous float32 [F, J]")
        F, J = maps.shape
        keys = self._keys(F)
        N.call("srpb_argmax", N.ptr(maps), F, J, N.ptr(keys), N.stream_handle(self.device))
        return self.keys_to_index(keys)

    @_on_plan_device
    def run(self, Y, path="approx", maps=True, weighting="phat", phat_floor=None):
        """Y [F, M, Kb] complex64 -> (maps | None, argmax) along ``path``.
        The approximate path fuses K1's cross-spectra into K3; with PHAT
        weighting the contractions run in 3xFP16 (bounded operands)."""
        bounded = weighting == "phat"
        if path == "conventional":
            F = Y.shape[0]
            if (bounded and self._conv_ready and self.harmonic and self.Kb % 2 == 0
                    and self._use_tc(F, "conv") and self._f16_ok("conv", True)):
                # K1 writes the fp16 operand split of psi directly (no psi
                # round trip through HBM, no split pass)
                F, wcode, abs_floor = self._check_spectra(Y, weighting, phat_floor)
                hi = torch.empty((F, 2 * self.P * self.Kb), dtype=torch.float16, device=self.device)
                lo = torch.empty_like(hi)
                floors = torch.empty(F, dtype=torch.float64, device=self.device)
                self._main("srpb_gcc_phat_split16", N.ptr(Y), F, Y.shape[1], self.Kb,
                           N.ptr(self.pair_m), N.ptr(self.pair_mp), self.P, wcode,
                           DEFAULT_PHAT_FLOOR_REL, abs_floor, None, N.ptr(hi), N.ptr(lo),
                           self.F16_UNIT_SCALE, N.ptr(floors), N.stream_handle(self.device))
                return self._conventional_tc16(hi, lo, F, maps)
            psi, _ = self.cross_spectra(Y, weighting, phat_floor)
            return self.conventional(psi, maps, _bounded=bounded)
        if path == "approx":
            F = Y.shape[0]
            f16 = self._f16_ok("interp", bounded)
            if self.sample_period is not None and self._use_tc(F, "interp16" if f16 else "interp"):
                out = torch.empty((F, self.J), dtype=torch.float32,
                                  device=self.device) if maps else None
                if f16:
                    xh, xl = self.lattice_from_spectra(Y, weighting, phat_floor, split="f16")
                    return self._approx_tc16(xh, xl, out)
                xh, xl = self.lattice_from_spectra(Y, weighting, phat_floor, split=True)
                return self._approx_tc(xh, xl, out, self._keys(F))
            return self.approx(self.lattice_from_spectra(Y, weighting, phat_floor), maps)
        raise ValueError(f"unknown path {path!r}")

    @classmethod
    def from_geometry(cls, mic_positions, points, bin_frequencies, speed_of_sound=340.0,
                      far_field=False, pair_m=None, pair_mp=None, **kw):
        """Build a plan without a host TDOA table: the candidate TDOAs and
        their phase / sinc splits are computed on the device
        (``srpb_tdoa_split``; geometry.build_tdoa_table ``geometry.py:365-398``).
        Pairs default to the canonical order (``geometry.py:141-176``);
        bounds are pair distance / c.  ``points`` are candidate positions
        (near field) or unit directions (far field).  Other keywords as in
        ``SrpPlan``."""
        pos = np.ascontiguousarray(mic_positions, dtype=np.float64)
        pts = np.ascontiguousarray(points, dtype=np.float64)
        if pos.ndim != 2 or pos.shape[1] != 3 or pts.ndim != 2 or pts.shape[1] != 3:
            raise ValueError("mic_positions and points must be (M, 3) and (J, 3)")
        if pair_m is None:
            pairs = [(m, mp) for mp in range(pos.shape[0]) for m in range(mp + 1, pos.shape[0])]
            pair_m = np.array([m for m, _ in pairs], dtype=np.int32)
            pair_mp = np.array([mp for _, mp in pairs], dtype=np.int32)
        pm, pmp = np.asarray(pair_m), np.asarray(pair_mp)
        dist = np.linalg.norm(pos[pm] - pos[pmp], axis=1)
        if np.any(dist == 0.0):
            raise ValueError("coincident microphones in a pair")
        bounds = dist / speed_of_sound
        dev = N.require_cuda(kw.get("device"))
        geom = {"pos": torch.as_tensor(pos, device=dev), "points": torch.as_tensor(pts, device=dev),
                "far_field": bool(far_field), "c": float(speed_of_sound),
                "bounds": torch.as_tensor(bounds, device=dev)}
        return cls(None, pm, pmp, bounds, bin_frequencies, _geometry=geom, **kw)

    @_on_plan_device
    def stft(self, x, frame_length, hop_length=None, window="sqrt_hann", out=None):
        """K0: audio ``x`` [M, L] float32 (CUDA) -> Y [F, M, frame_length/2]
        complex64 (``spectral.stft_analyze`` framing and window)."""
        hop = frame_length // 2 if hop_length is None else int(hop_length)
        if frame_length // 2 != self.Kb:
            raise ValueError(f"frame_length {frame_length} gives {frame_length // 2} bins, plan "
                             f"has {self.Kb}")
        if window not in ("sqrt_hann", "rectangular"):
            raise ValueError(f"window must be one of ('sqrt_hann', 'rectangular'), got {window!r}")
        if not isinstance(x, torch.Tensor) or x.device.type != "cuda" or x.dim() != 2 \
                or x.dtype != torch.float32 or not x.is_contiguous():
            raise ValueError("x must be a contiguous float32 CUDA tensor [M, L]")
        M, L = x.shape
        if L < frame_length:
            raise ValueError(f"signal of {L} samples is shorter than one frame ({frame_length})")
        F = (L - frame_length) // hop + 1
        Y = out if out is not None else torch.empty((F, M, self.Kb), dtype=torch.complex64,
                                                     device=self.device)
        N.call("srpb_stft", N.ptr(x), M, L, frame_length, hop,
               0 if window == "sqrt_hann" else 1, F, N.ptr(Y), N.stream_handle(self.device))
        return Y

    @_on_plan_device
    def run_audio(self, x, frame_length, hop_length=None, window="sqrt_hann", path="approx",
                  maps=True, weighting="phat", phat_floor=None):
        """K0 + ``run``: audio [M, L] -> (maps | None, argmax) per frame."""
        return self.run(self.stft(x, frame_length, hop_length, window), path, maps, weighting,
                        phat_floor)

    def capture(self, F, M=None, path="approx", maps=True, weighting="phat", phat_floor=None,
                audio=None):
        """Capture ``run`` for F frames of M channels into a CUDA graph
        (``CapturedStep``: static input, ``replay()``); ``audio=(L,
        frame_length, hop_length, window)`` captures STFT + run from [M, L]
        audio instead (F is then derived from L)."""
        return CapturedStep(self, F, M if M is not None else self.M, path, maps, weighting,
                            phat_floor, audio)


def standalone_argmax(maps: torch.Tensor) -> torch.Tensor:
    """K5 over any [F, J] fp32 CUDA tensor (no plan needed)."""
    N.require_cuda(maps.device)
    if maps.dim() == 1:
        maps = maps[None, :]
    maps = maps.contiguous()
    F, J = maps.shape
    s = N.stream_handle(maps.device)
    keys = torch.empty(F, dtype=torch.int64, device=maps.device)
    N.call("srpb_argmax_keys_reset", N.ptr(keys), F, s)
    N.call("srpb_argmax", N.ptr(maps), F, J, N.ptr(keys), s)
    idx = torch.empty(F, dtype=torch.int32, device=maps.device)
    N.call("srpb_keys_to_index", N.ptr(keys), F, N.ptr(idx), s)
    return idx


class CapturedStep:
    """One ``SrpPlan.run`` step captured in a CUDA graph.

    The step's kernels (K1a floor, fused K1b/K3 lattice, K4/K2 tensor-core
    contraction with the fused argmax, argmax key reset/decode; with
    ``audio=(L, frame_length, hop_length, window)`` also the K0 STFT) replay
    with a single graph launch, so host-side work (argument marshalling,
    tensor-map encoding) leaves the critical path.  The static input is ``Y``
    [F, M, Kb] complex64 or, for audio, ``x`` [M, L] float32; ``maps`` /
    ``argmax`` are the static outputs, overwritten by each replay.
    """

    def __init__(self, plan, F, M, path="approx", maps=True, weighting="phat", phat_floor=None,
                 audio=None):
        dev = plan.device
        self.plan, self.path = plan, path
        self.audio = audio
        if audio is not None:
            L, n, hop, window = audio
            hop = n // 2 if hop is None else int(hop)
            self.audio = (int(L), int(n), hop, window)
            self.x = torch.zeros((M, int(L)), dtype=torch.float32, device=dev)
            F = (int(L) - n) // hop + 1
        self.Y = torch.zeros((F, M, plan.Kb), dtype=torch.complex64, device=dev)
        timer, plan.kernel_timer = plan.kernel_timer, None

        def body():
            if self.audio is not None:
                _, n_, hop_, win_ = self.audio
                plan.stft(self.x, n_, hop_, win_, out=self.Y)
            return plan.run(self.Y, path, maps, weighting, phat_floor)

        tls = SrpPlan._owner_tls
        prev_owner = getattr(tls, "owner", None)
        try:
            # the graph owns its kernels' persistent state (keys, cursor):
            # replays of different steps may overlap on different streams
            tls.owner = id(self)
            with N.on_device(dev):
                # warm-up outside capture: lazily built operands (fp16 W
                # split), kernel attributes, allocator pools
                body()
                torch.cuda.synchronize(dev)
                self.graph = torch.cuda.CUDAGraph()
                n0 = N.launch_count()
                with torch.cuda.graph(self.graph):
                    self.maps, self.argmax = body()
                #: kernels launched by one replay
                self.launches = N.launch_count() - n0
        finally:
            tls.owner = prev_owner
            plan.kernel_timer = timer

    @property
    def input(self):
        """The static input buffer (``x`` for audio steps, else ``Y``)."""
        return self.x if self.audio is not None else self.Y

    def replay(self, inp=None):
        """Run the step (on the current stream); ``inp`` (optional) is copied
        into the static input first.  Returns the static (maps, argmax)."""
        if inp is not None:
            self.input.copy_(inp, non_blocking=True)
        self.graph.replay()
        return self.maps, self.argmax
