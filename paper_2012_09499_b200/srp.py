"""Drop-in for ``srpfast.srp`` on the B200 path.

Same names, signatures, validation errors (types and messages) and counter
semantics as the reference (``pkg/src/srpfast/srp.py``); every map, lattice
and sinc table is computed by ``libsrpb.so`` kernels through
:class:`~.plan.SrpPlan`.  Results stay on the device until a caller reads
``.values`` / ``.samples`` / ``.weights`` (materialised once per batch).

``srp_oracle`` (``srp.py:468-515``), the quadratic-form map the reference
uses to verify its fast paths, runs on the device too, in fp64 with direct
exponentials (``srpb_srp_quadform``): an independent full-scale check of the
conventional path, not a CPU fallback.
"""

from __future__ import annotations

import math
import weakref
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .plan import SrpPlan, is_harmonic, lattice_layout, standalone_argmax
from .spectral import CrossSpectra, _DeviceRows

__all__ = [
    "MultCounter",
    "GccLattice",
    "SincTable",
    "SrpMap",
    "ComplexityReport",
    "gcc_at_lag",
    "lattice_half_counts",
    "build_gcc_lattice",
    "build_gcc_lattice_frames",
    "precompute_sinc_table",
    "srp_conventional",
    "srp_conventional_frames",
    "srp_approx",
    "srp_approx_frames",
    "srp_oracle",
    "srp_oracle_frames",
    "argmax_candidate",
    "complexity_report",
]


@dataclass
class MultCounter:
    """Signal-dependent multiplication tally (``srp.py:53-77``)."""

    complex_mults: int = 0
    real_mults: int = 0

    def add_complex(self, n: int) -> None:
        self.complex_mults += int(n)

    def add_real(self, n: int) -> None:
        self.real_mults += int(n)

    def merge(self, other: "MultCounter") -> None:
        self.complex_mults += other.complex_mults
        self.real_mults += other.real_mults

    def reset(self) -> None:
        self.complex_mults = 0
        self.real_mults = 0


class SrpMap:
    """SRP values over a candidate grid (``srp.py:80-104``).

    ``values`` is a float64 numpy vector like the reference's; maps produced
    on the device keep the fused argmax and fetch values lazily.
    """

    def __init__(self, values, method, frame_index=0, _rows=None, _row=0, _argmax=None,
                 _num=None):
        self.method = method
        self.frame_index = frame_index
        # fused device argmax: an int, or (_DeviceRows of [F] indices, row)
        # fetched on first use (building maps never waits for the device)
        self._argmax = _argmax
        if _rows is not None:
            self._rows, self._row, self._host = _rows, _row, None
            self._n = int(_rows.tensor.shape[1])
        elif values is None and _argmax is not None:  # argmax-only (maps=False)
            self._rows, self._row, self._host, self._n = None, _row, None, int(_num or 0)
        else:
            v = np.asarray(values, dtype=float)
            if v.ndim != 1 or v.size == 0:
                raise ValueError(f"values must be a non-empty vector, got {v.shape}")
            self._rows, self._host, self._n = None, v, v.size

    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            if self._rows is None:
                raise ValueError("map values were not materialised (maps=False); "
                                 "only argmax_candidate is available")
            self._host = self._rows.host()[self._row]
        return self._host

    def device_values(self):
        """The fp32 device row, or None for host-built maps."""
        return None if self._rows is None else self._rows.tensor[self._row]

    @property
    def num_candidates(self) -> int:
        return self._n


def argmax_candidate(srp_map) -> int:
    """Index of the largest value, lowest index on ties (``srp.py:107-109``).

    Device maps return the argmax fused into the K2/K4 epilogue; host maps
    run the K5 reduction (fp64) on the device.
    """
    am = getattr(srp_map, "_argmax", None)
    if isinstance(am, tuple):
        rows, i = am
        return int(rows.host()[i])
    if am is not None:
        return int(am)
    dev_row = srp_map.device_values() if hasattr(srp_map, "device_values") else None
    if dev_row is not None and dev_row.dtype == torch.float32:
        return int(standalone_argmax(dev_row.contiguous())[0].item())
    dev = N.require_cuda()
    if dev_row is not None:  # fp64 device maps (srp_oracle)
        v = dev_row.contiguous()
    else:
        v = torch.as_tensor(np.ascontiguousarray(srp_map.values, dtype=np.float64), device=dev)
    idx = torch.empty(1, dtype=torch.int32, device=dev)
    N.call("srpb_argmax_f64", N.ptr(v), 1, v.numel(), N.ptr(idx), N.stream_handle(dev))
    return int(idx.item())


def _device_psi(crosses, device=None):
    """Stack frames' [P, K] cross-spectra into one [F, P, K] device tensor."""
    dev = N.require_cuda(device)
    rows = [getattr(c, "_rows", None) for c in crosses]
    if rows[0] is not None and all(r is rows[0] for r in rows) and rows[0].tensor.device == dev:
        idx = [c._row for c in crosses]
        t = rows[0].tensor
        if idx == list(range(t.shape[0])):
            return t
        return t[torch.as_tensor(idx, device=dev)].contiguous()
    vals = [
        c.device_values(dev) if isinstance(c, CrossSpectra)
        else torch.as_tensor(np.ascontiguousarray(c.values, dtype=np.complex64), device=dev)
        for c in crosses
    ]
    return (vals[0][None] if len(vals) == 1 else torch.stack(vals)).contiguous()


def gcc_at_lag(cross, pair_index: int, lag: float) -> float:
    """``xi_p(tau) = 2 sum_k Re[psi_p(k) e^{j w_k tau}]`` (``srp.py:112-120``),
    evaluated by the general-bin K2 kernel for one pair and one lag."""
    dev = N.require_cuda()
    psi = _device_psi([cross], dev)[:, pair_index:pair_index + 1, :].contiguous()
    omega = torch.as_tensor(np.asarray(cross.bin_frequencies, dtype=np.float64), device=dev)
    tau = torch.tensor([[float(lag)]], dtype=torch.float64, device=dev)
    out = torch.empty((1, 1), dtype=torch.float32, device=dev)
    N.call("srpb_conventional_general", N.ptr(psi), 1, 1, psi.shape[2], N.ptr(omega),
           N.ptr(tau), 1, N.ptr(out), None, N.stream_handle(dev))
    return float(out.item())


def lattice_half_counts(pairs: Sequence, sample_period: float) -> tuple:
    """``N_p = floor(tdoa_bound / T)`` (``srp.py:123-134``)."""
    if not (sample_period > 0 and math.isfinite(sample_period)):
        raise ValueError(f"sample_period must be positive, got {sample_period}")
    return tuple(int(math.floor(p.tdoa_bound / sample_period)) for p in pairs)


def _lattice_offsets(half_count: int, n_aux: int) -> np.ndarray:
    r = half_count + n_aux
    return np.arange(-r, r + 1)


class GccLattice:
    """Critically sampled GCCs of one frame (``srp.py:143-198``).

    Built on the device, it holds a row of the [F, T_pad] lattice tensor
    (concatenated pair rows, ``np.concatenate`` order); ``samples`` splits
    it into per-pair float64 arrays on first access.
    """

    def __init__(self, sample_period, n_aux, half_counts, samples=None, frame_index=0,
                 _rows=None, _row=0, _plan=None, _bounded=False):
        # _bounded: 0, or Kb of the PHAT cross-spectra the device samples come
        # from (|xi| <= 2 Kb: the 3xFP16 interpolation's operand bound)
        self._bounded = int(_bounded)
        self.sample_period = float(sample_period)
        self.n_aux = int(n_aux)
        self.half_counts = tuple(int(h) for h in half_counts)
        self.frame_index = frame_index
        self._rows, self._row, self._plan = _rows, _row, _plan
        self._samples = None
        if _rows is None:
            samples = tuple(np.asarray(s, dtype=float) for s in samples)
            if len(samples) != len(self.half_counts):
                raise ValueError("one sample row per half count required")
            for n_p, row in zip(self.half_counts, samples):
                if row.shape != (2 * (n_p + self.n_aux) + 1,):
                    raise ValueError(
                        f"pair with N_p={n_p} must hold {2 * (n_p + self.n_aux) + 1} "
                        f"samples, got {row.shape}"
                    )
            self._samples = samples

    @property
    def samples(self) -> tuple:
        if self._samples is None:
            flat = self._rows.host()[self._row]
            off = np.cumsum([0] + [2 * (h + self.n_aux) + 1 for h in self.half_counts])
            self._samples = tuple(flat[off[p]:off[p + 1]].astype(float)
                                  for p in range(len(self.half_counts)))
        return self._samples

    @property
    def num_pairs(self) -> int:
        return len(self.half_counts)

    @property
    def pair_counts(self) -> tuple:
        return tuple(2 * (h + self.n_aux) + 1 for h in self.half_counts)

    @property
    def total_samples(self) -> int:
        return sum(self.pair_counts)

    @property
    def average_count(self) -> float:
        return 2.0 / self.num_pairs * sum(self.half_counts) + 2.0 * self.n_aux + 1.0

    def lag_offsets(self, pair_index: int) -> np.ndarray:
        return _lattice_offsets(self.half_counts[pair_index], self.n_aux)

    def device_row(self, t_pad: int, device=None) -> torch.Tensor:
        """[T_pad] fp32 device row (uploads host-built samples once)."""
        dev = N.require_cuda(device)
        if self._rows is not None and self._rows.tensor.device == dev \
                and self._rows.tensor.shape[1] == t_pad:
            return self._rows.tensor[self._row]
        flat = np.zeros((1, t_pad), dtype=np.float32)
        cat = np.concatenate(self.samples)
        flat[0, :cat.size] = cat
        t = torch.as_tensor(flat, device=dev)
        self._rows, self._row = _DeviceRows(t, np.float64), 0
        self._bounded = 0
        return t[0]


# lattice twiddle plans, keyed on (pairs' bounds, bins, T, n_aux)
_LATTICE_PLANS: dict = {}


#: pair-derived parts of the key, built once per immutable pairs tuple (a
#: per-frame harness passes the same tuple every frame); keyed on identity
_PAIR_KEYS: dict = {}


def _pair_key(pairs):
    """(bounds fp64, pair_m int32, pair_mp int32, key bytes) of ``pairs``."""
    if isinstance(pairs, tuple):
        e = _PAIR_KEYS.get(id(pairs))
        if e is not None and e[0] is pairs:
            return e[1]
    bounds = np.array([p.tdoa_bound for p in pairs], dtype=np.float64)
    pm = np.array([p.index_m for p in pairs], dtype=np.int32)
    pmp = np.array([p.index_m_prime for p in pairs], dtype=np.int32)
    val = (bounds, pm, pmp, bounds.tobytes() + pm.tobytes() + pmp.tobytes())
    if isinstance(pairs, tuple):
        if len(_PAIR_KEYS) >= 16:
            _PAIR_KEYS.clear()
        _PAIR_KEYS[id(pairs)] = (pairs, val)   # holds `pairs`: the id cannot be reused
    return val


def _lattice_plan(pairs, omega, sample_period, n_aux, device):
    bounds, pm, pmp, pkey = _pair_key(pairs)
    key = (pkey, np.asarray(omega).tobytes(),
           float(sample_period), int(n_aux), str(device))
    plan = _LATTICE_PLANS.get(key)
    if plan is None:
        dummy = np.zeros((1, len(pairs)))
        plan = SrpPlan(dummy, pm, pmp, bounds, omega, sample_period=sample_period, n_aux=n_aux,
                       weights="onthefly", device=device, conventional=False)
        if len(_LATTICE_PLANS) > 64:
            _LATTICE_PLANS.clear()
        _LATTICE_PLANS[key] = plan
    return plan


def build_gcc_lattice_frames(crosses, sample_period, n_aux, counter=None, device=None):
    """Batched :func:`build_gcc_lattice`: one K3 launch for all frames."""
    if n_aux < 0 or int(n_aux) != n_aux:
        raise ValueError(f"n_aux must be a non-negative integer, got {n_aux}")
    crosses = list(crosses)
    if not crosses:
        return []
    pairs = crosses[0].pairs
    if not (sample_period > 0 and math.isfinite(sample_period)):
        raise ValueError(f"sample_period must be positive, got {sample_period}")
    # floor(bound / T) per pair (srp.py:123-134) from the cached bounds row
    halves = tuple(np.floor(_pair_key(pairs)[0] / sample_period).astype(np.int64).tolist())
    dev = N.require_cuda(device)
    plan = _lattice_plan(pairs, crosses[0].bin_frequencies, sample_period, int(n_aux), dev)
    psi = _device_psi(crosses, dev)
    xi = plan.lattice(psi)
    rows = _DeviceRows(xi, np.float64)
    total = plan.total_samples
    if counter is not None:
        for _ in crosses:
            counter.add_complex(total * crosses[0].num_bins)
    # PHAT samples are bounded by 2 Kb (Kb of these cross-spectra)
    bounded = crosses[0].num_bins if all(
        getattr(c, "weighting", None) == "phat" for c in crosses) else 0
    return [
        GccLattice(sample_period, n_aux, halves, frame_index=c.frame_index, _rows=rows, _row=i,
                   _plan=plan, _bounded=bounded)
        for i, c in enumerate(crosses)
    ]


def build_gcc_lattice(cross, sample_period: float, n_aux: int, counter=None) -> GccLattice:
    """Sample every pair's GCC on its critical lag lattice (``srp.py:201-247``)."""
    if n_aux < 0 or int(n_aux) != n_aux:
        raise ValueError(f"n_aux must be a non-negative integer, got {n_aux}")
    return build_gcc_lattice_frames([cross], sample_period, n_aux, counter)[0]


class SincTable:
    """Interpolation weights from lattice to candidates (``srp.py:264-284``).

    Holds an :class:`SrpPlan` with the device table ``W [J, T_pad]`` (or the
    on-the-fly sinc split when W does not fit); ``weights`` materialises the
    reference's per-pair (J, T_p) float64 tuple on first access.
    """

    def __init__(self, sample_period, n_aux, half_counts, weights=None, _plan=None):
        self.sample_period = float(sample_period)
        self.n_aux = int(n_aux)
        self.half_counts = tuple(int(h) for h in half_counts)
        self._plan = _plan
        self._weights = None if weights is None else tuple(np.asarray(w, float) for w in weights)

    @property
    def weights(self) -> tuple:
        if self._weights is None:
            plan = self._plan
            if plan.W is not None:
                W = plan.W.cpu().numpy()
            else:  # regenerate the table rows on the device, chunk by chunk
                W = np.empty((plan.J, plan.T_pad), dtype=np.float32)
                for lo in range(0, plan.J, 65536):
                    hi = min(plan.J, lo + 65536)
                    tmp = torch.empty((hi - lo, plan.T_pad), dtype=torch.float32,
                                      device=plan.device)
                    N.call("srpb_sinc_table", N.ptr(plan.sx_i[:, lo:hi].contiguous()),
                           N.ptr(plan.sx_f[:, lo:hi].contiguous()), hi - lo, plan.P,
                           N.ptr(plan.off), N.ptr(plan.reach), plan.T_pad, N.ptr(tmp),
                           N.stream_handle(plan.device))
                    W[lo:hi] = tmp.cpu().numpy()
            off = plan.off_np
            self._weights = tuple(W[:, off[p]:off[p + 1]].astype(float) for p in range(plan.P))
        return self._weights

    @property
    def num_candidates(self) -> int:
        return self._plan.J if self._plan is not None else self._weights[0].shape[0]

    @property
    def num_pairs(self) -> int:
        return len(self.half_counts)

    @property
    def plan(self):
        return self._plan


def precompute_sinc_table(grid, pairs: Sequence, sample_period: float, n_aux: int,
                          weights: str = "auto", device=None) -> SincTable:
    """Per-pair candidate-to-lattice sinc weights (``srp.py:287-317``), built
    on the device.  ``weights="onthefly"`` skips storing W (C4-sized grids)."""
    if n_aux < 0 or int(n_aux) != n_aux:
        raise ValueError(f"n_aux must be a non-negative integer, got {n_aux}")
    table = grid.require_table()
    if table.shape[1] != len(pairs):
        raise ValueError(f"grid table has {table.shape[1]} pair columns, expected {len(pairs)}")
    halves = lattice_half_counts(pairs, sample_period)
    plan = SrpPlan(table,
                   [p.index_m for p in pairs], [p.index_m_prime for p in pairs],
                   [p.tdoa_bound for p in pairs], np.zeros(1), sample_period=sample_period,
                   n_aux=int(n_aux), weights=weights, device=device, conventional=False)
    return SincTable(sample_period, n_aux, halves, _plan=plan)


def _check_lattice_table(lattice, table):
    if lattice.sample_period != table.sample_period:
        raise ValueError(
            f"lattice spacing {lattice.sample_period} != table spacing {table.sample_period}"
        )
    if lattice.n_aux != table.n_aux:
        raise ValueError(f"lattice n_aux {lattice.n_aux} != table n_aux {table.n_aux}")
    if tuple(lattice.half_counts) != tuple(table.half_counts):
        raise ValueError("lattice and table disagree on pair half counts")


def srp_approx_frames(lattices, table, counter=None, maps=True):
    """Batched :func:`srp_approx`: one K4 launch (+ fused argmax) for all
    frames sharing ``table``."""
    lattices = list(lattices)
    for lat in lattices:
        _check_lattice_table(lat, table)
    if not lattices:
        return []
    plan = table.plan
    if plan is None:
        raise ValueError("table was not built by precompute_sinc_table on this device path")
    dev = plan.device
    rows = [getattr(l, "_rows", None) for l in lattices]
    if (rows[0] is not None and all(r is rows[0] for r in rows)
            and rows[0].tensor.shape[1] == plan.T_pad and rows[0].tensor.device == dev):
        idx = [l._row for l in lattices]
        xi = rows[0].tensor
        if idx != list(range(xi.shape[0])):
            xi = xi[torch.as_tensor(idx, device=dev)].contiguous()
    elif len(lattices) == 1:
        xi = lattices[0].device_row(plan.T_pad, dev)[None].contiguous()
    else:
        xi = torch.stack([l.device_row(plan.T_pad, dev) for l in lattices]).contiguous()
    kbs = {getattr(l, "_bounded", 0) for l in lattices}
    bounded = kbs.pop() if len(kbs) == 1 else 0  # one bound for the batch
    out, am = plan.approx(xi, maps=maps, bounded=bounded)
    if counter is not None:
        for _ in lattices:
            counter.add_real(plan.J * plan.total_samples)
    mrows = _DeviceRows(out, np.float64) if out is not None else None
    arows = _DeviceRows(am, np.int64)
    return [SrpMap(None, "approximated", frame_index=l.frame_index, _rows=mrows, _row=i,
                   _argmax=(arows, i), _num=plan.J) for i, l in enumerate(lattices)]


def srp_approx(lattice, table, counter=None) -> SrpMap:
    """Reconstruct the map from lattice samples (``srp.py:320-347``)."""
    _check_lattice_table(lattice, table)
    if getattr(table, "plan", None) is None:  # a reference/host-built table
        raise ValueError("table was not built by precompute_sinc_table on this device path")
    return srp_approx_frames([lattice], table, counter)[0]


# conventional plans, keyed on the TDOA table object (weakly) and bins
_CONV_PLANS: dict = {}


def _conventional_plan(grid, crosses, device):
    table = grid.require_table()
    omega = np.asarray(crosses[0].bin_frequencies, dtype=np.float64)
    pairs = crosses[0].pairs
    key = (id(table), omega.tobytes(), str(device))
    hit = _CONV_PLANS.get(key)
    if hit is not None and hit[0]() is table:
        return hit[1]
    plan = SrpPlan(table, [p.index_m for p in pairs], [p.index_m_prime for p in pairs],
                   [p.tdoa_bound for p in pairs], omega, device=device)
    for k in [k for k, v in _CONV_PLANS.items() if v[0]() is None]:
        del _CONV_PLANS[k]
    _CONV_PLANS[key] = (weakref.ref(table), plan)
    return plan


def srp_conventional_frames(frames, grid, counter=None, maps=True) -> list:
    """Exact SRP maps for several frames (``srp.py:391-429``): one K2 launch
    with fused argmax."""
    frames = list(frames)
    if not frames:
        return []
    table = grid.require_table()
    n_pairs = table.shape[1]
    omega = np.asarray(frames[0].bin_frequencies, dtype=float)
    for fr in frames:
        if fr.num_pairs != n_pairs:
            raise ValueError(f"frame has {fr.num_pairs} pairs, grid table has {n_pairs}")
        fo = np.asarray(fr.bin_frequencies, dtype=float)
        if fo.shape != omega.shape or np.any(fo != omega):
            raise ValueError("all frames must share the same bin frequencies")
    dev = N.require_cuda()
    plan = _conventional_plan(grid, frames, dev)
    psi = _device_psi(frames, dev)
    bounded = all(getattr(fr, "weighting", None) == "phat" for fr in frames)
    out, am = plan.conventional(psi, maps=maps, _bounded=bounded)
    if counter is not None:
        for _ in range(n_pairs):
            counter.add_complex(table.shape[0] * omega.size * len(frames))
    mrows = _DeviceRows(out, np.float64) if out is not None else None
    arows = _DeviceRows(am, np.int64)
    return [SrpMap(None, "conventional", frame_index=fr.frame_index, _rows=mrows, _row=i,
                   _argmax=(arows, i), _num=plan.J) for i, fr in enumerate(frames)]


def srp_conventional(cross, grid, counter=None) -> SrpMap:
    """Exact SRP map of one frame (``srp.py:376-388``)."""
    return srp_conventional_frames([cross], grid, counter=counter)[0]


class _IndexPair:
    """Pair indices only: what the cross matrix of ``srp_oracle`` needs."""

    __slots__ = ("index_m", "index_m_prime")

    def __init__(self, m, mp):
        self.index_m, self.index_m_prime = m, mp


def _full_pair_count(n_pairs):
    m = int(round((1.0 + math.sqrt(1.0 + 8.0 * n_pairs)) / 2.0))
    if m * (m - 1) // 2 != n_pairs:
        raise ValueError(f"{n_pairs} pair rows do not form a full pair set")
    return m


def srp_oracle_frames(frames, grid, weighting="phat", phat_floor=None) -> list:
    """Batched :func:`srp_oracle`: one ``srpb_srp_quadform`` launch (fp64).

    Scope of the check: the quadratic form, steering vectors and sums run in
    fp64 with direct exponentials, independently of K2's phase generator and
    tensor-core contraction; given spectral frames, the weighted cross
    matrix comes from K1 (complex64 psi), so this cross-check covers K2
    onward, not K1 (K1 is pinned to the reference's golden vectors in
    tests/test_parity_gpu.py)."""
    frames = list(frames)
    if not frames:
        return []
    table = grid.require_table()
    dev = N.require_cuda()
    if all(hasattr(fr, "pairs") for fr in frames):  # CrossSpectra (srp.py:484-487)
        crosses = frames
        m = _full_pair_count(len(crosses[0].pairs))
    else:  # spectral frames: the pair rows of the weighted cross matrix (:488-491)
        from .spectral import cross_spectrum_frames
        m = int(getattr(frames[0], "num_channels", 0) or np.shape(frames[0].spectra)[0])
        pairs = [_IndexPair(b, a) for a in range(m) for b in range(a + 1, m)]
        crosses = cross_spectrum_frames(frames, pairs, weighting, phat_floor, device=dev)
    if table.shape[1] != m * (m - 1) // 2:
        raise ValueError(
            f"grid table has {table.shape[1]} pair columns, expected "
            f"{m * (m - 1) // 2} for {m} channels"
        )
    omega = np.asarray(crosses[0].bin_frequencies, dtype=np.float64)
    for cr in crosses:
        if len(cr.pairs) != len(crosses[0].pairs) or np.any(
                np.asarray(cr.bin_frequencies, dtype=np.float64) != omega):
            raise ValueError("all frames must share the same pairs and bin frequencies")
    pm = torch.as_tensor([p.index_m for p in crosses[0].pairs], dtype=torch.int32, device=dev)
    pmp = torch.as_tensor([p.index_m_prime for p in crosses[0].pairs], dtype=torch.int32,
                          device=dev)
    # delays of each mic relative to mic 0: canonical columns 0 .. M-2 (:495-498)
    tau_rel = np.concatenate([np.zeros((table.shape[0], 1)), table[:, : m - 1]], axis=1)
    maps = quadform_maps(_device_psi(crosses, dev), omega, torch.as_tensor(
        np.ascontiguousarray(tau_rel), device=dev), pm, pmp)
    rows = _DeviceRows(maps, np.float64)
    return [SrpMap(None, "oracle", frame_index=getattr(fr, "frame_index", 0), _rows=rows, _row=i)
            for i, fr in enumerate(frames)]


def srp_oracle(data, grid, weighting="phat", phat_floor=None, candidate_chunk=256) -> SrpMap:
    """Quadratic-form SRP map, trace removed (``srp.py:468-515``), in fp64 on
    the device.  Accepts a spectral frame or pair cross-spectra, like the
    reference; ``candidate_chunk`` is accepted for signature parity (the
    kernel tiles candidates itself)."""
    return srp_oracle_frames([data], grid, weighting, phat_floor)[0]


def quadform_maps(psi, omega, tau_rel, pair_m, pair_mp) -> torch.Tensor:
    """``srpb_srp_quadform``: psi [F, P, Kb] complex64, tau_rel [J, M] fp64
    (device) -> maps [F, J] fp64."""
    dev = psi.device
    psi, tau_rel = psi.contiguous(), tau_rel.contiguous()
    F, P, Kb = psi.shape
    J, M = tau_rel.shape
    om = torch.as_tensor(np.ascontiguousarray(omega, dtype=np.float64), device=dev)
    maps = torch.empty((F, J), dtype=torch.float64, device=dev)
    N.call("srpb_srp_quadform", N.ptr(psi), F, P, Kb, N.ptr(om), N.ptr(tau_rel), J, M, N.ptr(pair_m), N.ptr(pair_mp), N.ptr(maps),
           N.stream_handle(dev))
    return maps


@dataclass(frozen=True)
class ComplexityReport:
    """Closed-form counts of both paths (``srp.py:518-570``)."""

    num_candidates: int
    num_pairs: int
    num_bins: int
    n_aux: int
    sample_period: float
    half_counts: tuple
    total_samples: int
    avg_samples_per_pair: float
    mults_conventional: int
    mults_sampling: int
    mults_interpolation: int
    ratio_sampling: float
    ratio_interpolation: float
    ratio_total: float
    measured_conventional: int | None = None
    measured_sampling: int | None = None
    measured_interpolation: int | None = None
    measured_frames: int | None = None

    def as_dict(self) -> dict:
        d = dict(self.__dict__)
        d["half_counts"] = list(self.half_counts)
        return d


def complexity_report(num_candidates, num_bins, pairs, sample_period, n_aux,
                      measured_conventional=None, measured_sampling=None,
                      measured_interpolation=None, measured_frames=None) -> ComplexityReport:
    """Per-frame closed forms (``srp.py:573-619``)."""
    if num_candidates < 1 or num_bins < 1:
        raise ValueError("need at least one candidate and one bin")
    halves = lattice_half_counts(pairs, sample_period)
    n_pairs = len(halves)
    total = sum(2 * (h + int(n_aux)) + 1 for h in halves)
    avg = 2.0 / n_pairs * sum(halves) + 2.0 * n_aux + 1.0
    return ComplexityReport(
        num_candidates=num_candidates, num_pairs=n_pairs, num_bins=num_bins, n_aux=int(n_aux),
        sample_period=float(sample_period), half_counts=halves, total_samples=total,
        avg_samples_per_pair=avg, mults_conventional=num_candidates * n_pairs * num_bins,
        mults_sampling=total * num_bins, mults_interpolation=total * num_candidates,
        ratio_sampling=avg / num_candidates, ratio_interpolation=avg / num_bins,
        ratio_total=avg / num_candidates + avg / num_bins,
        measured_conventional=measured_conventional, measured_sampling=measured_sampling,
        measured_interpolation=measured_interpolation, measured_frames=measured_frames,
    )
