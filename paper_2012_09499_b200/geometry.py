"""Host-side geometry constants feeding the hot path.

Mirrors the reference's geometry API (``pkg/src/srpfast/geometry.py``) so
callers can build pair tables and TDOA tables without the reference
installed: canonical pair order (``:141-176``), pair bounds ``d / c``
(``:165-174``), near/far-field TDOA tables with the bound assertion
(``:365-398``).  These are signal-independent constants computed once per
geometry; the SRP kernels consume them through :class:`~.plan.SrpPlan`.
Reference objects (``srpfast.geometry.MicPair`` etc.) are accepted anywhere
these are, by duck typing.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

UNIT_NORM_TOL = 1e-12     # geometry.py:34-35
TDOA_BOUND_SLACK = 1e-12  # geometry.py:37-38


@dataclass(frozen=True)
class MicPair:
    """Unordered pair ``(m, m')`` with ``m > m'`` (``geometry.py:41-70``)."""

    index_m: int
    index_m_prime: int
    distance: float
    tdoa_bound: float

    def __post_init__(self) -> None:
        if self.index_m <= self.index_m_prime:
            raise ValueError(
                f"pair indices must satisfy m > m', got ({self.index_m}, {self.index_m_prime})"
            )
        if not (self.distance > 0.0 and math.isfinite(self.distance)):
            raise ValueError(f"pair distance must be positive, got {self.distance}")
        if not (self.tdoa_bound > 0.0 and math.isfinite(self.tdoa_bound)):
            raise ValueError(f"tdoa bound must be positive, got {self.tdoa_bound}")


def enumerate_pairs(positions, speed_of_sound: float = 340.0) -> tuple:
    """Canonical order: lexicographic in ``(m', m)``, ``m' < m``."""
    if isinstance(positions, MicArray):
        return positions.pairs
    pos = np.asarray(positions, dtype=float)
    out = []
    for mp in range(pos.shape[0]):
        for m in range(mp + 1, pos.shape[0]):
            d = float(np.linalg.norm(pos[m] - pos[mp]))
            if d == 0.0:
                raise ValueError(f"microphones {mp} and {m} are coincident")
            out.append(MicPair(m, mp, d, d / speed_of_sound))
    return tuple(out)


class MicArray:
    """Immutable microphone positions + speed of sound (``geometry.py:73-138``)."""

    def __init__(self, positions, speed_of_sound: float = 340.0):
        pos = np.array(positions, dtype=float)
        if pos.ndim != 2 or pos.shape[1] != 3:
            raise ValueError(f"positions must have shape (M, 3), got {pos.shape}")
        if pos.shape[0] < 2:
            raise ValueError("an array needs at least 2 microphones")
        if not np.all(np.isfinite(pos)):
            raise ValueError("positions must be finite")
        if not (speed_of_sound > 0.0 and math.isfinite(speed_of_sound)):
            raise ValueError(f"speed of sound must be positive, got {speed_of_sound}")
        pos.setflags(write=False)
        self._positions = pos
        self._c = float(speed_of_sound)
        self._pairs = enumerate_pairs(pos, self._c)

    positions = property(lambda self: self._positions)
    speed_of_sound = property(lambda self: self._c)
    pairs = property(lambda self: self._pairs)
    num_mics = property(lambda self: self._positions.shape[0])
    num_pairs = property(lambda self: len(self._pairs))
    center = property(lambda self: self._positions.mean(axis=0))
    diameter = property(lambda self: max(p.distance for p in self._pairs))


def circular_array(num_mics, radius, center=(0.0, 0.0, 0.0), speed_of_sound=340.0,
                   start_angle=0.0) -> MicArray:
    """Uniform circular array in a z = const plane (``geometry.py:179-204``)."""
    if num_mics < 2:
        raise ValueError("need at least 2 microphones")
    if not radius > 0.0:
        raise ValueError(f"radius must be positive, got {radius}")
    c = np.asarray(center, dtype=float)
    ang = start_angle + 2.0 * np.pi * np.arange(num_mics) / num_mics
    pos = np.stack([c[0] + radius * np.cos(ang), c[1] + radius * np.sin(ang),
                    np.full(num_mics, c[2])], axis=1)
    return MicArray(pos, speed_of_sound=speed_of_sound)


def tdoa_nearfield(array, pair, point) -> float:
    q = np.asarray(point, dtype=float)
    if q.shape != (3,):
        raise ValueError(f"point must have shape (3,), got {q.shape}")
    pos = array.positions
    return (float(np.linalg.norm(pos[pair.index_m] - q))
            - float(np.linalg.norm(pos[pair.index_m_prime] - q))) / array.speed_of_sound


def tdoa_farfield(array, pair, direction) -> float:
    r = np.asarray(direction, dtype=float)
    if r.shape != (3,):
        raise ValueError(f"direction must have shape (3,), got {r.shape}")
    nrm = float(np.linalg.norm(r))
    if abs(nrm - 1.0) > UNIT_NORM_TOL:
        raise ValueError(f"direction must be unit length, |r| = {nrm!r}")
    pos = array.positions
    return float((pos[pair.index_m] - pos[pair.index_m_prime]) @ r) / array.speed_of_sound


@dataclass(frozen=True, eq=False)
class CandidateGrid:
    """Candidate positions/directions + optional (J, P) TDOA table
    (``geometry.py:239-303``)."""

    mode: str
    entries: np.ndarray
    angles_deg: np.ndarray | None = None
    tdoa_table: np.ndarray | None = None

    def __post_init__(self) -> None:
        if self.mode not in ("far_field", "near_field"):
            raise ValueError(f"unknown grid mode {self.mode!r}")
        e = np.array(self.entries, dtype=float)
        if e.ndim != 2 or e.shape[1] != 3 or e.shape[0] == 0:
            raise ValueError(f"entries must have shape (J, 3), got {e.shape}")
        if not np.all(np.isfinite(e)):
            raise ValueError("grid entries must be finite")
        if self.mode == "far_field":
            worst = float(np.max(np.abs(np.linalg.norm(e, axis=1) - 1.0)))
            if worst > UNIT_NORM_TOL:
                raise ValueError(f"far-field entries must be unit vectors (worst |r|-1 = {worst:g})")
        e.setflags(write=False)
        object.__setattr__(self, "entries", e)
        if self.angles_deg is not None:
            a = np.array(self.angles_deg, dtype=float)
            if a.shape != (e.shape[0], 2):
                raise ValueError(f"angles_deg must have shape (J, 2), got {a.shape}")
            a.setflags(write=False)
            object.__setattr__(self, "angles_deg", a)
        if self.tdoa_table is not None:
            t = np.array(self.tdoa_table, dtype=float)
            if t.ndim != 2 or t.shape[0] != e.shape[0]:
                raise ValueError(f"tdoa_table must have shape (J, P), got {t.shape}")
            t.setflags(write=False)
            object.__setattr__(self, "tdoa_table", t)

    @property
    def num_candidates(self) -> int:
        return self.entries.shape[0]

    def require_table(self) -> np.ndarray:
        if self.tdoa_table is None:
            raise ValueError("grid has no TDOA table; call build_tdoa_table first")
        return self.tdoa_table


def build_tdoa_table(array, grid, chunk: int = 65536):
    """Per-candidate, per-pair TDOAs (``geometry.py:365-398``), candidate
    chunks bound the (chunk, M) distance temporary at C3/C4 sizes."""
    pos = array.positions
    c = array.speed_of_sound
    pairs = array.pairs
    pm = np.array([p.index_m for p in pairs])
    pmp = np.array([p.index_m_prime for p in pairs])
    e = grid.entries
    table = np.empty((e.shape[0], len(pairs)))
    for lo in range(0, e.shape[0], chunk):
        q = e[lo:lo + chunk]
        if grid.mode == "far_field":
            diff = pos[pm] - pos[pmp]                    # (P, 3)
            table[lo:lo + chunk] = (q @ diff.T) / c
        else:
            dist = np.linalg.norm(q[:, None, :] - pos[None, :, :], axis=2)
            table[lo:lo + chunk] = (dist[:, pm] - dist[:, pmp]) / c
    bounds = np.array([p.tdoa_bound for p in pairs])
    if np.any(np.abs(table) > bounds[None, :] + TDOA_BOUND_SLACK):
        raise AssertionError("TDOA magnitude exceeded its physical bound")
    return CandidateGrid(mode=grid.mode, entries=grid.entries, angles_deg=grid.angles_deg,
                         tdoa_table=table)
