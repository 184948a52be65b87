"""Multi-GPU execution of the SRP hot path: one process per GPU.

Frames are independent units (map f depends only on Psi_f: ``srp.py:419-422``,
``srp.py:340-343``), so a batch shards into contiguous frame ranges with the
geometry, TDOA split and sinc table replicated per rank -- no collective on
the data path.  The only exchange is collecting results: per-frame maps
``[F_local, J]`` and argmaxes ``[F_local]`` gathered with NCCL all-gather
over NVLink (``torch.distributed``, backend ``nccl``; ``gloo`` on CPU for
tests).  Batch-1 (C5) cannot shard frames; it shards candidates instead and
reduces the packed argmax keys with an all-reduce MAX.

Packed keys (``common.cuh``) are unsigned: ``orderable(value) << 32 |
(0xFFFFFFFF - j)``.  torch has no uint64 reduction, so keys travel as int64
with the top bit flipped, which maps unsigned order onto signed order.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

_TOP = -(1 << 63)  # int64 with only the sign bit set


def frame_ranges(num_frames: int, world: int):
    """Contiguous, balanced [lo, hi) frame range per rank (first ranks get
    the extra frame when F % world != 0)."""
    base, extra = divmod(int(num_frames), int(world))
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def candidate_ranges(num_candidates: int, world: int, align: int = 128):
    """Contiguous candidate ranges aligned to the 128-candidate kernel tile."""
    tiles = (int(num_candidates) + align - 1) // align
    out = []
    for lo_t, hi_t in frame_ranges(tiles, world):
        out.append((min(lo_t * align, num_candidates), min(hi_t * align, num_candidates)))
    return out


def gather_frames(local: torch.Tensor, num_frames: int, group=None) -> torch.Tensor:
    """All-gather per-rank frame blocks ``[F_r, ...]`` into ``[F, ...]`` in
    rank order (uneven blocks are padded to the largest, then trimmed)."""
    world = dist.get_world_size(group)
    ranges = frame_ranges(num_frames, world)
    width = max(hi - lo for lo, hi in ranges)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * width,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = [out[r * width: r * width + (hi - lo)] for r, (lo, hi) in enumerate(ranges)]
    return torch.cat(parts, dim=0)


def keys_to_signed(keys_u: torch.Tensor) -> torch.Tensor:
    """uint64 packed keys (stored in int64 tensors) -> order-preserving int64."""
    return keys_u ^ _TOP


def keys_from_signed(keys_s: torch.Tensor) -> torch.Tensor:
    return keys_s ^ _TOP


def rebase_keys(keys_u: torch.Tensor, j_offset: int) -> torch.Tensor:
    """Re-express keys computed over a candidate slice in global indices:
    low word ``0xFFFFFFFF - j_local`` becomes ``0xFFFFFFFF - (j_local + j0)``."""
    if j_offset == 0:
        return keys_u
    empty = keys_u == 0
    out = keys_u - int(j_offset)  # low word decreases by j0 (no borrow: j_local + j0 < 2^32)
    return torch.where(empty, keys_u, out)


def allreduce_argmax(keys_u: torch.Tensor, group=None) -> torch.Tensor:
    """MAX all-reduce of packed keys across ranks (candidate sharding):
    largest value wins, lowest global index on ties."""
    s = keys_to_signed(keys_u.clone())
    dist.all_reduce(s, op=dist.ReduceOp.MAX, group=group)
    return keys_from_signed(s)


def keys_index(keys_u: torch.Tensor) -> torch.Tensor:
    """Candidate index held by packed keys (host-side mirror of
    ``srpb_keys_to_index``)."""
    return (0xFFFFFFFF - (keys_u & 0xFFFFFFFF)).to(torch.int64)


def run_frame_sharded(plan, Y_all, path="approx", maps=True, gather=True, group=None):
    """Run ``plan`` on this rank's frame range of ``Y_all`` [F, M, Kb] and
    optionally gather maps/argmax from all ranks (NCCL all-gather)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    F = Y_all.shape[0]
    lo, hi = frame_ranges(F, world)[rank]
    m, am = plan.run(Y_all[lo:hi].contiguous(), path, maps=maps)
    if not gather or world == 1:
        return m, am
    am_all = gather_frames(am.to(torch.int64), F, group).to(torch.int32)
    m_all = gather_frames(m, F, group) if m is not None else None
    return m_all, am_all
