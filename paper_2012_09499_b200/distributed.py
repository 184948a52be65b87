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


def keys_from_maps(maps: torch.Tensor, argmax: torch.Tensor, j_offset: int = 0) -> torch.Tensor:
    """Packed keys (``common.cuh`` make_key) of each frame's maximum, from
    fp32 maps [F, J_r] and their argmax [F] over a candidate slice starting
    at global index ``j_offset`` (uint64 bits in an int64 tensor)."""
    v = maps.gather(1, argmax.to(torch.int64)[:, None])[:, 0].float() + 0.0  # -0 -> +0
    b = v.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    neg = (b & 0x80000000) != 0
    ordered = torch.where(neg, (~b) & 0xFFFFFFFF, b | 0x80000000)
    j = argmax.to(torch.int64) + int(j_offset)
    return (ordered << 32) | (0xFFFFFFFF - j)


def gather_candidates(local: torch.Tensor, num_candidates: int, align: int = 128,
                      group=None) -> torch.Tensor:
    """All-gather per-rank candidate blocks ``[F, J_r]`` into ``[F, J]``
    (ranges from :func:`candidate_ranges`; uneven blocks padded, trimmed)."""
    world = dist.get_world_size(group)
    ranges = candidate_ranges(num_candidates, world, align)
    width = max(max(hi - lo for lo, hi in ranges), 1)
    F = local.shape[0]
    pad = torch.zeros((width, F), dtype=local.dtype, device=local.device)
    pad[: local.shape[1]] = local.t()
    out = torch.empty((world * width, F), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = [out[r * width: r * width + (hi - lo)] for r, (lo, hi) in enumerate(ranges)]
    return torch.cat(parts, dim=0).t().contiguous()


def run_candidate_sharded(plan_local, Y, j_offset, num_candidates, path="approx", maps=True,
                          align=128, group=None):
    """Batch-1 / small-batch sharding: ``plan_local`` covers
    this rank's candidate range ``[j_offset, j_offset + plan_local.J)`` of
    :func:`candidate_ranges`; every rank runs all frames of ``Y``.  The
    global argmax is one all-reduce MAX of the packed keys (largest value,
    then lowest global index -- deterministic); maps are all-gathered only
    when requested.  Returns (maps [F, J] or None, argmax [F] int32)."""
    m, am = plan_local.run(Y, path, maps=True)
    keys = keys_from_maps(m, am, j_offset)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        keys = allreduce_argmax(keys, group)
        m = gather_candidates(m, num_candidates, align, group) if maps else None
    elif not maps:
        m = None
    return m, keys_index(keys).to(torch.int32)


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
    return gather_results(m, am, F, group)


def gather_results(maps_local, argmax_local, num_frames, group=None):
    """All-gather one rank's frame-block results: per-frame maps
    ``[F_r, J]`` (or None) and argmax ``[F_r]`` -> (maps [F, J] | None,
    argmax [F] int32) on every rank, in frame order (NCCL over NVLink on the
    GPU; the bench's multi-GPU step ends with this call)."""
    am_all = gather_frames(argmax_local.to(torch.int64), num_frames, group).to(torch.int32)
    m_all = gather_frames(maps_local, num_frames, group) if maps_local is not None else None
    return m_all, am_all
