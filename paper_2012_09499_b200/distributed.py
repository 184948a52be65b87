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


def round_widths(per_rank: int, rounds: int = 4, tile: int = 160):
    """Per-rank frame widths of the rounds of :class:`ShardedRunner`: whole
    tensor-core frame tiles (``tile`` frames) per round where the frames
    allow, the leftover frames in the first round and the extra tiles in the
    earliest rounds -- the last round's gather is the only one no compute
    hides, so it is the smallest."""
    per_rank, rounds = int(per_rank), max(1, int(rounds))
    if per_rank <= 0:
        return []
    tiles, rem = divmod(per_rank, tile)
    if tiles == 0:
        return [per_rank]
    rounds = min(rounds, tiles)
    base, extra = divmod(tiles, rounds)
    widths = [(base + (1 if c < extra else 0)) * tile for c in range(rounds)]
    widths[0] += rem
    return widths


class ShardedRunner:
    """Strong-scaling frame split whose result gathers hide under compute.

    The F frames are cut into rounds; round c covers the global frames
    ``[W*s_c, W*(s_c + w_c))`` (W ranks, per-rank width ``w_c``, ``s_c`` the
    widths before it) and rank r runs the r-th ``w_c``-frame block of it as
    one graph-captured step (``SrpPlan.capture``).  An all-gather of a
    round's per-rank blocks therefore lands in frame order in the static
    ``[F, J]`` / ``[F]`` outputs with no padding, concatenation or copy, and
    it is issued asynchronously (the collective's own stream, NCCL over
    NVLink) right after the round's replay, so it runs while the next round
    computes; only the last -- smallest -- round's gather is exposed.
    ``F % W`` leftover frames run as a one-frame tail on the first ranks and
    travel through the padded :func:`gather_frames`.

    The reference's only parallelism is a process pool over scenes
    (``experiment.py:631-641``); this is its replacement for one long batch.
    """

    def __init__(self, plan, F, M=None, path="approx", maps=True, rounds=4, tile=160,
                 group=None):
        self.plan, self.F, self.path, self.want_maps, self.group = plan, int(F), path, maps, group
        on = self._dist = dist.is_initialized()
        self.world = dist.get_world_size(group) if on else 1
        self.rank = dist.get_rank(group) if on else 0
        W, r = self.world, self.rank
        base = self.F // W
        self.tail = self.F - base * W          # < W leftover frames
        #: (global first frame of the round, per-rank width)
        self.rounds, s = [], 0
        for w in round_widths(base, rounds, tile):
            self.rounds.append((W * s, w))
            s += w
        #: this rank's global [lo, hi) frame range per round
        self.mine = [(g0 + r * w, g0 + (r + 1) * w) for g0, w in self.rounds]
        self.tail_frame = base * W + r if r < self.tail else None
        kw = {} if M is None else {"M": M}
        self.steps = [plan.capture(w, path=path, maps=maps, **kw) for _, w in self.rounds]
        self.tail_step = plan.capture(1, path=path, maps=maps, **kw) if self.tail else None
        ref = self.steps[0] if self.steps else self.tail_step
        dev = ref.argmax.device
        #: kernels launched by one ``run`` on this rank
        self.launches = sum(getattr(st, "launches", 0) for st in self.steps) + \
            (getattr(self.tail_step, "launches", 0) if self.tail_frame is not None else 0)
        self.argmax = torch.empty((self.F,), dtype=ref.argmax.dtype, device=dev)
        self.maps = (torch.empty((self.F, ref.maps.shape[1]), dtype=ref.maps.dtype, device=dev)
                     if maps else None)

    @property
    def local_frames(self):
        """Global frame indices this rank computes, in its processing order."""
        idx = [torch.arange(lo, hi) for lo, hi in self.mine]
        if self.tail_frame is not None:
            idx.append(torch.tensor([self.tail_frame]))
        return torch.cat(idx) if idx else torch.empty(0, dtype=torch.int64)

    def load(self, Y_all):
        """Copy this rank's frames of ``Y_all`` [F, M, Kb] (host, pinned for an
        asynchronous copy, or device) into the rounds' static inputs."""
        for st, (lo, hi) in zip(self.steps, self.mine):
            st.Y.copy_(Y_all[lo:hi], non_blocking=True)
        if self.tail_frame is not None:
            self.tail_step.Y.copy_(Y_all[self.tail_frame:self.tail_frame + 1], non_blocking=True)

    def run(self):
        """One step over the loaded frames -> (maps [F, J] | None, argmax
        [F]) of ALL frames on every rank, valid on the current stream."""
        W, works = self.world, []
        for st, (g0, w) in zip(self.steps, self.rounds):
            m, am = st.replay()
            if not self._dist:   # one process, no group: plain copies
                self.argmax[g0:g0 + w].copy_(am)
                if self.want_maps:
                    self.maps[g0:g0 + w].copy_(m)
                continue
            works.append(dist.all_gather_into_tensor(self.argmax[g0:g0 + W * w], am,
                                                     group=self.group, async_op=True))
            if self.want_maps:
                works.append(dist.all_gather_into_tensor(self.maps[g0:g0 + W * w], m,
                                                         group=self.group, async_op=True))
        for wk in works:      # the current stream waits for the gathers
            wk.wait()
        if self.tail:
            t0 = self.F - self.tail
            if self.tail_frame is not None:
                m, am = self.tail_step.replay()
            else:             # nothing to run: contributes padding only
                m = self.maps[:0] if self.want_maps else None
                am = self.argmax[:0]
            self.argmax[t0:].copy_(_gather_tail(am, self.tail, W, self.group))
            if self.want_maps:
                self.maps[t0:].copy_(_gather_tail(m, self.tail, W, self.group))
        return self.maps, self.argmax


def _gather_tail(local, tail, world, group=None):
    """Ranks ``< tail`` hold one row each, the others none: all-gather the
    padded rows and keep the first ``tail``."""
    pad = torch.zeros((1,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return out[:tail]
