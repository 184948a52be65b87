"""Multi-process (world_size 2, gloo, CPU) tests of the sharding/gather logic
used by the multi-GPU path (paper_2012_09499_b200/distributed.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2012_09499_b200 import distributed as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def orderable(v):
    b = np.array([v + 0.0], dtype=np.float32).view(np.uint32)[0]
    return int(~b & 0xFFFFFFFF) if b & 0x80000000 else int(b | 0x80000000)


def make_key(v, j):
    """Python mirror of common.cuh make_key (uint64 bits in an int64)."""
    u = (orderable(v) << 32) | (0xFFFFFFFF - j)
    return u - (1 << 64) if u >= (1 << 63) else u


def _worker(rank, world, port, F, J, maps_all, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # frame sharding: each rank "computes" its frame block, then gathers
        lo, hi = D.frame_ranges(F, world)[rank]
        local = torch.from_numpy(maps_all[lo:hi].copy())
        full = D.gather_frames(local, F)
        ok_frames = torch.equal(full, torch.from_numpy(maps_all))
        am_local = torch.from_numpy(np.argmax(maps_all[lo:hi], axis=1).astype(np.int64))
        am_full = D.gather_frames(am_local, F)
        ok_am = torch.equal(am_full, torch.from_numpy(np.argmax(maps_all, axis=1)))
        # candidate sharding (batch-1): per-rank keys over a candidate slice,
        # rebased to global indices and MAX-reduced
        jlo, jhi = D.candidate_ranges(J, world, align=8)[rank]
        keys = []
        for f in range(F):
            row = maps_all[f, jlo:jhi]
            best = 0
            for jl, v in enumerate(row):
                k = make_key(float(v), jl)
                best = k if (best == 0 or (k ^ D._TOP) > (best ^ D._TOP)) else best
            keys.append(best)
        kt = D.rebase_keys(torch.tensor(keys, dtype=torch.int64), jlo)
        red = D.allreduce_argmax(kt)
        idx = D.keys_index(red)
        ok_cand = torch.equal(idx, torch.from_numpy(np.argmax(maps_all, axis=1)))
        # the torch key builder used by run_candidate_sharded agrees
        sl = torch.from_numpy(maps_all[:, jlo:jhi].copy())
        am_l = torch.from_numpy(np.argmax(maps_all[:, jlo:jhi], axis=1))
        k2 = D.keys_from_maps(sl, am_l, jlo)
        ok_keys = torch.equal(k2, kt)
        idx2 = D.keys_index(D.allreduce_argmax(k2))
        ok_cand = ok_cand and torch.equal(idx2, idx)
        # candidate-block gather reassembles the full maps
        ok_gather = torch.equal(D.gather_candidates(sl, J, align=8), torch.from_numpy(maps_all))
        ret[rank] = (ok_frames, ok_am, ok_cand and ok_keys and ok_gather)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("F", [7, 16])
def test_two_rank_gather_and_candidate_argmax(F):
    rng = np.random.default_rng(F)
    J = 37
    maps_all = rng.standard_normal((F, J)).astype(np.float32)
    maps_all[0, 5] = maps_all[0, 30] = 9.0   # exact tie across ranks: lowest j wins
    maps_all[1, :] = 0.0                       # all-equal frame -> index 0
    maps_all[2, :] = -1.0                      # negative maximum, ties everywhere
    maps_all[2, 20] = -0.5
    mgr = mp.Manager()
    ret = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, F, J, maps_all, ret), nprocs=2, join=True)
    assert dict(ret) == {0: (True, True, True), 1: (True, True, True)}


def test_ranges_cover_and_balance():
    for F in (1, 2, 5, 311, 4096):
        for w in (1, 2, 3, 8):
            r = D.frame_ranges(F, w)
            assert r[0][0] == 0 and r[-1][1] == F
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [hi - lo for lo, hi in r]
            assert max(sizes) - min(sizes) <= 1
    c = D.candidate_ranges(200000, 8)
    assert c[0][0] == 0 and c[-1][1] == 200000
    assert all(lo % 128 == 0 for lo, _ in c)


class _StubPlan:
    """Stands in for SrpPlan on CPU: a deterministic per-frame map (frame
    index and spectra dependent, so a misplaced frame shows) and its argmax."""

    J = 23

    def run(self, Y, path="approx", maps=True):
        F = Y.shape[0]
        base = Y.real.sum(dim=(1, 2)).to(torch.float32)[:, None]
        j = torch.arange(self.J, dtype=torch.float32)[None, :]
        m = torch.sin(base * 0.37 + j * 0.11) + (0.0 if path == "approx" else 1.0)
        return (m if maps else None), torch.argmax(m, dim=1).to(torch.int32)


def _sharded_worker(rank, world, port, Y, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = _StubPlan()
        ref_m, ref_a = plan.run(Y, "approx")
        ok = []
        for maps in (True, False):
            m, a = D.run_frame_sharded(plan, Y, "approx", maps=maps)
            ok.append(torch.equal(a, ref_a) and (torch.equal(m, ref_m) if maps else m is None))
        # without gathering each rank holds only its own frame block
        lo, hi = D.frame_ranges(Y.shape[0], world)[rank]
        m, a = D.run_frame_sharded(plan, Y, "conventional", gather=False)
        ok.append(m.shape[0] == hi - lo and torch.equal(a, plan.run(Y[lo:hi], "conventional")[1]))
        ret[rank] = all(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("F", [5, 64])
def test_run_frame_sharded_two_ranks_end_to_end(F):
    """run_frame_sharded on 2 gloo ranks: each rank runs its contiguous frame
    range through the plan and the all-gather returns every frame's map and
    argmax in frame order -- identical to one process running all frames
    (the bench's strong-scaling C4 step on N GPUs)."""
    g = torch.Generator().manual_seed(F)
    Y = torch.complex(torch.randn((F, 4, 8), generator=g), torch.randn((F, 4, 8), generator=g))
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_sharded_worker, args=(2, _free_port(), Y, ret), nprocs=2, join=True)
    assert dict(ret) == {0: True, 1: True}


class _StubStep:
    """CPU stand-in for CapturedStep: static input ``Y``, ``replay()``."""

    def __init__(self, plan, F, M, path, maps):
        self.plan, self.path, self.want = plan, path, maps
        self.Y = torch.zeros((F, M, 8), dtype=torch.complex64)
        self.maps, self.argmax = plan.run(self.Y, path, maps)

    def replay(self):
        m, a = self.plan.run(self.Y, self.path, self.want)
        if self.want:
            self.maps.copy_(m)
        self.argmax.copy_(a)
        return self.maps, self.argmax


class _StubCapturePlan(_StubPlan):
    M = 4

    def capture(self, F, M=None, path="approx", maps=True):
        return _StubStep(self, F, M if M is not None else self.M, path, maps)


def test_round_widths():
    assert D.round_widths(512, 4) == [192, 160, 160]
    assert D.round_widths(2048, 4) == [608, 480, 480, 480]
    assert D.round_widths(1024, 4) == [384, 320, 160, 160]
    assert D.round_widths(4096, 1) == [4096]
    assert D.round_widths(100, 4) == [100]
    assert D.round_widths(0, 4) == []
    for n in (1, 159, 160, 161, 777, 4096):
        for r in (1, 2, 3, 8):
            w = D.round_widths(n, r)
            assert sum(w) == n and all(x > 0 for x in w) and w == sorted(w, reverse=True)


def _runner_worker(rank, world, port, Y, rounds, tile, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = _StubCapturePlan()
        ok = []
        for path, maps in (("approx", True), ("conventional", True), ("approx", False)):
            ref_m, ref_a = plan.run(Y, path)
            rn = D.ShardedRunner(plan, Y.shape[0], path=path, maps=maps, rounds=rounds, tile=tile)
            rn.load(Y)
            for _ in range(2):   # static outputs are reusable
                m, a = rn.run()
                ok.append(torch.equal(a, ref_a))
                ok.append(torch.equal(m, ref_m) if maps else m is None)
            mine = rn.local_frames
            ok.append(len(mine) in (Y.shape[0] // world, Y.shape[0] // world + 1))
        # every frame is computed by exactly one rank
        got = [None] * world
        dist.all_gather_object(got, mine.tolist())
        ok.append(sorted(sum(got, [])) == list(range(Y.shape[0])))
        ret[rank] = all(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("F,rounds,tile", [(64, 4, 8), (37, 3, 4), (5, 4, 160), (1, 2, 160)])
def test_sharded_runner_two_ranks(F, rounds, tile):
    """ShardedRunner on 2 gloo ranks (rounds of whole tiles, each round's
    blocks all-gathered asynchronously into frame order, odd tail frame):
    maps and argmax of every frame on every rank, identical to one process."""
    g = torch.Generator().manual_seed(F)
    Y = torch.complex(torch.randn((F, 4, 8), generator=g), torch.randn((F, 4, 8), generator=g))
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_runner_worker, args=(2, _free_port(), Y, rounds, tile, ret), nprocs=2, join=True)
    assert dict(ret) == {0: True, 1: True}


def test_sharded_runner_single_process():
    g = torch.Generator().manual_seed(3)
    Y = torch.complex(torch.randn((50, 4, 8), generator=g), torch.randn((50, 4, 8), generator=g))
    plan = _StubCapturePlan()
    rn = D.ShardedRunner(plan, 50, rounds=3, tile=8)
    rn.load(Y)
    m, a = rn.run()
    ref_m, ref_a = plan.run(Y)
    assert torch.equal(m, ref_m) and torch.equal(a, ref_a)
    assert [w for _, w in rn.rounds] == [18, 16, 16]
