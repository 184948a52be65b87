"""ShardedRunner (the multi-GPU strong-scaling step of bench.py) on one B200:
a one-rank NCCL group drives the same code path N ranks take -- graph-captured
rounds, each round's blocks all-gathered asynchronously into the static
[F, J] / [F] outputs -- and the result must agree with ``SrpPlan.run`` on all
frames (same argmax; maps to 3e-6: a round's frame count can select another
kernel family than the full batch) and with the reference's golden maps
within 1e-5 (the 2-rank
frame placement is covered on CPU by tests/test_distributed_cpu.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2012_09499_b200.distributed import ShardedRunner
from paper_2012_09499_b200.plan import SrpPlan
from helpers import assert_maps_match

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "c1.npz")


@pytest.fixture()
def nccl_one_rank():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        yield
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("path,key,amkey", [("approx", "approx_2", "argmax_approx_2"),
                                            ("conventional", "conv", "argmax_conv")])
def test_sharded_runner_nccl_one_rank(nccl_one_rank, path, key, amkey):
    with np.load(GOLDEN) as z:
        g = {k: z[k] for k in z.files}
    plan = SrpPlan(g["tdoa"], g["pair_m"], g["pair_mp"], g["bounds"], g["omega"],
                   sample_period=1.0 / 16000.0, n_aux=2)
    Y = torch.as_tensor(g["Y"])
    F = Y.shape[0]
    rn = ShardedRunner(plan, F, Y.shape[1], path, maps=True, rounds=3, tile=2)
    assert len(rn.rounds) == 3 and sum(w for _, w in rn.rounds) == F
    rn.load(Y.pin_memory())
    ref_m, ref_a = plan.run(Y.cuda(), path)
    for _ in range(2):
        m, a = rn.run()
        torch.cuda.synchronize()
        assert torch.equal(a, ref_a)
        err = (m - ref_m).norm(dim=1) / ref_m.norm(dim=1)
        assert float(err.max()) <= 3e-6, float(err.max())
    assert_maps_match(m.cpu().numpy(), g[key], a.cpu().numpy(), what=f"sharded {path}")
    assert list(a.cpu().numpy()) == list(g[amkey])
    rn2 = ShardedRunner(plan, F, Y.shape[1], path, maps=False, rounds=2, tile=2)
    rn2.load(Y.cuda())
    m2, a2 = rn2.run()
    torch.cuda.synchronize()
    assert m2 is None and torch.equal(a2, ref_a)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_plan_on_a_non_current_device():
    """A plan built with ``device='cuda:1'`` launches on that GPU (the C-ABI
    calls run under ``torch.cuda.device``), whatever the current device is."""
    with np.load(GOLDEN) as z:
        g = {k: z[k] for k in z.files}
    torch.cuda.set_device(0)
    plan = SrpPlan(g["tdoa"], g["pair_m"], g["pair_mp"], g["bounds"], g["omega"],
                   sample_period=1.0 / 16000.0, n_aux=2, device="cuda:1")
    Y = torch.as_tensor(g["Y"]).to("cuda:1")
    for path, key, amkey in (("approx", "approx_2", "argmax_approx_2"),
                             ("conventional", "conv", "argmax_conv")):
        maps, am = plan.run(Y, path)
        torch.cuda.synchronize("cuda:1")
        assert maps.device == torch.device("cuda", 1) and torch.cuda.current_device() == 0
        assert_maps_match(maps.cpu().numpy(), g[key], am.cpu().numpy(), what=f"cuda:1 {path}")
        assert list(am.cpu().numpy()) == list(g[amkey])
