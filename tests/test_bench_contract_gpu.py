"""The driver's bench contract on a reduced frame count (C4 geometry, all
600k candidates, 192 frames): ``bench.py`` prints ONE JSON line on stdout
with the contract's keys, its parity block passes, and the sharded
(multi-GPU) code path gives the same line shape through a one-rank NCCL
group.  The reference arm prints its line with ``impl: reference``."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
SMALL = ["--frames", "192", "--steps", "1", "--warmup", "1", "--conv-steps", "1", "--no-sweeps",
         "--no-cpu-baseline"]


def _one_json_line(stdout):
    lines = [ln for ln in stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, lines[:5]
    return json.loads(lines[0])


def _check_line(d, n_gpus=1):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "clocks", "parity"):
        assert k in d, k
    assert d["n_gpus"] == n_gpus and d["higher_is_better"] is True and d["vs_baseline"] is None
    assert d["unit"] == "frames*candidates/s" and d["value"] > 0 and d["gpu_launches"] >= 2
    assert "workload" in d["config"] and d["config"]["frames"] == 192
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 192 * 32 * 512 * 8
    assert e["d2h_bytes_per_step"] == 192 * 600000 * 4 + 192 * 4
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and "traffic" in r
    for path in ("approx", "conventional"):
        p = d["parity"][path]
        assert p["pass"] and p["rel_l2_worst"] <= 1e-5 and p["argmax_mismatches"] == 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_bench_line_contract_small():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *SMALL],
                         capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    _check_line(_one_json_line(out.stdout))


def test_bench_sharded_path_one_rank_nccl():
    env = dict(os.environ, SRPB_BENCH_SHARDED="1")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
         "--master-addr", "127.0.0.1", "--master-port", str(port),
         os.path.join(ROOT, "bench.py"), "--gpus", "1", *SMALL],
        capture_output=True, text=True, cwd=ROOT, env=env, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    d = _one_json_line(out.stdout)
    _check_line(d)
    assert d["gpu_launches"] >= 3   # the only full-tile round of 192 frames: lattice, fix-up, K4


def test_bench_refuses_more_gpus_than_visible():
    import torch

    n = torch.cuda.device_count()
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n + 1),
                          *SMALL], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.returncode != 0 and "CUDA devices are visible" in (out.stderr + out.stdout)


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--cpu-cands", "64",
                          "--cpu-conv-cands", "64"],
                         capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    d = _one_json_line(out.stdout)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "frames*candidates/s"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
