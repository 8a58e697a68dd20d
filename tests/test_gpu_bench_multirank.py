"""bench.py's multi-rank path (torchrun, per-rank shards, max over ranks,
rank-0 JSON line) exercised on a 1-GPU box: BENCH_SINGLE_DEVICE_TEST puts
both ranks on device 0 with gloo for the host-side collectives.  Checks the
contract fields, not the numbers (two ranks share one GPU): an external
torchrun launch, and `bench.py --gpus 2` re-executing itself under
torch.distributed.run (with the config-3 / config-4 fields and their bitwise
checks against the 1-GPU result)."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("config", [2, 4])
def test_two_rank_bench_line(config):
    env = dict(os.environ, BENCH_SINGLE_DEVICE_TEST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--config", str(config), "--no-cpu", "--no-e2e", "--no-extra"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0
    assert d["scaling"] == ("strong" if config == 4 else "weak")
    assert "dp2" in d["config"]["parallelism"]


def test_bench_gpus_flag_self_launches():
    env = dict(os.environ, BENCH_SINGLE_DEVICE_TEST="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and "dp2" in d["config"]["parallelism"]
    for k in ("config3", "config4"):
        assert d[k]["scaling"] == "strong" and d[k]["value"] > 0
        assert d[k]["bitwise_vs_1gpu"] is True, d[k]
