"""bench.py under torchrun with two ranks (gloo, both on cuda:0 — gpurun has
one GPU): the sharded-store path (one world x R archive, Store shard k % 2 on
each rank), the barrier + max-over-ranks timing and the JSON line the driver
parses, for the decode bench and the DDP training bench (c5)."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(*bench_args):
    env = dict(os.environ, RINR_BENCH_BACKEND="gloo", RINR_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", "2",
           *bench_args]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_two_ranks_sharded():
    d = _torchrun("--steps", "3", "--warmup", "1", "--no-cpu", "--no-e2e", "--no-subs", "--store-records", "4096")
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["config"]["store_records_total"] == 8192 and d["config"]["store_records_per_gpu"] == 4096
    assert "shard" in d["config"]["parallelism"]


def test_bench_c5_two_ranks_ddp():
    d = _torchrun("--config", "c5", "--steps", "2", "--warmup", "1", "--store-records", "4096")
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["store_records_total"] == 8192 and d["config"]["store_records_per_gpu"] == 4096
    assert d["final_loss"] == d["final_loss"]  # finite
