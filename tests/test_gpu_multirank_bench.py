"""The N > 1 bench path end to end on one GPU: `torchrun --nproc-per-node 2
bench.py --gpus 2` with the host-staged gloo halo transport
(TOFR_DIST_BACKEND=gloo, both ranks on cuda:0).  Covers what the one-process
band tests do not: rendezvous, per-rank band sessions, the exchange callback
through torch.distributed, max-over-ranks timing and the rank-0 JSON line.
The NCCL transport differs only in the backend the same P2P ops run on."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("workload", ["c1"])
def test_two_rank_bench_line(workload):
    env = dict(os.environ, TOFR_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--workload", workload, "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"].startswith("rowband2")
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
