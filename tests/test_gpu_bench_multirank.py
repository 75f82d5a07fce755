"""bench.py's N > 1 code path on a one-GPU box (PROTOX_BENCH_SHARED_GPU=1:
both ranks on cuda:0, gloo process group, the fused push halo between the two
processes through CUDA IPC): the run must finish and print one JSON line
with n_gpus = 2, the max-over-ranks timing, the `halo` block and an e2e
number.  Guards the driver's multi-GPU scaling run, which this repo cannot
otherwise execute before round end."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_shared_gpu():
    env = dict(os.environ, PROTOX_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2
    assert d["config"]["halo"].startswith("p2p") and d["config"]["partition"] == "slabs x2"
    h = d["halo"]
    assert h["bytes_per_neighbour_direction"] == (16384 + 2) * 8
    assert h["kernel_ms"] > 0 and h["ms_per_exchange_period"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 2 * 16384 * 16384 * 8
    assert d["gpu_launches"] > 0
