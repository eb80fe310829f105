"""bench.py contract at N > 1 on a one-GPU box: two torchrun ranks on device 0 (gloo
process group, copy-engine IPC ring) must print ONE JSON line with the whole-job
value, max-over-ranks timing and the measured ring timeline.  The numbers are not a
measurement (both ranks share one GPU); the code path is what is tested."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_gpu():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, BURST_BENCH_ONE_GPU="1", BURST_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "1", "--config", "c2", "--comm", "ce"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "ring sp2"
    m = d["comm"]["measured"]
    assert m["fwd_bytes_per_rank"] > 0 and 0.0 <= m["fwd_hidden_frac"] <= 1.0
    assert d["e2e"]["h2d_bytes_per_step"] > 0
