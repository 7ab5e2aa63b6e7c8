"""bench.py's N > 1 path end to end on a one-GPU box: torchrun with two ranks
sharing GPU 0 (FGB_DIST_BACKEND=gloo: torch.distributed over gloo, the
sharded build exchanging through the host communicator), the corpus
generated once by rank 0 into /dev/shm and mapped by rank 1, queries split
by contiguous range, max-over-ranks timing.  On the 8-GPU box the same
launcher runs one rank per GPU over NCCL."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_bench_on_one_gpu():
    env = dict(os.environ, FGB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "1", "--docs", "20000", "--queries", "2000", "--eval-queries", "200",
           "--no-cpu-baseline", "--no-build-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["config"]["queries_per_gpu"] == 1000
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["recall_at_10"] >= 0.9
    assert "host-staged" in line["config"]["parallelism"]
