"""GPU: bench.py's N > 1 path end to end (torchrun, 2 ranks, the fused P2P
exchange) on the one available GPU -- both ranks share device 0
(MBX_BENCH_ONE_DEVICE=1), so the number is meaningless but the plumbing
(row shards, IPC setup over gloo, barriers, max-over-ranks timing, e2e,
collective teardown) is the one a multi-GPU run executes."""
import json
import os
import socket
import subprocess
import sys

import pytest
from conftest import gpu_shared_between_processes

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not gpu_shared_between_processes(),
                    reason="device 0 is in an exclusive compute mode")
def test_bench_two_ranks_fused_exchange():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, MBX_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--steps", "1", "--warmup", "3", "--scale", "16", "--no-extras", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert "fused P2P" in d["config"]["workload"]
    assert abs(d["e2e"]["mass"] - 1.0) <= 1e-5
