"""The multi-rank bench path (torchrun, TP groups, the peer-memory TP sum fused into K3 and
its start-up checks) run end to end with every rank on the one GPU (MLRA_BENCH_SHARED_GPU:
gloo instead of NCCL, time-sliced contexts -- a correctness run, not a measurement)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [2, 4])
def test_bench_runs_with_tp_ranks_sharing_one_gpu(n):
    import socket

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = str(s.getsockname()[1])
    env = dict(os.environ, MLRA_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", port, "bench.py", "--gpus", str(n), "--steps", "2",
           "--warmup", "3", "--quick", "--no-cpu"]
    res = subprocess.run(cmd, cwd=repo, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == n and line["config"]["parallelism"] == f"tp{n}"
    assert "fused into K3" in line["config"]["allreduce"]  # the fused sum passed its check
    assert line["gpu_launches"] == 3 * line["steps"]
