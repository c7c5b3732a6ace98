"""bench.py's multi-rank run on one GPU (-m gpu).

torchrun with 2 ranks sharing cuda:0 (MASPCG_BENCH_SHARED_GPU=1: gloo process group, peer-memory
communicator over CUDA IPC). It checks the N > 1 code path of the bench contract: the slab extents, the
IPC handle exchange, the barriers, the max over ranks, and a single JSON line printed by rank 0. The
time-sliced numbers are not measurements; the cross-GPU NCCL variant needs more than one GPU.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(400)]


@pytest.mark.parametrize("path", [1, 4])
def test_bench_two_ranks_shared_gpu(path):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    env = dict(os.environ, MASPCG_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29530 + path), "bench.py", "--gpus", "2",
           "--comm", "peer", "--path", str(path), "--steps", "1", "--warmup", "3", "--maxit", "20",
           "--no-cpu-baseline", "--no-e2e"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=360)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 1 and d["config"]["iters_per_solve"] == 20
    assert "x2 peer-memory communicator" in d["config"]["parallelism"]
    assert d["value"] > 0 and d["gpu_launches"] > 0 and "test_mode" in d
