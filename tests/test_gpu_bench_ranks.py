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
    assert d["n_gpus"] == 2 and d["steps"] == 1 and d["run"]["iters_per_solve"] == 20
    assert "x2 peer-memory communicator" in d["config"]["parallelism"]
    assert d["value"] > 0 and d["gpu_launches"] > 0 and "test_mode" in d


def test_bench_self_launches_ranks_without_torchrun():
    """`python bench.py --gpus 2` with WORLD_SIZE unset launches its two ranks itself (torch.distributed.run
    on 127.0.0.1) instead of silently running one: one JSON line with n_gpus 2 (ranks sharing cuda:0 in the
    MASPCG_BENCH_SHARED_GPU test mode, peer communicator)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["MASPCG_BENCH_SHARED_GPU"] = "1"
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--comm", "peer", "--steps", "1", "--warmup", "3",
           "--maxit", "20", "--no-cpu-baseline", "--no-e2e"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=360)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and "x2 peer-memory communicator" in d["config"]["parallelism"]
    assert "torch.distributed.run" in out.stderr


def test_bench_refuses_more_gpus_than_visible():
    """Without the shared-GPU test mode, asking for more ranks than visible GPUs exits 2 (no silent N=1)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK",
                                                           "MASPCG_BENCH_SHARED_GPU")}
    n = torch.cuda.device_count() + 1
    out = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--steps", "1"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 2 and "refusing" in out.stderr
    assert not [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
