"""Multi-GPU: KV-head-sharded decode over NCCL with the real kernels (needs >= 2 GPUs)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("transport,fused,host,sync", [
    ("nccl", "1", "0", "-"), ("nccl", "0", "0", "-"), ("peer", "1", "0", "kernel"),
    ("peer", "1", "1", "kernel"), ("peer", "1", "0", "stream"), ("peer", "1", "1", "stream"),
    ("peer", "1", "0", "step"), ("peer", "1", "1", "step"), ("peer", "1", "0", "step-relay"),
    ("peer", "1", "1", "step-relay")])
@pytest.mark.parametrize("nproc", [2, 4])
def test_sharded_engine_matches_oracle(built, nproc, transport, fused, host, sync):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", "--master-port=29531",
           str(ROOT / "tests" / "dist_gpu_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=dict(os.environ, PYTHONPATH=str(ROOT), LAM_TEST_FUSED=fused,
                                LAM_TEST_TRANSPORT=transport, LAM_TEST_HOST=host,
                                LAM_TEST_SYNC=sync))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("OK") == nproc


@pytest.mark.parametrize("transport,sync", [("nccl", "-"), ("peer", "kernel"), ("peer", "step")])
@pytest.mark.parametrize("nproc", [2, 4])
def test_request_sharded_engine_matches_oracle(built, nproc, transport, sync):
    """request_partition-based pool (KV heads not divisible by N), real kernels, over NCCL or
    the zero-copy peer transport (row map, lam_peer_io.row_src)."""
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", "--master-port=29532",
           str(ROOT / "tests" / "dist_gpu_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=dict(os.environ, PYTHONPATH=str(ROOT), LAM_TEST_SHARD="request",
                                LAM_TEST_TRANSPORT=transport, LAM_TEST_SYNC=sync))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("OK") == nproc
