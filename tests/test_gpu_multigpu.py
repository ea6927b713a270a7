"""Multi-GPU parity (real part over NCCL/NVLink + per-shard synthesis).

Runs tests/mgpu_worker.py under torch.distributed.run on every visible GPU
(2 or 4 on a gpurun --gpus box); skipped when only one GPU is visible.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_multi_gpu_collectives_match_oracle():
    n = min(torch.cuda.device_count(), 4)
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mgpu_worker.py")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), worker],
                       capture_output=True, text=True, timeout=420)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"MGPU OK {n}" in r.stdout
