"""GPU, >= 2 GPUs: emulated vs baseline (the reference's cemu-bench
`microbench` and `e2e`, proj/tools/cemu_bench.cpp:196-290, :346-380).

Baseline: every rank real, NCCL over NVLink.  Emulated: rank 0 alone in a
world of the same size, its peers emulated, the network delay calibrated
from the baseline's own size sweep (paper_2405_02969_b200/fidelity.py).
Checks: per-call latency emulated / baseline <= 1.05 at >= 2 MiB (the
reference's rule, :281), and the reference's e2e training loops (bert-like,
ResNet-50 with 25 MiB buckets) within 1% of the baseline iteration time;
the real-compute MLP within 2% once calibrated under load with NCCL's SM
footprint."""
from __future__ import annotations

import json
import os
import re
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_emulated_matches_baseline():
    n = min(torch.cuda.device_count(), 4)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), "-m",
                        "paper_2405_02969_b200.fidelity", "--segments", "3", "--max-mib", "64",
                        "--e2e-iters", "12", "--mlp-iters", "12"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    m = re.search(r"FIDELITY (\{.*\})", r.stdout)
    assert m, r.stdout[-3000:]
    res = json.loads(m.group(1))
    assert res["k"] == n
    assert res["microbench_check"]["pass_table"], res["microbench"]
    for row in res["e2e"]:
        assert row["rel_err_table"] < 0.01, row
    # the real-compute MLP: NCCL's SM footprint emulated and the emulator's
    # memory pass held to it; 12 noisy iterations per repeat
    # here, so the regression bound is looser than the < 1% the full runs
    # show -- and without the footprint the error is 6-9%
    mlp = res["mlp"]
    best = min(mlp[f"rel_err_{t}"] for t in ("table_footprint", "loaded_footprint", "in_situ_footprint"))
    assert best < 0.02, mlp
    assert mlp["rel_err_table"] > best, mlp
