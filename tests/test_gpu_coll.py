"""The collective exerciser (paper_2405_02969_b200.coll), the counterpart of
the reference's cemu-coll (proj/tools/cemu_coll.cpp): verify mode checks
every element against a host recomputation, timing mode prints the
reference's RESULT lines and CSV columns."""
from __future__ import annotations

import csv
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _run(args, nproc=1, timeout=300):
    if nproc == 1:
        cmd = [sys.executable, "-m", "paper_2405_02969_b200.coll"] + args
    else:
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), "-m", "paper_2405_02969_b200.coll"] + args
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return r.stdout


@pytest.mark.parametrize("op", ["allreduce", "allgather"])
def test_verify_mode(cuda, tmp_path, op):
    cfg = tmp_path / "job.cfg"
    cfg.write_text("world_size = 16\nreal_ranks = 0\nbucket_bytes = 1\npayload.seed = 9\n")
    out = _run(["--config", str(cfg), "--mode", "verify", "--op", op, "--trials", "4", "--seed", "3"])
    assert f"VERIFY ok op={op} n=16 trials=4" in out


@pytest.mark.parametrize("host", [False, True])
def test_timing_mode_lines_and_csv(cuda, tmp_path, host):
    cfg = tmp_path / "job.cfg"
    cfg.write_text("world_size = 8\nreal_ranks = 0\nbucket_bytes = 1\n")
    out_csv = tmp_path / "t.csv"
    args = ["--config", str(cfg), "--mode", "timing", "--sizes", "4096", "1048577", "--reps", "5",
            "--warmup", "2", "--csv", str(out_csv)] + (["--host-buffers"] if host else [])
    out = _run(args)
    lines = [l for l in out.splitlines() if l.startswith("RESULT ")]
    assert [l.split()[2] for l in lines] == ["bytes=4096", "bytes=1048576"]
    rows = list(csv.reader(open(out_csv)))
    assert rows[0] == ["op", "size_bytes", "repetitions", "mean_us", "stddev_us"]
    assert [r[1] for r in rows[1:]] == ["4096", "1048576"] and all(float(r[3]) > 0 for r in rows[1:])


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("op", ["allreduce", "allgather"])
def test_verify_mode_two_real_ranks(tmp_path, op):
    cfg = tmp_path / "job.cfg"
    cfg.write_text("world_size = 12\nreal_ranks = 0,1\nbucket_bytes = 1\n")
    out = _run(["--config", str(cfg), "--mode", "verify", "--op", op, "--trials", "3"], nproc=2)
    assert f"VERIFY ok op={op} n=12 trials=3" in out
