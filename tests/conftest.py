"""Shared test setup.

Markers: ``gpu`` -- needs a B200 (run with ``-m gpu``); everything else runs
on the CPU-only build container (``-m "not gpu"``).
"""
from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    # the built libraries are git-ignored: a fresh checkout builds them here
    # (the same recipe as __graft_entry__.build; nvcc cross-compiles sm_100a)
    libs = [os.path.join(ROOT, "paper_2405_02969_b200", "libcemu_b200.so"),
            os.path.join(ROOT, "oracle", "liboracle.so")]
    if not all(os.path.exists(p) for p in libs):
        import subprocess
        jobs = str(min(8, os.cpu_count() or 1))
        subprocess.run(["make", "-j", jobs, "-C", os.path.join(ROOT, "paper_2405_02969_b200")], check=True)
        subprocess.run(["make", "-j", jobs, "-C", os.path.join(ROOT, "oracle"), "all"], check=True)


def golden(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)
