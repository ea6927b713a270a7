"""GPU: the paper's interposition route.  tests/apps/nccl_app is an ordinary
NCCL program; with LD_PRELOAD=libnccl_cemu.so and CEMU_CONFIG set, its
ncclAllReduce becomes the emulated collective (world 8, 7 emulated ranks),
bit-exact against the oracle.  Without the preload it is real NCCL."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from oracle import port as P

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
APP = os.path.join(ROOT, "tests", "apps", "nccl_app")
SHIM = os.path.join(ROOT, "paper_2405_02969_b200", "libnccl_cemu.so")


def _run(tmp_path, env_extra, nranks, count):
    out = tmp_path / f"out_{nranks}_{count}.bin"
    env = dict(os.environ, **env_extra)
    r = subprocess.run([APP, str(nranks), str(count), str(out)], env=env, capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    return np.fromfile(out, dtype=np.float32), r.stdout


def test_unmodified_nccl_app_under_ld_preload(cuda, tmp_path):
    cfg = tmp_path / "job.cfg"
    cfg.write_text("world_size = 8\nreal_ranks = 0\nbucket_bytes = 65536\n")
    count = (1 << 20) + 3
    x = (np.arange(count) % 97).astype(np.float32) * 0.25
    got, log = _run(tmp_path, {"CEMU_CONFIG": str(cfg), "LD_PRELOAD": SHIM}, 8, count)
    assert "world 8" in log
    want = P.allreduce(7, P.PAYLOAD_HASH, 8, [0], 0, 1, [x], count)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_same_app_is_plain_nccl_without_preload(cuda, tmp_path):
    count = 4099
    got, log = _run(tmp_path, {}, 1, count)  # a one-rank NCCL world: identity
    assert np.array_equal(got, (np.arange(count) % 97).astype(np.float32) * 0.25)


def test_world_size_mismatch_is_reported(cuda, tmp_path):
    cfg = tmp_path / "job.cfg"
    cfg.write_text("world_size = 8\nreal_ranks = 0\nbucket_bytes = 65536\n")
    r = subprocess.run([APP, "4", "16", str(tmp_path / "x.bin")],
                       env=dict(os.environ, CEMU_CONFIG=str(cfg), LD_PRELOAD=SHIM),
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "ncclCommInitRank" in r.stderr


def test_shim_refuses_what_it_does_not_emulate(cuda, tmp_path):
    """Entry points outside the emulated world fail loudly in the shim instead
    of reaching the real libnccl with an emulated communicator; the config /
    abort / registration entry points work."""
    import ctypes as C
    shim = C.CDLL(os.path.join(ROOT, "paper_2405_02969_b200", "libnccl_cemu.so"))
    cfg = tmp_path / "job.cfg"
    cfg.write_text("world_size = 4\nreal_ranks = 0\nbucket_bytes = 1\n")
    os.environ["CEMU_CONFIG"] = str(cfg)
    comm = C.c_void_p()
    from paper_2405_02969_b200._capi import UniqueId
    uid = UniqueId()  # passed by value, as ncclUniqueId is
    assert shim.ncclCommInitRankConfig(C.byref(comm), 4, uid, 0, None) == 0
    shim.ncclGetLastError.restype = C.c_char_p
    assert shim.ncclSend(None, C.c_size_t(4), 7, 1, comm, None) == 5
    assert b"point-to-point" in shim.ncclGetLastError(comm)
    assert shim.ncclReduce(None, None, C.c_size_t(4), 7, 0, 0, comm, None) == 5
    h = C.c_void_p(1)
    assert shim.ncclCommRegister(comm, None, C.c_size_t(0), C.byref(h)) == 0 and not h.value
    assert shim.ncclCommAbort(comm) == 0


def test_integration_recipe_cpp_session(cuda, tmp_path):
    """INTEGRATION.md's C++ drop-in for WorkerSession (tests/apps/
    b200_session.cpp): host-span allreduce (int32 lanes) and allgather
    (bytes) through the C-ABI, real rank 2 of a world of 6."""
    app = os.path.join(ROOT, "tests", "apps", "b200_session")
    cfg = tmp_path / "job.cfg"
    cfg.write_text("world_size = 6\nreal_ranks = 2\nbucket_bytes = 65536\n")
    n, blk, W, rank = 100003, 1000, 6, 2
    out = tmp_path / "out.bin"
    r = subprocess.run([app, str(cfg), str(rank), str(n), str(out)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"b200_session ok rank {rank} world {W}" in r.stdout
    raw = np.fromfile(out, dtype=np.uint8)
    got_ar = raw[:4 * n].view(np.int32)
    got_ag = raw[4 * n:]
    x = (np.arange(n, dtype=np.int64) * 7 + rank).astype(np.int32)
    want_ar = P.allreduce(2, P.PAYLOAD_HASH, W, [rank], rank, 1, [x], n)
    assert np.array_equal(got_ar, want_ar)
    own = ((np.arange(blk) + rank + 1) % 256).astype(np.uint8)
    want_ag = P.allgather(1, P.PAYLOAD_HASH, W, [rank], rank, 1, [own], blk)
    assert np.array_equal(got_ag, want_ag)
