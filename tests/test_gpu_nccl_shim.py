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


def run_mp_app(tmp_path, n, world, count, mode, iters=3, extra_env=None):
    """Starts tests/apps/nccl_mp_app on GPUs 0..n-1 (real ranks 0..n-1 of a
    world of `world`) under the interposer; returns [(result, stdout, stderr)]."""
    app = os.path.join(ROOT, "tests", "apps", "nccl_mp_app")
    cfg = tmp_path / f"job_{mode}.cfg"
    cfg.write_text(f"world_size = {world}\nreal_ranks = {','.join(map(str, range(n)))}\nbucket_bytes = 1\n")
    idfile = tmp_path / f"id_{mode}"
    env = dict(os.environ, CEMU_CONFIG=str(cfg), LD_PRELOAD=SHIM, CEMU_DEBUG="INFO", **(extra_env or {}))
    procs = []
    for r in range(n):
        out = tmp_path / f"out_{mode}_{r}.bin"
        procs.append((out, subprocess.Popen([app, str(world), str(r), str(r), str(count), mode, str(idfile), str(out),
                                             str(iters)], env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
    res = []
    for out, p in procs:
        so, se = p.communicate(timeout=240)
        assert p.returncode == 0, so + se
        res.append((np.fromfile(out, dtype=np.float32), so, se))
    return res


def mp_inputs(n, count):
    i = np.arange(count, dtype=np.int64)
    return [(((7 * i + 13 * r) % 61) - 30).astype(np.float32) * 0.125 for r in range(n)]


@pytest.mark.skipif(not __import__("torch").cuda.is_available() or __import__("torch").cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode,path", [("plain", "nccl reduce-scatter"), ("register", "fused"), ("window", "fused")])
def test_multi_process_nccl_app_reaches_the_fused_path(tmp_path, mode, path):
    """An unmodified multi-process NCCL job (one process per GPU) under
    LD_PRELOAD: buffers it registers (ncclCommRegister on cudaMalloc memory,
    or ncclMemAlloc + ncclCommWindowRegister) take the fused NVLink kernel;
    unregistered ones the NCCL reduce-scatter + synthesis + allgather path.
    Every rank's result equals the oracle bit for bit."""
    import torch
    n = min(torch.cuda.device_count(), 4)
    world, count = 8 * n, (3 << 20) + 16 * n
    sends = mp_inputs(n, count)
    for r, (got, so, se) in enumerate(run_mp_app(tmp_path, n, world, count, mode)):
        assert f"mode {mode}" in so and "async_error 0" in so, so
        assert f"allreduce {count * 4} B -> {path}" in se, se[-2000:]
        want = P.allreduce(7, P.PAYLOAD_HASH, world, list(range(n)), r, 1, sends, count)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (mode, r)
