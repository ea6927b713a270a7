"""ctypes binding of _ref/libcemu_ref.so: the REFERENCE cemu_core itself.

TEST INFRASTRUCTURE ONLY.  Built here from /root/reference/proj/src by
``oracle/Makefile``; the prebuilt .so travels to the GPU box (git-ignored,
not gpurun-ignored).  ``available()`` is False when it was never built.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(_HERE, "_ref", "libcemu_ref.so")
_LIB = None


def available() -> bool:
    return os.path.exists(PATH)


def lib():
    global _LIB
    if _LIB is None:
        if not available():
            raise RuntimeError(f"reference not built: {PATH} (run `make -C oracle ref`)")
        L = C.CDLL(PATH)
        u32, u64, i64, dbl, vp, cp, sz = (C.c_uint32, C.c_uint64, C.c_int64, C.c_double,
                                          C.c_void_p, C.c_char_p, C.c_size_t)
        L.ref_config_render.restype = C.c_int
        L.ref_config_render.argtypes = [cp, cp, sz, C.POINTER(u64), cp, sz]
        L.ref_chunk_bytes.restype = u64
        L.ref_chunk_bytes.argtypes = [u32, u64, u32, u32]
        L.ref_chunk_offset_bytes.restype = u64
        L.ref_chunk_offset_bytes.argtypes = [u32, u64, u32, u32]
        L.ref_dump_dag.restype = C.c_int
        L.ref_dump_dag.argtypes = [C.c_int, u32, u64, u32, u32, cp, sz, cp, sz]
        L.ref_dump_boundary.restype = C.c_int
        L.ref_dump_boundary.argtypes = [C.c_int, u32, u64, u32, vp, C.c_int, C.c_int, cp, sz, cp, sz]
        L.ref_ring_allreduce_delay_us.restype = dbl
        L.ref_ring_allreduce_delay_us.argtypes = [u32, u64, dbl, dbl, dbl]
        L.ref_ring_allgather_delay_us.restype = dbl
        L.ref_ring_allgather_delay_us.argtypes = [u32, u64, dbl, dbl]
        common = [C.c_int, u32, u64, u32, vp, C.c_int, C.c_int, dbl, dbl, dbl, dbl, dbl]
        L.ref_release_offsets.restype = C.c_int
        L.ref_release_offsets.argtypes = common + [vp, sz, cp, sz]
        L.ref_opstate_floors.restype = C.c_int
        L.ref_opstate_floors.argtypes = common + [i64, vp, sz, cp, sz]
        L.ref_simulated_call_latency_us.restype = i64
        L.ref_simulated_call_latency_us.argtypes = [C.c_int, u32, u64, u32, C.c_int, dbl, dbl, dbl,
                                                    dbl, dbl, vp, sz, cp, sz]
        L.ref_reduce_add_i32.restype = None
        L.ref_reduce_add_i32.argtypes = [vp, vp, sz]
        L.ref_reduce_add_u8.restype = None
        L.ref_reduce_add_u8.argtypes = [vp, vp, sz]
        L.ref_reduce_backend.restype = C.c_char_p
        L.ref_emulated_collective.restype = C.c_int
        L.ref_emulated_collective.argtypes = [u32, C.c_int, vp, u64, u32, C.c_int, dbl, dbl, dbl, dbl,
                                              dbl, C.c_int, C.c_int, vp, cp, sz]
        L.ref_trace_open.restype = None
        L.ref_trace_open.argtypes = [cp]
        L.ref_model_render.restype = C.c_int
        L.ref_model_render.argtypes = [cp, cp, sz, cp, sz]
        L.ref_bucketize.restype = C.c_int
        L.ref_bucketize.argtypes = [cp, u64, vp, sz, cp, sz]
        L.ref_run_training_loop.restype = C.c_int
        L.ref_run_training_loop.argtypes = [cp, u32, u64, C.c_int, dbl, dbl, dbl, dbl, dbl, vp, sz, cp, sz]
        L.ref_real_ring.restype = C.c_int
        L.ref_real_ring.argtypes = [u32, C.c_int, vp, u64, u32, cp, sz]
        L.ref_emulator_start.restype = vp
        L.ref_emulator_start.argtypes = [cp, cp, sz]
        L.ref_emulator_sessions.restype = u64
        L.ref_emulator_sessions.argtypes = [vp]
        L.ref_emulator_stop.restype = None
        L.ref_emulator_stop.argtypes = [vp]
        L.ref_config_digest.restype = u64
        L.ref_config_digest.argtypes = [cp]
        _LIB = L
    return _LIB


class RefError(RuntimeError):
    pass


def _text_call(fn, *args):
    cap = 1 << 16
    while True:
        out = C.create_string_buffer(cap)
        err = C.create_string_buffer(1024)
        r = fn(*args, out, cap, err, 1024)
        if r == -1 and err.value:
            raise RefError(err.value.decode())
        if r >= 0:
            return out.value.decode()
        cap = -r + 16


def config_render(text: str):
    """-> (canonical render, digest) exactly as config.cpp:264-312 produce."""
    cap = 1 << 16
    out = C.create_string_buffer(cap)
    err = C.create_string_buffer(1024)
    dig = C.c_uint64(0)
    r = lib().ref_config_render(text.encode(), out, cap, C.byref(dig), err, 1024)
    if r < 0:
        raise RefError(err.value.decode())
    return out.value.decode(), dig.value


def chunk_bytes(n, total, elem, c):
    return lib().ref_chunk_bytes(n, total, elem, c)


def chunk_offset_bytes(n, total, elem, c):
    return lib().ref_chunk_offset_bytes(n, total, elem, c)


def dump_dag(coll, n, nbytes, elem=1, op_id=0):
    return _text_call(lib().ref_dump_dag, coll, n, nbytes, elem, op_id)


def dump_boundary(coll, n, nbytes, elem=1, real=(0,), side=0):
    arr = np.asarray(sorted(real), dtype=np.uint32)
    return _text_call(lib().ref_dump_boundary, coll, n, nbytes, elem, arr.ctypes.data, len(arr), side)


def ring_allreduce_delay_us(n, nbytes, a, b, g):
    return lib().ref_ring_allreduce_delay_us(n, nbytes, a, b, g)


def ring_allgather_delay_us(n, nbytes, a, b):
    return lib().ref_ring_allgather_delay_us(n, nbytes, a, b)


def _delay_args(kind, a, b, g, fixed, inject):
    return [kind, a, b, g, fixed, inject]


def release_offsets(coll, n, nbytes, elem=1, real=(0,), kind=0, a=0.0, b=0.0, g=0.0,
                    fixed=0.0, inject=0.0):
    arr = np.asarray(sorted(real), dtype=np.uint32)
    cap = 4 * n * max(len(arr), 1) + 8
    out = np.zeros(cap, dtype=np.float64)
    err = C.create_string_buffer(1024)
    k = lib().ref_release_offsets(coll, n, nbytes, elem, arr.ctypes.data, len(arr),
                                  *_delay_args(kind, a, b, g, fixed, inject),
                                  out.ctypes.data, cap, err, 1024)
    if k < 0:
        raise RefError(err.value.decode())
    return out[:k]


def opstate_floors(coll, n, nbytes, elem=1, real=(0,), kind=0, a=0.0, b=0.0, g=0.0,
                   fixed=0.0, inject=0.0, now=0):
    arr = np.asarray(sorted(real), dtype=np.uint32)
    cap = 4 * n * max(len(arr), 1) + 8
    out = np.zeros(cap, dtype=np.int64)
    err = C.create_string_buffer(1024)
    k = lib().ref_opstate_floors(coll, n, nbytes, elem, arr.ctypes.data, len(arr),
                                 *_delay_args(kind, a, b, g, fixed, inject), now,
                                 out.ctypes.data, cap, err, 1024)
    if k < 0:
        raise RefError(err.value.decode())
    return out[:k]


def simulated_call_latency_us(coll, n, nbytes, elem=1, kind=0, a=0.0, b=0.0, g=0.0,
                              fixed=0.0, inject=0.0):
    cap = 4 * n + 8
    rel = np.zeros(cap, dtype=np.int64)
    err = C.create_string_buffer(1024)
    t = lib().ref_simulated_call_latency_us(coll, n, nbytes, elem, kind, a, b, g, fixed, inject,
                                            rel.ctypes.data, cap, err, 1024)
    if t < 0:
        raise RefError(err.value.decode())
    k = 2 * (n - 1) if coll == 0 else n - 1
    return t, rel[:k]


def emulated_collective(n, coll, buf: np.ndarray, plan_bytes, elem, kind=0, a=0.0, b=0.0,
                        g=0.0, fixed=0.0, inject=0.0, warmup=0, reps=1):
    """Runs the reference WorkerSession(rank 0) against an in-thread
    EmulatorServer on loopback; `buf` is updated in place with the last call's
    result.  Returns the per-call wall times (us) of the timed reps."""
    assert buf.flags.c_contiguous
    times = np.zeros(max(reps, 1), dtype=np.float64)
    err = C.create_string_buffer(2048)
    r = lib().ref_emulated_collective(n, coll, buf.ctypes.data, plan_bytes, elem, kind, a, b, g,
                                      fixed, inject, warmup, reps, times.ctypes.data, err, 2048)
    if r != 0:
        raise RefError(err.value.decode())
    return times[:reps]


def real_ring(n, coll, bufs, plan_bytes, elem):
    """n real reference WorkerSessions (threads) over loopback; bufs updated."""
    for b in bufs:
        assert b.flags.c_contiguous
    ptrs = (C.c_void_p * n)(*[b.ctypes.data for b in bufs])
    err = C.create_string_buffer(2048)
    r = lib().ref_real_ring(n, coll, C.cast(ptrs, C.c_void_p), plan_bytes, elem, err, 2048)
    if r != 0:
        raise RefError(err.value.decode())


def run_training_loop(model_text: str, n: int, bucket_bytes: int, kind=0, a=0.0, b=0.0, g=0.0, fixed=0.0,
                      inject=0.0):
    """The reference's run_training_loop (harness.cpp:191-254) against its
    emulator over loopback; returns per-iteration wall times in us."""
    cap = 100000
    out = np.zeros(cap, dtype=np.float64)
    err = C.create_string_buffer(2048)
    k = lib().ref_run_training_loop(model_text.encode(), n, bucket_bytes, kind, a, b, g, fixed, inject,
                                    out.ctypes.data, cap, err, 2048)
    if k < 0:
        raise RefError(err.value.decode())
    return out[:k]


def model_render(text: str) -> str:
    """render_model_spec(parse_model_spec(text)) (harness.cpp:27-114)."""
    return _text_call(lib().ref_model_render, text.encode())


def bucketize(text: str, bucket_bytes: int):
    out = np.zeros(3 * 4096, dtype=np.uint64)
    err = C.create_string_buffer(1024)
    k = lib().ref_bucketize(text.encode(), bucket_bytes, out.ctypes.data, len(out), err, 1024)
    if k < 0:
        raise RefError(err.value.decode())
    return [tuple(int(v) for v in out[3 * i:3 * i + 3]) for i in range(k)]


def trace_open(path: str) -> None:
    """Opens the reference's process-wide EventLog (trace.cpp:9-19)."""
    lib().ref_trace_open(path.encode())


class Emulator:
    """A reference EmulatorServer (emulator.cpp) serving in a thread of this
    process, on the config's emulated endpoint -- the `cemu-emulator` the
    B200 wire mode talks to in the interop tests."""

    def __init__(self, cfg_text: str):
        err = C.create_string_buffer(1024)
        self._h = lib().ref_emulator_start(cfg_text.encode(), err, 1024)
        if not self._h:
            raise RefError(err.value.decode())

    @property
    def sessions(self) -> int:
        return lib().ref_emulator_sessions(self._h)

    def stop(self):
        if self._h:
            lib().ref_emulator_stop(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.stop()


def config_digest(text: str) -> int:
    return lib().ref_config_digest(text.encode())
