"""ctypes binding of liboracle.so (the C restatement).  TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

ALLREDUCE, ALLGATHER, REDUCESCATTER, BROADCAST = 0, 1, 2, 3
DELAY_NONE, DELAY_ALPHA_BETA, DELAY_FIXED = 0, 1, 2
ALGO_RING, ALGO_TREE, ALGO_HIER = 0, 1, 2
PAYLOAD_HASH, PAYLOAD_ZERO = 0, 1

# ncclDataType_t codes -> numpy storage dtypes (fp16/bf16 stored as uint16)
DTYPES = {
    0: np.int8, 1: np.uint8, 2: np.int32, 3: np.uint32, 4: np.int64,
    5: np.uint64, 6: np.uint16, 7: np.float32, 8: np.float64, 9: np.uint16,
}


class DelayModel(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("algo", C.c_int),
        ("alpha_us", C.c_double), ("beta_us_per_byte", C.c_double),
        ("gamma_us_per_byte", C.c_double),
        ("fixed_us", C.c_double), ("inject_us", C.c_double),
        ("gpus_per_node", C.c_uint32),
        ("intra_alpha_us", C.c_double), ("intra_beta_us_per_byte", C.c_double),
    ]


def delay_model(kind=DELAY_NONE, algo=ALGO_RING, alpha=0.0, beta=0.0, gamma=0.0,
                fixed=0.0, inject=0.0, gpus_per_node=1, intra_alpha=None,
                intra_beta=None) -> DelayModel:
    return DelayModel(kind, algo, alpha, beta, gamma, fixed, inject, gpus_per_node,
                      alpha if intra_alpha is None else intra_alpha,
                      beta if intra_beta is None else intra_beta)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle not built: {path} (run `make -C oracle oracle`)")
        L = C.CDLL(path)
        u32, u64, i64, dbl, vp = C.c_uint32, C.c_uint64, C.c_int64, C.c_double, C.c_void_p
        L.or_chunk_bytes.restype = u64
        L.or_chunk_bytes.argtypes = [u32, u64, u32, u32]
        L.or_chunk_offset_bytes.restype = u64
        L.or_chunk_offset_bytes.argtypes = [u32, u64, u32, u32]
        L.or_positions.restype = u32
        L.or_positions.argtypes = [C.c_int, u32]
        L.or_send_chunk_at.restype = u32
        L.or_send_chunk_at.argtypes = [C.c_int, u32, u32, u32]
        L.or_dump_boundary_single_real.restype = C.c_int
        L.or_dump_boundary_single_real.argtypes = [C.c_int, u32, u64, u32, u32, C.c_char_p, C.c_size_t]
        L.or_to_real_count.restype = u32
        L.or_to_real_count.argtypes = [C.c_int, u32, vp, u32]
        L.or_ring_allreduce_delay_us.restype = dbl
        L.or_ring_allreduce_delay_us.argtypes = [u32, u64, dbl, dbl, dbl]
        L.or_ring_allgather_delay_us.restype = dbl
        L.or_ring_allgather_delay_us.argtypes = [u32, u64, dbl, dbl]
        L.or_model_total_us.restype = dbl
        L.or_model_total_us.argtypes = [C.POINTER(DelayModel), C.c_int, u32, u64]
        L.or_release_offsets.restype = C.c_int
        L.or_release_offsets.argtypes = [C.POINTER(DelayModel), C.c_int, u32, u64, u32, vp]
        L.or_release_floors.restype = C.c_int
        L.or_release_floors.argtypes = [C.POINTER(DelayModel), C.c_int, u32, u64, u32, i64, vp]
        L.or_call_latency_us.restype = i64
        L.or_call_latency_us.argtypes = [C.POINTER(DelayModel), C.c_int, u32, u64, u32]
        L.or_payload_key.restype = u32
        L.or_payload_key.argtypes = [u64, u32]
        L.or_payload_word.restype = u32
        L.or_payload_word.argtypes = [u32, u64]
        L.or_payload.restype = None
        L.or_payload.argtypes = [C.c_int, u32, u64, u64, vp]
        for name in ("or_allreduce", "or_allgather", "or_reducescatter"):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = [C.c_int, C.c_int, u32, vp, u32, u32, u64, vp, vp, u64]
        L.or_broadcast.restype = C.c_int
        L.or_broadcast.argtypes = [C.c_int, C.c_int, u32, vp, u32, u32, u32, u64, vp, vp, u64]
        L.or_ring_execute_allreduce.restype = C.c_int
        L.or_ring_execute_allreduce.argtypes = [C.c_int, u32, vp, u64, u32, vp]
        L.or_f32_to_bf16.restype = C.c_uint16
        L.or_f32_to_bf16.argtypes = [C.c_float]
        _LIB = L
    return _LIB


# ---- thin numpy-facing helpers -------------------------------------------
def chunk_bytes(n, total, elem, c):
    return lib().or_chunk_bytes(n, total, elem, c)


def chunk_offset_bytes(n, total, elem, c):
    return lib().or_chunk_offset_bytes(n, total, elem, c)


def send_chunk_at(coll, n, rank, p):
    return lib().or_send_chunk_at(coll, n, rank, p)


def positions(coll, n):
    return lib().or_positions(coll, n)


def dump_boundary(coll, n, nbytes, elem, real=0) -> str:
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        r = lib().or_dump_boundary_single_real(coll, n, nbytes, elem, real, buf, cap)
        if r >= 0:
            return buf.value.decode()
        cap = -r + 16


def to_real_count(coll, n, real):
    arr = np.asarray(sorted(real), dtype=np.uint32)
    return lib().or_to_real_count(coll, n, arr.ctypes.data, len(arr))


def model_total_us(m: DelayModel, coll, n, nbytes):
    return lib().or_model_total_us(C.byref(m), coll, n, nbytes)


def release_offsets(m: DelayModel, coll, n, nbytes, k):
    out = np.zeros(max(k, 1), dtype=np.float64)
    lib().or_release_offsets(C.byref(m), coll, n, nbytes, k, out.ctypes.data)
    return out[:k]


def release_floors(m: DelayModel, coll, n, nbytes, k, now_us=0):
    out = np.zeros(max(k, 1), dtype=np.int64)
    lib().or_release_floors(C.byref(m), coll, n, nbytes, k, now_us, out.ctypes.data)
    return out[:k]


def call_latency_us(m: DelayModel, coll, n, nbytes, k):
    return lib().or_call_latency_us(C.byref(m), coll, n, nbytes, k)


def payload_key(seed, rank):
    return lib().or_payload_key(seed, rank)


def payload_word(key, j):
    return lib().or_payload_word(key, j)


def payload(dtype, key, first, count):
    out = np.zeros(max(count, 1), dtype=DTYPES[dtype])
    lib().or_payload(dtype, key, first, count, out.ctypes.data)
    return out[:count]


def _ptrs(arrs):
    keep = [np.ascontiguousarray(a) for a in arrs]
    ptrs = (C.c_void_p * len(keep))(*[a.ctypes.data for a in keep])
    return keep, ptrs


def allreduce(dtype, mode, W, real, me, seed, sends, count):
    keep, ptrs = _ptrs(sends)
    real_arr = np.asarray(sorted(real), dtype=np.uint32)
    out = np.zeros(max(count, 1), dtype=DTYPES[dtype])
    rc = lib().or_allreduce(dtype, mode, W, real_arr.ctypes.data, len(real_arr), me, seed,
                            C.cast(ptrs, C.c_void_p), out.ctypes.data, count)
    if rc != 0:
        raise ValueError(f"or_allreduce rc={rc}")
    return out[:count]


def allgather(dtype, mode, W, real, me, seed, sends, sendcount):
    keep, ptrs = _ptrs(sends)
    real_arr = np.asarray(sorted(real), dtype=np.uint32)
    out = np.zeros(max(W * sendcount, 1), dtype=DTYPES[dtype])
    rc = lib().or_allgather(dtype, mode, W, real_arr.ctypes.data, len(real_arr), me, seed,
                            C.cast(ptrs, C.c_void_p), out.ctypes.data, sendcount)
    if rc != 0:
        raise ValueError(f"or_allgather rc={rc}")
    return out[: W * sendcount]


def reducescatter(dtype, mode, W, real, me, seed, sends, recvcount):
    keep, ptrs = _ptrs(sends)
    real_arr = np.asarray(sorted(real), dtype=np.uint32)
    out = np.zeros(max(recvcount, 1), dtype=DTYPES[dtype])
    rc = lib().or_reducescatter(dtype, mode, W, real_arr.ctypes.data, len(real_arr), me, seed,
                                C.cast(ptrs, C.c_void_p), out.ctypes.data, recvcount)
    if rc != 0:
        raise ValueError(f"or_reducescatter rc={rc}")
    return out[:recvcount]


def broadcast(dtype, mode, W, real, me, root, seed, root_send, count):
    real_arr = np.asarray(sorted(real), dtype=np.uint32)
    out = np.zeros(max(count, 1), dtype=DTYPES[dtype])
    src = None if root_send is None else np.ascontiguousarray(root_send)
    rc = lib().or_broadcast(dtype, mode, W, real_arr.ctypes.data, len(real_arr), me, root, seed,
                            None if src is None else src.ctypes.data, out.ctypes.data, count)
    if rc != 0:
        raise ValueError(f"or_broadcast rc={rc}")
    return out[:count]


def ring_execute_allreduce(dtype, inputs, me):
    keep, ptrs = _ptrs(inputs)
    count = len(inputs[0])
    out = np.zeros(max(count, 1), dtype=DTYPES[dtype])
    rc = lib().or_ring_execute_allreduce(dtype, len(inputs), C.cast(ptrs, C.c_void_p), count, me,
                                         out.ctypes.data)
    if rc != 0:
        raise ValueError("ring execute: unsupported dtype")
    return out[:count]
