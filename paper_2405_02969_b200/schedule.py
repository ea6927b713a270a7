"""Python view of the host-side schedule / delay-model C-ABI (cemu_b200.h)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._capi import DelayModel, ShardPlan, lib

ALLREDUCE, ALLGATHER, REDUCESCATTER, BROADCAST = 0, 1, 2, 3
NONE, ALPHA_BETA, FIXED = 0, 1, 2
RING, TREE, HIERARCHICAL = 0, 1, 2


def delay_model(kind=NONE, algo=RING, alpha=0.0, beta=0.0, gamma=0.0, fixed=0.0, inject=0.0,
                gpus_per_node=1, intra_alpha=None, intra_beta=None) -> DelayModel:
    return DelayModel(kind, algo, alpha, beta, gamma, fixed, inject, gpus_per_node,
                      alpha if intra_alpha is None else intra_alpha,
                      beta if intra_beta is None else intra_beta)


def chunk_bytes(n, total, elem, c):
    return lib.cemuChunkBytes(n, total, elem, c)


def chunk_offset_bytes(n, total, elem, c):
    return lib.cemuChunkOffsetBytes(n, total, elem, c)


def positions(coll, n):
    return lib.cemuPositions(coll, n)


def send_chunk_at(coll, n, rank, p):
    return lib.cemuSendChunkAt(coll, n, rank, p)


def boundary_dump(coll, n, nbytes, elem=1, real=0) -> str:
    need = -lib.cemuBoundaryDump(coll, n, nbytes, elem, real, None, 0)
    buf = C.create_string_buffer(need)
    lib.cemuBoundaryDump(coll, n, nbytes, elem, real, buf, need)
    return buf.value.decode()


def to_real_count(coll, n, real) -> int:
    arr = np.asarray(sorted(real), dtype=np.uint32)
    return lib.cemuToRealCount(coll, n, arr.ctypes.data, len(arr))


def model_total_us(m, coll, n, nbytes) -> float:
    return lib.cemuModelTotalUs(C.byref(m), coll, n, nbytes)


def release_offsets(m, coll, n, nbytes, k):
    out = np.zeros(max(k, 1), dtype=np.float64)
    lib.cemuReleaseOffsets(C.byref(m), coll, n, nbytes, k, out.ctypes.data)
    return out[:k]


def release_floors(m, coll, n, nbytes, k, now_us=0):
    out = np.zeros(max(k, 1), dtype=np.int64)
    lib.cemuReleaseFloors(C.byref(m), coll, n, nbytes, k, now_us, out.ctypes.data)
    return out[:k]


def call_latency_us(m, coll, n, nbytes, k) -> int:
    return lib.cemuCallLatencyUs(C.byref(m), coll, n, nbytes, k)


def payload_key(seed, rank) -> int:
    return lib.cemuPayloadKey(seed, rank)


def payload_word(key, j) -> int:
    return lib.cemuPayloadWord(key, j)


def plan_shards(count, k, li) -> dict:
    """Which elements real GPU `li` of `k` owns in a multi-GPU allreduce."""
    p = ShardPlan()
    lib.cemuPlanShards(count, k, li, C.byref(p))
    return {"shard": (p.shardOffset, p.shardCount), "tail": (p.tailOffset, p.tailCount)}
