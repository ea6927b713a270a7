"""ctypes binding of libcemu_b200.so (the C-ABI declared in include/cemu_b200.h).

The product path: every collective goes through this library's sm_100a
kernels.  There is no fallback -- if the library is missing, importing the
package raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcemu_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "cemu_b200.h")

# ncclResult_t-valued codes
SUCCESS, UNHANDLED_CUDA, SYSTEM, INTERNAL, INVALID_ARGUMENT, INVALID_USAGE = 0, 1, 2, 3, 4, 5


class CemuError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class UniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


class DelayModel(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("algo", C.c_int32),
        ("alpha_us", C.c_double), ("beta_us_per_byte", C.c_double),
        ("gamma_us_per_byte", C.c_double),
        ("fixed_us", C.c_double), ("inject_us", C.c_double),
        ("gpus_per_node", C.c_uint32),
        ("intra_alpha_us", C.c_double), ("intra_beta_us_per_byte", C.c_double),
    ]


class ShardPlan(C.Structure):
    _fields_ = [("shardOffset", C.c_uint64), ("shardCount", C.c_uint64),
                ("tailOffset", C.c_uint64), ("tailCount", C.c_uint64)]


# int (*)(int coll, uint32 world, uint64 bytes, uint32 k, double* offsets, void* user)
DELAY_MODEL_FN = C.CFUNCTYPE(C.c_int, C.c_int, C.c_uint32, C.c_uint64, C.c_uint32, C.POINTER(C.c_double),
                             C.c_void_p)


class TopoNode(C.Structure):
    _fields_ = [("isReal", C.c_int32), ("nodeClass", C.c_char * 64)]


class TopoEdge(C.Structure):
    _fields_ = [("src", C.c_uint32), ("dst", C.c_uint32), ("alphaUs", C.c_double),
                ("betaUsPerByte", C.c_double), ("gammaUsPerByte", C.c_double)]


class PlanEntry(C.Structure):
    _fields_ = [("coll", C.c_int32), ("bytes", C.c_uint64), ("elemSize", C.c_uint32)]


class CallRecord(C.Structure):
    _fields_ = [
        ("call_id", C.c_uint64), ("coll", C.c_int32), ("delay_active", C.c_int32),
        ("steps", C.c_uint32), ("world", C.c_uint32), ("model_bytes", C.c_uint64),
        ("model_latency_us", C.c_int64), ("t_start_ns", C.c_int64), ("t_end_ns", C.c_int64),
        ("device_latency_us", C.c_int64), ("t_origin_ns", C.c_int64), ("late_ns", C.c_int64),
        ("overshoot_ns", C.c_int64), ("stall_ns", C.c_int64),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built: run `make -C paper_2405_02969_b200` or "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    u32, u64, i64, dbl, vp, cp, sz, i32 = (C.c_uint32, C.c_uint64, C.c_int64, C.c_double, C.c_void_p,
                                           C.c_char_p, C.c_size_t, C.c_int)
    sig = {
        "cemuGetVersion": (i32, [C.POINTER(i32)]),
        "cemuGetUniqueId": (i32, [C.POINTER(UniqueId)]),
        "cemuCommInitRank": (i32, [C.POINTER(vp), i32, UniqueId, i32]),
        "cemuCommInitRankConfig": (i32, [C.POINTER(vp), cp, UniqueId, i32, i32]),
        "cemuCommInitAll": (i32, [vp, i32, vp]),
        "cemuCommDestroy": (i32, [vp]),
        "cemuCommCount": (i32, [vp, C.POINTER(i32)]),
        "cemuCommUserRank": (i32, [vp, C.POINTER(i32)]),
        "cemuCommCuDevice": (i32, [vp, C.POINTER(i32)]),
        "cemuGetErrorString": (cp, [i32]),
        "cemuGetLastError": (cp, [vp]),
        "cemuAllReduce": (i32, [vp, vp, sz, i32, i32, vp, vp]),
        "cemuAllGather": (i32, [vp, vp, sz, i32, vp, vp]),
        "cemuAllReduceHost": (i32, [vp, vp, sz, i32, i32, vp, vp]),
        "cemuCommAttachEmulator": (i32, [vp, vp, sz, i32]),
        "cemuCommDetachEmulator": (i32, [vp]),
        "cemuAllGatherHost": (i32, [vp, vp, sz, i32, vp, vp]),
        "cemuReduceScatter": (i32, [vp, vp, sz, i32, i32, vp, vp]),
        "cemuBroadcast": (i32, [vp, vp, sz, i32, i32, vp, vp]),
        "cemuMemAlloc": (i32, [vp, sz, C.POINTER(vp)]),
        "cemuMemFree": (i32, [vp, vp]),
        "cemuCommRegister": (i32, [vp, vp, sz, C.POINTER(vp)]),
        "cemuCommDeregister": (i32, [vp, vp]),
        "cemuCommSetSynthCache": (i32, [vp, sz, u32]),
        "cemuCommSynthCacheStats": (i32, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(sz)]),
        "cemuCommGetAsyncError": (i32, [vp, C.POINTER(i32)]),
        "cemuGroupStart": (i32, []),
        "cemuGroupEnd": (i32, []),
        "cemuCommLastCallId": (i32, [vp, C.POINTER(u64)]),
        "cemuCommCallRecord": (i32, [vp, u64, C.POINTER(CallRecord), vp, vp, vp, sz]),
        "cemuCommKernelLaunches": (u64, [vp]),
        "cemuCommEventLog": (i32, [vp, u64, cp, sz]),
        "cemuConfigParse": (i32, [cp, C.POINTER(vp), cp, sz]),
        "cemuConfigLoad": (i32, [cp, C.POINTER(vp), cp, sz]),
        "cemuConfigFree": (None, [vp]),
        "cemuConfigRender": (i32, [vp, cp, sz]),
        "cemuConfigDigest": (u64, [vp]),
        "cemuConfigWorldSize": (u32, [vp]),
        "cemuConfigRealRanks": (u32, [vp, vp, sz]),
        "cemuChunkBytes": (u64, [u32, u64, u32, u32]),
        "cemuChunkOffsetBytes": (u64, [u32, u64, u32, u32]),
        "cemuPositions": (u32, [i32, u32]),
        "cemuSendChunkAt": (u32, [i32, u32, u32, u32]),
        "cemuBoundaryDump": (i32, [i32, u32, u64, u32, u32, cp, sz]),
        "cemuToRealCount": (u32, [i32, u32, vp, u32]),
        "cemuModelTotalUs": (dbl, [C.POINTER(DelayModel), i32, u32, u64]),
        "cemuReleaseOffsets": (i32, [C.POINTER(DelayModel), i32, u32, u64, u32, vp]),
        "cemuReleaseFloors": (i32, [C.POINTER(DelayModel), i32, u32, u64, u32, i64, vp]),
        "cemuCallLatencyUs": (i64, [C.POINTER(DelayModel), i32, u32, u64, u32]),
        "cemuPlanShards": (None, [u64, u32, u32, C.POINTER(ShardPlan)]),
        "cemuPayloadKey": (u32, [u64, u32]),
        "cemuPayloadWord": (u32, [u32, u64]),
        "cemuCommSetDelayModel": (i32, [vp, DELAY_MODEL_FN, vp]),
        "cemuCommSetQueueChaining": (i32, [vp, i64]),
        "cemuCommSetDelayFootprint": (i32, [vp, i32, sz]),
        "cemuConfigTopology": (u32, [vp, C.POINTER(TopoNode), C.POINTER(TopoEdge), sz]),
        "cemuRingSuccessor": (u32, [u32, u32]),
        "cemuRingPredecessor": (u32, [u32, u32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


def check(code: int, comm=None) -> None:
    if code != SUCCESS:
        msg = lib.cemuGetLastError(comm).decode() or lib.cemuGetErrorString(code).decode()
        raise CemuError(code, msg)
