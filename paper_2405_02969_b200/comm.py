"""Python host mirror of the reference's collective boundary, over the C-ABI.

Two layers, both thin:

* :class:`Communicator` -- the NCCL-shaped API of include/cemu_b200.h on
  torch CUDA tensors (device memory + streams are the only things torch
  provides here).
* :class:`WorkerSession` -- the reference's own interposition boundary,
  ``cemu::WorkerSession`` (proj/include/cemu/collective.hpp:50-131), with the
  same names, argument meaning and errors: ``allreduce_async(buffer,
  elem_size)`` / ``allgather_async(full, elem_size)`` return a handle,
  ``wait(handle)`` blocks, the optional declared plan is enforced the way
  ``submit`` does (collective.cpp:181-211), and ``elem_size == 4`` sums int32
  lanes while anything else sums bytes (collective.cpp:343-350).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import torch

from . import _capi
from ._capi import CallRecord, CemuError, UniqueId, check, lib

ALLREDUCE, ALLGATHER, REDUCESCATTER, BROADCAST = 0, 1, 2, 3

_TORCH_DT = {
    torch.int8: 0, torch.uint8: 1, torch.int32: 2, torch.int64: 4, torch.float16: 6,
    torch.float32: 7, torch.float64: 8, torch.bfloat16: 9,
}
for _name, _code in (("uint32", 3), ("uint64", 5)):
    if hasattr(torch, _name):
        _TORCH_DT[getattr(torch, _name)] = _code


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _TORCH_DT[dt]
    except KeyError:
        raise CemuError(_capi.INVALID_ARGUMENT, f"unsupported tensor dtype {dt}") from None


class TransportError(RuntimeError):
    """Mirror of cemu::TransportError (proj/include/cemu/transport.hpp:16-20)."""


class JobConfig:
    """Parsed job config (reference key=value format, proj/src/config.cpp)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def parse(cls, text: str) -> "JobConfig":
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = lib.cemuConfigParse(text.encode(), C.byref(h), err, 1024)
        if rc != 0:
            raise CemuError(rc, err.value.decode())
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "JobConfig":
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = lib.cemuConfigLoad(str(path).encode(), C.byref(h), err, 1024)
        if rc != 0:
            raise CemuError(rc, err.value.decode())
        return cls(h)

    def render(self) -> str:
        n = lib.cemuConfigRender(self._h, None, 0)
        buf = C.create_string_buffer(-n)
        lib.cemuConfigRender(self._h, buf, -n)
        return buf.value.decode()

    @property
    def digest(self) -> int:
        return lib.cemuConfigDigest(self._h)

    @property
    def world_size(self) -> int:
        return lib.cemuConfigWorldSize(self._h)

    @property
    def real_ranks(self) -> list[int]:
        n = lib.cemuConfigRealRanks(self._h, None, 0)
        arr = (C.c_uint32 * max(n, 1))()
        lib.cemuConfigRealRanks(self._h, arr, n)
        return list(arr[:n])

    def topology(self):
        """synthesize_global_topology (config.cpp:314-331): (nodes, edges),
        nodes = [(is_real, node_class)], edges = [(src, dst, alpha, beta, gamma)]."""
        n = lib.cemuConfigTopology(self._h, None, None, 0)
        nodes = (_capi.TopoNode * max(n, 1))()
        edges = (_capi.TopoEdge * max(n, 1))()
        lib.cemuConfigTopology(self._h, nodes, edges, n)
        return ([(bool(v.isReal), v.nodeClass.decode()) for v in nodes[:n]],
                [(e.src, e.dst, e.alphaUs, e.betaUsPerByte, e.gammaUsPerByte) for e in edges[:n]])

    def __del__(self):
        if getattr(self, "_h", None):
            lib.cemuConfigFree(self._h)
            self._h = None


def group_start() -> None:
    check(lib.cemuGroupStart())


def group_end() -> None:
    check(lib.cemuGroupEnd())


def get_unique_id() -> bytes:
    uid = UniqueId()
    check(lib.cemuGetUniqueId(C.byref(uid)))
    # raw 128 bytes: reading `uid.internal` would stop at the first NUL
    return C.string_at(C.addressof(uid), C.sizeof(uid))


class _DeviceBuffer:
    """__cuda_array_interface__ view of a cemuMemAlloc allocation."""

    def __init__(self, ptr: int, numel: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


_TYPESTR = {torch.float32: ("<f4", None), torch.int32: ("<i4", None), torch.uint8: ("|u1", None),
            torch.int8: ("|i1", None), torch.float16: ("<f2", None), torch.bfloat16: ("<i2", torch.bfloat16),
            torch.float64: ("<f8", None), torch.int64: ("<i8", None)}


def _stream_ptr(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


class Communicator:
    """One real rank of an emulated world (cemuCommInitRankConfig)."""

    def __init__(self, config_text: str, rank: int, device: int | None = None,
                 unique_id: bytes | None = None):
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        self._h = C.c_void_p()
        uid = UniqueId()
        if unique_id is not None:
            if len(unique_id) != C.sizeof(uid):
                raise CemuError(_capi.INVALID_ARGUMENT, f"unique id must be {C.sizeof(uid)} bytes")
            C.memmove(C.addressof(uid), unique_id, C.sizeof(uid))
        check(lib.cemuCommInitRankConfig(C.byref(self._h), config_text.encode(), uid, rank, device))
        self.config = JobConfig.parse(config_text)
        self.rank = rank
        self.world_size = self.config.world_size

    @classmethod
    def init_all(cls, config_path: str, devices: list[int]) -> list["Communicator"]:
        """cemuCommInitAll (ncclCommInitAll shape): one process, one
        communicator per device, serving the config's real ranks in order.
        Issue their collectives inside group_start()/group_end()."""
        import os
        os.environ["CEMU_CONFIG"] = str(config_path)
        n = len(devices)
        handles = (C.c_void_p * n)()
        devs = (C.c_int * n)(*devices)
        check(lib.cemuCommInitAll(handles, n, devs))
        text = open(config_path).read()
        cfg = JobConfig.parse(text)
        out = []
        for i, (h, r) in enumerate(zip(handles, cfg.real_ranks)):
            c = cls.__new__(cls)
            c.device, c._h, c.config, c.rank, c.world_size = devices[i], C.c_void_p(h), cfg, r, cfg.world_size
            out.append(c)
        return out

    # -- collectives (NCCL argument meaning; out-of-place or in-place) -------
    def all_reduce(self, send: torch.Tensor, recv: torch.Tensor | None = None, stream=None):
        recv = send if recv is None else recv
        self._check_same(send, recv, send.numel())
        check(lib.cemuAllReduce(_ptr(send), _ptr(recv), send.numel(), dtype_code(send.dtype), 0,
                                self._h, _stream_ptr(stream)), self._h)
        return recv

    def all_gather(self, send: torch.Tensor, recv: torch.Tensor, stream=None):
        self._check_same(send, recv, send.numel() * self.world_size)
        check(lib.cemuAllGather(_ptr(send), _ptr(recv), send.numel(), dtype_code(send.dtype),
                                self._h, _stream_ptr(stream)), self._h)
        return recv

    # -- host buffers (WorkerSession's span shape, collective.hpp:68-78) ------
    def all_reduce_host(self, send: torch.Tensor, recv: torch.Tensor | None = None, stream=None):
        """Allreduce of a HOST tensor (pin it for overlapped copies).  Stream-
        ordered: synchronize `stream` before reading `recv`."""
        recv = send if recv is None else recv
        self._check_host(send, recv, send.numel())
        check(lib.cemuAllReduceHost(_ptr(send), _ptr(recv), send.numel(), dtype_code(send.dtype), 0,
                                    self._h, _stream_ptr(stream)), self._h)
        return recv

    def all_gather_host(self, send: torch.Tensor, recv: torch.Tensor, stream=None):
        self._check_host(send, recv, send.numel() * self.world_size)
        check(lib.cemuAllGatherHost(_ptr(send), _ptr(recv), send.numel(), dtype_code(send.dtype),
                                    self._h, _stream_ptr(stream)), self._h)
        return recv

    # -- delay-model plugin (DelayModelFn, proj/include/cemu/delay.hpp:52-55) --
    def set_delay_model(self, fn) -> None:
        """fn(coll, world_size, bytes, k) -> k release offsets (us from the
        call's start), evaluated on the host when each call is enqueued; the
        device applies llround floors and the head-of-line release.  None
        restores the job config's model."""
        if fn is None:
            check(lib.cemuCommSetDelayModel(self._h, _capi.DELAY_MODEL_FN(), None), self._h)
            self._delay_cb = None
            return

        def cb(coll, n, nbytes, k, out, _user):
            try:
                vals = list(fn(coll, n, nbytes, k))
                if len(vals) != k:
                    return 2
                for j, v in enumerate(vals):
                    out[j] = float(v)
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a failed plugin call
                return 1
        self._delay_cb = _capi.DELAY_MODEL_FN(cb)  # kept alive with the communicator
        check(lib.cemuCommSetDelayModel(self._h, self._delay_cb, None), self._h)

    def set_queue_chaining(self, gap_us: int) -> None:
        """cemuCommSetQueueChaining: a delayed call queued within gap_us
        behind the previous delayed call on its stream starts its schedule at
        that call's end (0 = off, the default)."""
        check(lib.cemuCommSetQueueChaining(self._h, int(gap_us)), self._h)

    def set_delay_footprint(self, ctas: int, smem_bytes: int = 0) -> None:
        """cemuCommSetDelayFootprint: every delayed call also holds `ctas`
        CTAs (512 threads, smem_bytes each) until its modelled end -- the SMs
        a real collective's kernel would take from compute beside it."""
        check(lib.cemuCommSetDelayFootprint(self._h, int(ctas), int(smem_bytes)), self._h)

    # -- wire mode (interop with a reference cemu-emulator) -------------------
    def attach_emulator(self, plan: list, timeout_ms: int = 10000) -> None:
        """cemuCommAttachEmulator: dial the config's emulator endpoint and
        handshake with `plan` (CollectivePlanEntry list); all_reduce /
        all_gather then run the CEMU wire protocol, host-synchronously."""
        arr = (_capi.PlanEntry * max(len(plan), 1))()
        for i, e in enumerate(plan):
            arr[i].coll = {"allreduce": 0, "allgather": 1}[e.kind]
            arr[i].bytes = e.bytes
            arr[i].elemSize = e.elem_size
        check(lib.cemuCommAttachEmulator(self._h, arr, len(plan), timeout_ms), self._h)

    def detach_emulator(self) -> None:
        check(lib.cemuCommDetachEmulator(self._h), self._h)

    def _check_host(self, send, recv, recv_numel):
        if send.dtype != recv.dtype:
            raise CemuError(_capi.INVALID_ARGUMENT, "send/recv dtypes differ")
        if recv.numel() != recv_numel:
            raise CemuError(_capi.INVALID_ARGUMENT, f"recv has {recv.numel()} elements, expected {recv_numel}")
        for t in (send, recv):
            if t.is_cuda or not t.is_contiguous():
                raise CemuError(_capi.INVALID_ARGUMENT, "host collectives take contiguous CPU tensors")

    def reduce_scatter(self, send: torch.Tensor, recv: torch.Tensor, stream=None):
        if send.numel() != recv.numel() * self.world_size:
            raise CemuError(_capi.INVALID_ARGUMENT,
                            f"reduce_scatter: send has {send.numel()} elements, expected "
                            f"{recv.numel()} x {self.world_size}")
        self._check_same(send, recv, recv.numel())
        check(lib.cemuReduceScatter(_ptr(send), _ptr(recv), recv.numel(), dtype_code(send.dtype), 0,
                                    self._h, _stream_ptr(stream)), self._h)
        return recv

    def broadcast(self, send: torch.Tensor | None, recv: torch.Tensor, root: int, stream=None):
        check(lib.cemuBroadcast(_ptr(send), _ptr(recv), recv.numel(), dtype_code(recv.dtype), root,
                                self._h, _stream_ptr(stream)), self._h)
        return recv

    def _check_same(self, send, recv, recv_numel):
        if send.dtype != recv.dtype:
            raise CemuError(_capi.INVALID_ARGUMENT, "send/recv dtypes differ")
        if recv.numel() != recv_numel:
            raise CemuError(_capi.INVALID_ARGUMENT,
                            f"recv has {recv.numel()} elements, expected {recv_numel}")
        for t in (send, recv):
            if not t.is_cuda or not t.is_contiguous():
                raise CemuError(_capi.INVALID_ARGUMENT, "buffers must be contiguous CUDA tensors")

    # -- symmetric memory (fused multi-GPU path) -------------------------------
    def alloc(self, numel: int, dtype: torch.dtype) -> torch.Tensor:
        """Tensor in cemuMemAlloc memory (collective across the real ranks).
        Allreduces between such buffers (same offsets on every rank) run as
        one fused kernel over NVLink peer memory."""
        es = torch.empty(0, dtype=dtype).element_size()
        p = C.c_void_p()
        check(lib.cemuMemAlloc(self._h, max(numel * es, 1), C.byref(p)), self._h)
        self._allocs = getattr(self, "_allocs", [])
        self._allocs.append(p.value)
        typestr, view = _TYPESTR[dtype]
        with torch.cuda.device(self.device):
            t = torch.as_tensor(_DeviceBuffer(p.value, numel, typestr), device=f"cuda:{self.device}")
        return t.view(view) if view is not None else t

    def free(self, t: torch.Tensor) -> None:
        ptr = t.data_ptr()
        check(lib.cemuMemFree(self._h, C.c_void_p(ptr)), self._h)
        self._allocs.remove(ptr)

    def register(self, t: torch.Tensor) -> int:
        """cemuCommRegister (ncclCommRegister): collective over the real
        ranks; collectives on registered tensors (same offsets on every rank)
        take the fused kernels.  Returns the handle for deregister()."""
        h = C.c_void_p()
        check(lib.cemuCommRegister(self._h, C.c_void_p(t.data_ptr()), t.numel() * t.element_size(),
                                   C.byref(h)), self._h)
        return h.value or 0

    def deregister(self, handle: int) -> None:
        check(lib.cemuCommDeregister(self._h, C.c_void_p(handle)), self._h)

    # -- synthesis cache -------------------------------------------
    def set_synth_cache(self, cap_bytes: int, min_peers: int = 16) -> None:
        """Bound (0 = off) the per-element cache of the emulated ranks' sums;
        drops every entry."""
        check(lib.cemuCommSetSynthCache(self._h, cap_bytes, min_peers), self._h)

    def synth_cache_stats(self) -> dict:
        f, h, b = C.c_uint64(), C.c_uint64(), C.c_size_t()
        check(lib.cemuCommSynthCacheStats(self._h, C.byref(f), C.byref(h), C.byref(b)), self._h)
        return {"fills": f.value, "hits": h.value, "bytes": b.value}

    def async_error(self) -> str | None:
        e = C.c_int()
        check(lib.cemuCommGetAsyncError(self._h, C.byref(e)), self._h)
        return None if e.value == 0 else lib.cemuGetLastError(self._h).decode()

    # -- observability --------------------------------------------------------
    @property
    def last_call_id(self) -> int:
        v = C.c_uint64()
        check(lib.cemuCommLastCallId(self._h, C.byref(v)), self._h)
        return v.value

    def call_record(self, call_id: int | None = None) -> dict:
        """Per-call schedule record (read after the stream is synchronized)."""
        if call_id is None:
            call_id = self.last_call_id
        rec = CallRecord()
        cap = 1 << 16
        import numpy as np
        floors = np.zeros(cap, dtype=np.int64)
        release = np.zeros(cap, dtype=np.int64)
        offsets = np.zeros(cap, dtype=np.float64)
        check(lib.cemuCommCallRecord(self._h, call_id, C.byref(rec), floors.ctypes.data,
                                     release.ctypes.data, offsets.ctypes.data, cap), self._h)
        k = rec.steps if rec.delay_active else 0
        return {
            "call_id": rec.call_id, "coll": rec.coll, "delay_active": bool(rec.delay_active),
            "steps": rec.steps, "world": rec.world, "model_bytes": rec.model_bytes,
            "model_latency_us": rec.model_latency_us, "t_start_ns": rec.t_start_ns,
            "t_end_ns": rec.t_end_ns, "device_latency_us": rec.device_latency_us,
            "t_origin_ns": rec.t_origin_ns, "late_ns": rec.late_ns, "overshoot_ns": rec.overshoot_ns,
            "stall_ns": rec.stall_ns,
            "floors_us": floors[:k].copy(), "release_ns": release[:k].copy(),
            "offsets_us": offsets[:k].copy(),
        }

    def event_log(self, call_id: int | None = None) -> list[str]:
        """EventLog lines (trace.hpp:10-34) of one delayed call."""
        if call_id is None:
            call_id = self.last_call_id
        n = lib.cemuCommEventLog(self._h, call_id, None, 0)
        if n == -1:
            raise CemuError(_capi.INVALID_USAGE, lib.cemuGetLastError(self._h).decode())
        buf = C.create_string_buffer(-n)
        lib.cemuCommEventLog(self._h, call_id, buf, -n)
        return buf.value.decode().splitlines()

    @property
    def kernel_launches(self) -> int:
        return lib.cemuCommKernelLaunches(self._h)

    def close(self):
        if getattr(self, "_h", None):
            lib.cemuCommDestroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# WorkerSession mirror
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class CollectivePlanEntry:
    """proj/include/cemu/transport.hpp:25-31 (bytes = per-rank block for allgather)."""
    kind: str  # "allreduce" | "allgather"
    bytes: int
    elem_size: int = 1


class CollHandle:
    """Completion handle of one asynchronous call (collective.hpp:22-40)."""

    def __init__(self, event: torch.cuda.Event, issue_us: int, call_id: int):
        self._event = event
        self.issue_us = issue_us
        self.complete_us = 0
        self.call_id = call_id

    def done(self) -> bool:
        return self._event.query()

    def failed(self) -> bool:
        return False


def _now_us() -> int:
    return time.monotonic_ns() // 1000


class WorkerSession:
    """cemu::WorkerSession on the B200 path (one real rank, stream-ordered)."""

    def __init__(self, config_text: str, rank: int, plan: list[CollectivePlanEntry] | None = None,
                 device: int | None = None, unique_id: bytes | None = None, stream=None):
        self.comm = Communicator(config_text, rank, device, unique_id)
        self._rank = rank
        self.plan = list(plan) if plan is not None else None
        self._next_op = 0
        self._closing = False
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.comm.device)

    def rank(self) -> int:
        return self._rank

    def world_size(self) -> int:
        return self.comm.world_size

    @staticmethod
    def _typed(buf: torch.Tensor, elem_size: int) -> torch.Tensor:
        # collective.cpp:343-350: elem_size 4 -> int32 lanes, else bytes; a
        # typed (non-uint8) tensor is taken as is.
        if buf.dtype != torch.uint8:
            return buf
        if elem_size == 4:
            if buf.numel() % 4:
                raise TransportError(f"buffer of {buf.numel()} bytes is not a multiple of elem_size 4")
            return buf.view(torch.int32)
        return buf

    def _submit(self, kind: str, buffer: torch.Tensor, elem_size: int) -> None:
        if self._closing:
            raise TransportError("session is closing")
        nbytes = buffer.numel() * buffer.element_size()
        if self.plan is not None:
            if not self.plan:
                raise TransportError("no collectives were declared for this session")
            e = self.plan[self._next_op % len(self.plan)]
            if e.kind != kind or e.elem_size != elem_size:
                raise TransportError("collective call does not match the declared plan")
            want = e.bytes if kind == "allreduce" else e.bytes * self.comm.world_size
            if nbytes != want:
                raise TransportError(f"buffer size {nbytes} does not match plan entry ({want})")
        if elem_size == 0 or nbytes % elem_size:
            raise TransportError(f"payload size {nbytes} is not a multiple of elem_size {elem_size}")
        self._next_op += 1

    def _handle(self, issue_us: int) -> CollHandle:
        ev = torch.cuda.Event()
        ev.record(self.stream)
        return CollHandle(ev, issue_us, self.comm.last_call_id)

    def allreduce_async(self, buffer: torch.Tensor, elem_size: int) -> CollHandle:
        issue = _now_us()
        self._submit("allreduce", buffer, elem_size)
        t = self._typed(buffer, elem_size)
        if t.is_cuda:
            self.comm.all_reduce(t, t, stream=self.stream)
        else:  # a host span, as the reference's (cemuAllReduceHost)
            self.comm.all_reduce_host(t, t, stream=self.stream)
        return self._handle(issue)

    def allgather_async(self, full: torch.Tensor, elem_size: int) -> CollHandle:
        issue = _now_us()
        self._submit("allgather", full, elem_size)
        t = self._typed(full, elem_size)
        block = t.numel() // self.comm.world_size
        if block * self.comm.world_size != t.numel():
            raise TransportError("allgather buffer is not world_size blocks")
        own = t[self._rank * block:(self._rank + 1) * block]
        if t.is_cuda:
            self.comm.all_gather(own, t, stream=self.stream)
        else:
            self.comm.all_gather_host(own, t, stream=self.stream)
        return self._handle(issue)

    def wait(self, h: CollHandle) -> None:
        if h is None:
            raise ValueError("wait on null collective handle")
        h._event.synchronize()
        if not h.complete_us:
            h.complete_us = _now_us()

    def allreduce(self, buffer: torch.Tensor, elem_size: int) -> None:
        self.wait(self.allreduce_async(buffer, elem_size))

    def allgather(self, full: torch.Tensor, elem_size: int) -> None:
        self.wait(self.allgather_async(full, elem_size))

    def close(self) -> None:
        if self._closing:
            return
        self._closing = True
        torch.cuda.synchronize(self.comm.device)
        self.comm.close()
