"""paper_2405_02969_b200 -- B200-native collective emulation (NeuronaBox hot path).

A collective call whose world contains emulated remote ranks: the emulated
peers' payloads are synthesised on the GPU from a counter-based hash and
reduced with the local buffer in one HBM pass (sm_100a kernels), the real
part among local GPUs runs over NCCL/NVLink, and the alpha-beta network delay
is evaluated on the device and injected by a %globaltimer spin kernel on the
collective's stream.  See DESIGN.md.

The compute path is libcemu_b200.so (C-ABI: include/cemu_b200.h).  Importing
this package without it raises -- there is no CPU fallback.
"""
from ._capi import CemuError, lib  # noqa: F401  (loads libcemu_b200.so or raises)
from .comm import (  # noqa: F401
    ALLGATHER, ALLREDUCE, BROADCAST, REDUCESCATTER, CollectivePlanEntry, CollHandle, Communicator,
    JobConfig, TransportError, WorkerSession, dtype_code, get_unique_id, group_end, group_start,
)
from . import schedule  # noqa: F401

__all__ = [
    "CemuError", "Communicator", "WorkerSession", "JobConfig", "CollectivePlanEntry", "CollHandle",
    "TransportError", "get_unique_id", "dtype_code", "schedule",
]
