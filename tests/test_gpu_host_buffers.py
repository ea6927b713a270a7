"""Host-buffer collectives (cemuAllReduceHost / cemuAllGatherHost).

The reference's boundary, WorkerSession, takes host spans
(proj/include/cemu/collective.hpp:68-78) and returns when `wait` does; the
host forms keep that shape, stream-ordered.  With one real GPU the buffer is
pipelined through the device in chunks (H2D / synthesis / D2H on three
streams over four rotating device buffers): the tests force 1 MiB chunks so
that buffers rotate many times, and check every byte against the oracle --
pinned and pageable memory, in and out of place, ragged sizes, every
datatype, the staged zero-payload path, delay injection and graph capture.
"""
from __future__ import annotations

import os
import time

import pytest
import torch

import paper_2405_02969_b200 as pb
from gpu_util import TORCH, assert_bit_equal, config, host_input, to_np
from oracle import port as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small_chunks(cuda):
    old = os.environ.get("CEMU_HOST_CHUNK_MIB")
    os.environ["CEMU_HOST_CHUNK_MIB"] = "1"  # read when a communicator first builds its pipe
    yield
    if old is None:
        os.environ.pop("CEMU_HOST_CHUNK_MIB", None)
    else:
        os.environ["CEMU_HOST_CHUNK_MIB"] = old


def _sync():
    torch.cuda.current_stream().synchronize()


@pytest.mark.parametrize("pinned", [True, False])
def test_allreduce_host_rotating_chunks_bit_exact(small_chunks, pinned):
    comm = pb.Communicator(config(8), 0, 0)
    for dt in (7, 9, 1, 2, 4):
        es = torch.empty(0, dtype=TORCH[dt]).element_size()
        count = (5 << 20) // es * 2 + 12345  # ~10 MiB: ten 1 MiB chunks, ragged tail
        h = host_input(dt, count, seed=dt)
        src = h.pin_memory() if pinned else h.clone()
        out = torch.empty_like(src).pin_memory() if pinned else torch.empty_like(src)
        comm.all_reduce_host(src, out)
        _sync()
        want = P.allreduce(dt, P.PAYLOAD_HASH, 8, [0], 0, 1, [to_np(h)], count)
        assert_bit_equal(to_np(out), want, f"host allreduce dt={dt} pinned={pinned}")
        assert torch.equal(src, h)  # out of place: send untouched
    comm.close()


def test_allreduce_host_in_place_small_and_many_peers(small_chunks):
    for W in (2, 64, 300):
        comm = pb.Communicator(config(W), 0, 0)
        for count in (1, 5, 4099, (1 << 20) + 7):
            h = host_input(7, count, seed=W + count)
            buf = h.pin_memory()
            comm.all_reduce_host(buf)
            _sync()
            want = P.allreduce(7, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(h)], count)
            assert_bit_equal(to_np(buf), want, f"in place W={W} n={count}")
        comm.close()


def test_allreduce_host_equals_device_call(small_chunks):
    comm = pb.Communicator(config(16, seed=77), 0, 0)
    h = host_input(9, 3 << 20, seed=9)
    d_out = torch.empty_like(h, device="cuda")
    comm.all_reduce(h.cuda(), d_out)
    out = torch.empty_like(h).pin_memory()
    comm.all_reduce_host(h.pin_memory(), out)
    _sync()
    assert torch.equal(out.view(torch.int16), d_out.cpu().view(torch.int16))
    comm.close()


@pytest.mark.parametrize("in_place", [True, False])
def test_allgather_host(small_chunks, in_place):
    W = 8
    comm = pb.Communicator(config(W, real=(3,)), 3, 0)
    for dt in (7, 9, 1):
        sc = (300 << 10) + 3
        h = host_input(dt, sc, seed=dt)
        recv = torch.zeros(sc * W, dtype=h.dtype).pin_memory()
        if in_place:
            recv[3 * sc:4 * sc] = h
            send = recv[3 * sc:4 * sc]
        else:
            send = h.pin_memory()
        comm.all_gather_host(send, recv)
        _sync()
        want = P.allgather(dt, P.PAYLOAD_HASH, W, [3], 3, 1, [to_np(h)], sc)
        assert_bit_equal(to_np(recv), want, f"host allgather dt={dt} in_place={in_place}")
    comm.close()


def test_zero_payload_host_path_reproduces_reference_emulator(small_chunks):
    comm = pb.Communicator(config(4, mode="zero"), 0, 0)
    h = host_input(2, 4096 + 4, seed=4)
    out = torch.empty_like(h)
    comm.all_reduce_host(h, out)
    _sync()
    want = P.allreduce(2, P.PAYLOAD_ZERO, 4, [0], 0, 1, [to_np(h)], h.numel())
    assert_bit_equal(to_np(out), want, "zero mode host allreduce")
    comm.close()


def test_host_call_carries_the_injected_delay(small_chunks):
    comm = pb.Communicator(config(8, extra="delay.inject_us = 20000\n"), 0, 0)
    h = host_input(7, 1 << 20, seed=1).pin_memory()
    out = torch.empty_like(h).pin_memory()
    comm.all_reduce_host(h, out)  # warm
    _sync()
    t0 = time.perf_counter()
    comm.all_reduce_host(h, out)
    _sync()
    dt = time.perf_counter() - t0
    assert dt >= 0.0199, dt
    rec = comm.call_record()
    assert rec["model_latency_us"] == 20000
    assert rec["t_end_ns"] - rec["t_start_ns"] >= 20_000_000  # released on the device clock
    want = P.allreduce(7, P.PAYLOAD_HASH, 8, [0], 0, 1, [to_np(h)], h.numel())
    assert_bit_equal(to_np(out), want, "delayed host allreduce")
    comm.close()


def test_host_allreduce_graph_capture(small_chunks):
    comm = pb.Communicator(config(8), 0, 0)
    h = host_input(7, (3 << 20) // 4 + 5, seed=2)
    src = h.pin_memory()
    out = torch.empty_like(h).pin_memory()
    comm.all_reduce_host(src, out)  # builds the pipe outside capture
    _sync()
    out.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        comm.all_reduce_host(src, out)
    for _ in range(2):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        want = P.allreduce(7, P.PAYLOAD_HASH, 8, [0], 0, 1, [to_np(h)], h.numel())
        assert_bit_equal(to_np(out), want, "graph-replayed host allreduce")
    comm.close()


def test_host_usage_errors(cuda):
    comm = pb.Communicator(config(4), 0, 0)
    with pytest.raises(pb.CemuError, match="CPU tensors"):
        comm.all_reduce_host(torch.zeros(4, device="cuda"))
    from paper_2405_02969_b200._capi import lib
    x = torch.zeros(16)
    assert lib.cemuGroupStart() == 0
    r = lib.cemuAllReduceHost(x.data_ptr(), x.data_ptr(), 16, 7, 0, comm._h, None)
    assert lib.cemuGroupEnd() == 0
    assert r == 5 and b"cannot be grouped" in lib.cemuGetLastError(None)
    comm.close()


def test_worker_session_mirror_takes_host_spans(small_chunks):
    """pb.WorkerSession with CPU tensors = the reference's host-span calls
    (allreduce_async(span, elem_size) + wait), through the host C-ABI."""
    W = 4
    plan = [pb.CollectivePlanEntry("allreduce", 4 * 4099, 4), pb.CollectivePlanEntry("allgather", 1000, 1)]
    s = pb.WorkerSession(config(W), 0, plan)
    h = host_input(2, 4099, seed=11)
    buf = h.clone().view(torch.uint8)
    s.wait(s.allreduce_async(buf, 4))
    want = P.allreduce(2, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(h)], 4099)
    assert_bit_equal(buf.view(torch.int32).numpy(), want, "session allreduce (host span)")
    full = torch.zeros(1000 * W, dtype=torch.uint8)
    own = host_input(1, 1000, seed=12)
    full[:1000] = own
    s.allgather(full, 1)
    want = P.allgather(1, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(own)], 1000)
    assert_bit_equal(full.numpy(), want, "session allgather (host span)")
    s.close()
