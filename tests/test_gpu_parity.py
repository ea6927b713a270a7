"""GPU parity: the sm_100a path through the C-ABI against the CPU oracle.

Bit-exact for every datatype (integer, byte and float alike: the float fold
is defined as one rounding of local + an exact dyadic sum, so the oracle
reproduces it exactly; the north star's 1e-6 / 1e-2 tolerances are asserted
against the ring-order fold in test_oracle.py and below).  Sizes are such
that the oracle finishes in seconds; full-size runs are checked through
size-independent properties (sampled windows, linearity, idempotence).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2405_02969_b200 as pb
from conftest import golden
from gpu_util import FLOATS, TORCH, assert_bit_equal, config, host_input, oracle_mode, to_np
from oracle import port as P

pytestmark = pytest.mark.gpu

DTYPES = [7, 9, 6, 2, 1, 0, 4, 8]
COUNTS = [1, 3, 17, 1000, 4096 + 7, 65536 + 3]


@pytest.fixture(scope="module")
def comms(cuda):
    cache = {}

    def get(W, mode="hash", seed=1, real=(0,), rank=0):
        key = (W, mode, seed, real, rank)
        if key not in cache:
            cache[key] = pb.Communicator(config(W, real, mode, seed), rank, 0)
        return cache[key]
    yield get
    for c in cache.values():
        c.close()


def _allreduce(comm, h, inplace):
    d = h.cuda()
    r = d if inplace else torch.empty_like(d)
    comm.all_reduce(d, r)
    torch.cuda.synchronize()
    return to_np(r)


@pytest.mark.parametrize("W", [2, 8, 64])
@pytest.mark.parametrize("dt", DTYPES)
def test_allreduce_hash_bit_exact(comms, W, dt):
    comm = comms(W)
    for i, count in enumerate(COUNTS):
        h = host_input(dt, count, seed=count + dt)
        want = P.allreduce(dt, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(h)], count)
        assert_bit_equal(_allreduce(comm, h, inplace=bool(i % 2)), want, f"allreduce W={W} dt={dt} n={count}")


@pytest.mark.parametrize("W", [257, 1024])
def test_allreduce_many_peers_grouped_lanes(comms, W):
    """> 256 emulated peers: 16-bit SWAR lanes are flushed per 256-peer group."""
    comm = comms(W)
    for dt in (7, 9, 1, 2):
        count = 2048 + 5
        h = host_input(dt, count, seed=W + dt)
        want = P.allreduce(dt, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(h)], count)
        assert_bit_equal(_allreduce(comm, h, inplace=False), want, f"W={W} dt={dt}")


def _special_values(dt: int, count: int, seed: int, W: int) -> torch.Tensor:
    """IEEE edge cases scattered over a random buffer: signed zeros, infs,
    NaN, subnormals at both ends, the largest finite values (the fold may
    overflow to inf) and halfway cases for the final rounding."""
    h = host_input(dt, count, seed=seed)
    fi = torch.finfo(TORCH[dt])
    sub = fi.smallest_normal * fi.eps  # smallest subnormal
    specials = [0.0, -0.0, float("inf"), float("-inf"), float("nan"), sub, -sub, fi.smallest_normal - sub,
                -(fi.smallest_normal - sub), fi.smallest_normal, fi.max, -fi.max, fi.max * 0.999, 1.0 + fi.eps / 2,
                0.5 * fi.eps, 2.0 ** -7, -(2.0 ** -8), 3.0 * 2 ** -9]
    g = torch.Generator().manual_seed(seed)
    pos = torch.randperm(count, generator=g)[: 40 * len(specials)]
    vals = torch.tensor(specials * 40, dtype=torch.float64).to(TORCH[dt])
    h[pos] = vals
    # where the emulated sum is exactly 0 the fold must return x itself:
    # put subnormals there (a flush-to-zero add would show up)
    zeros = torch.zeros(count, dtype=TORCH[dt])
    d = P.allreduce(dt, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(zeros)], count)
    s0 = np.nonzero(np.ascontiguousarray(d).view(np.uint8).reshape(count, -1).max(axis=1) == 0)[0]
    tiny = torch.tensor([sub, -sub, fi.smallest_normal - sub, 3 * sub, -0.0], dtype=torch.float64).to(TORCH[dt])
    h[torch.from_numpy(s0)] = tiny[torch.arange(len(s0)) % len(tiny)]
    return h


@pytest.mark.parametrize("W", [2, 8, 300])
@pytest.mark.parametrize("dt", [7, 9, 6])
def test_float_fold_ieee_edge_cases(comms, W, dt):
    """The fold is one fp32 rounding of x + S * 2^-7 then one rounding to the
    element type; the vector kernel computes S * 2^-7 by a magic-number
    conversion and the add with sm_100 packed / mixed-precision adds, so the
    edge cases are checked bit for bit (NaN positions by mask: NaN payload
    bits are not part of the contract)."""
    comm = comms(W)
    count = 16384 + 8
    h = _special_values(dt, count, seed=W * 10 + dt, W=W)
    want = P.allreduce(dt, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(h)], count)
    got = _allreduce(comm, h, inplace=False)
    tdt = TORCH[dt]
    gt = torch.from_numpy(got.view(np.int16) if dt in (6, 9) else got).view(tdt).double().numpy()
    wt = torch.from_numpy(want.view(np.int16) if dt in (6, 9) else want).view(tdt).double().numpy()
    assert np.array_equal(np.isnan(gt), np.isnan(wt)), "NaN positions differ"
    keep = ~np.isnan(wt)
    assert_bit_equal(got[keep], want[keep], f"edge cases W={W} dt={dt}")


@pytest.mark.parametrize("W", [4097, 20000])
def test_very_large_emulated_worlds(comms, W):
    """Beyond 6143 emulated peers the key table needs > 48 KB of shared
    memory (opted into per kernel); allreduce and allgather stay bit-exact."""
    comm = comms(W)
    for dt in (7, 9, 2):
        count = 1000 + 3
        h = host_input(dt, count, seed=W + dt)
        want = P.allreduce(dt, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(h)], count)
        assert_bit_equal(_allreduce(comm, h, inplace=False), want, f"W={W} dt={dt}")
    sc = 40
    h = host_input(7, sc, seed=1)
    recv = torch.empty(sc * W, dtype=torch.float32, device="cuda")
    comm.all_gather(h.cuda(), recv)
    torch.cuda.synchronize()
    want = P.allgather(7, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(h)], sc)
    assert_bit_equal(to_np(recv), want, f"allgather W={W}")


def test_world_beyond_the_key_table_fails_at_init(cuda):
    with pytest.raises(pb.CemuError, match="emulated ranks exceed"):
        pb.Communicator(config(30000), 0, 0)


def test_real_rank_not_zero_and_other_seed(comms):
    comm = comms(16, seed=0xBEEF, real=(5,), rank=5)
    for dt in (7, 2):
        h = host_input(dt, 5000, seed=3)
        want = P.allreduce(dt, P.PAYLOAD_HASH, 16, [5], 5, 0xBEEF, [to_np(h)], 5000)
        assert_bit_equal(_allreduce(comm, h, False), want, f"rank5 dt={dt}")


def test_misaligned_buffers_take_the_scalar_path(comms):
    comm = comms(8)
    for dt in (7, 9, 1, 2):
        count = 3001
        big = host_input(dt, count + 3, seed=dt).cuda()
        src = big[1:1 + count]            # not 16-byte aligned
        out = torch.empty(count + 2, dtype=big.dtype, device="cuda")[1:1 + count]
        comm.all_reduce(src, out)
        torch.cuda.synchronize()
        want = P.allreduce(dt, P.PAYLOAD_HASH, 8, [0], 0, 1, [to_np(src)], count)
        assert_bit_equal(to_np(out), want, f"misaligned dt={dt}")


def test_count_zero_is_a_noop(comms):
    comm = comms(8)
    x = torch.empty(0, device="cuda")
    comm.all_reduce(x, x)
    torch.cuda.synchronize()


@pytest.mark.parametrize("mode", ["hash", "zero"])
@pytest.mark.parametrize("W", [2, 5, 64])
def test_allgather(comms, mode, W):
    comm = comms(W, mode)
    for dt in (7, 9, 1, 2, 8):
        for count in (1, 33, 1024, 4099):
            h = host_input(dt, count, seed=count)
            want = P.allgather(dt, oracle_mode(mode), W, [0], 0, 1, [to_np(h)], count)
            recv = torch.full((W * count,), 3, dtype=TORCH[dt], device="cuda")
            comm.all_gather(h.cuda(), recv)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(recv), want, f"allgather {mode} W={W} dt={dt} n={count}")
            # in place: own block already at rank * count
            full = torch.zeros(W * count, dtype=TORCH[dt], device="cuda")
            full[:count] = h.cuda()
            comm.all_gather(full[:count], full)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(full), want, f"allgather in-place {mode} W={W} dt={dt}")


@pytest.mark.parametrize("mode", ["hash", "zero"])
def test_reduce_scatter(comms, mode):
    for W, rank in ((4, 0), (8, 3), (64, 63)):
        comm = comms(W, mode, real=(rank,), rank=rank)
        for dt in (7, 9, 2, 1):
            for rc in (1, 100, 4096):
                h = host_input(dt, rc * W, seed=rc + W)
                want = P.reducescatter(dt, oracle_mode(mode), W, [rank], rank, 1, [to_np(h)], rc)
                recv = torch.empty(rc, dtype=TORCH[dt], device="cuda")
                comm.reduce_scatter(h.cuda(), recv)
                torch.cuda.synchronize()
                assert_bit_equal(to_np(recv), want, f"rs {mode} W={W} dt={dt} rc={rc}")


@pytest.mark.parametrize("mode", ["hash", "zero"])
def test_broadcast(comms, mode):
    W = 8
    comm = comms(W, mode)
    for dt in (7, 9, 2, 1):
        for root in (0, 3, 7):
            h = host_input(dt, 1003, seed=root)
            want = P.broadcast(dt, oracle_mode(mode), W, [0], 0, root, 1, to_np(h) if root == 0 else None, 1003)
            recv = torch.empty(1003, dtype=TORCH[dt], device="cuda")
            comm.broadcast(h.cuda() if root == 0 else None, recv, root)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(recv), want, f"bcast {mode} root={root} dt={dt}")


def test_zero_mode_reproduces_reference_emulator(comms):
    """Outputs of the reference's own WorkerSession + EmulatorServer
    (tests/golden/emulated_zero.json), including the n=2 KAT
    {0,0,0,0,5,6,7,8} of test_transport.cpp:129-144."""
    g = golden("emulated_zero.json")
    for c in g["allreduce"]:
        comm = comms(c["n"], "zero")
        dt = torch.int32 if c["elem"] == 4 else torch.uint8
        x = torch.tensor(c["input"], dtype=dt, device="cuda")
        comm.all_reduce(x, x)
        torch.cuda.synchronize()
        assert x.cpu().tolist() == c["output"], (c["n"], c["elem"])
    for c in g["allgather"]:
        comm = comms(c["n"], "zero")
        dt = torch.int32 if c["elem"] == 4 else torch.uint8
        full = torch.tensor(c["input"], dtype=dt, device="cuda")
        block = full.numel() // c["n"]
        comm.all_gather(full[:block], full)
        torch.cuda.synchronize()
        assert full.cpu().tolist() == c["output"]


def test_integer_hash_equals_reference_real_ring(comms):
    """The emulated integer allreduce/allgather equal the reference's
    all-real TCP ring run with every rank holding its hash payload."""
    g = golden("real_ring_hash.json")
    for c in g["allreduce"]:
        comm = comms(c["n"], "hash", c["seed"])
        mine = torch.from_numpy(P.payload(c["dtype"], P.payload_key(c["seed"], 0), 0, c["count"]).copy()).cuda()
        comm.all_reduce(mine, mine)
        torch.cuda.synchronize()
        got = mine.cpu().numpy()
        assert got.tolist() == c["output"], (c["n"], c["dtype"], c["count"])
    for c in g["allgather"]:
        comm = comms(c["n"], "hash", c["seed"])
        mine = torch.from_numpy(P.payload(c["dtype"], P.payload_key(c["seed"], 0), 0, c["block"]).copy()).cuda()
        recv = torch.empty(c["block"] * c["n"], dtype=mine.dtype, device="cuda")
        comm.all_gather(mine, recv)
        torch.cuda.synchronize()
        assert recv.cpu().numpy().tolist() == c["output"]


def test_float_tolerances_vs_ring_order_fold(comms):
    """North-star tolerances (fp32 1e-6 relative, bf16 1e-2) against an fp32
    ring executed in the reference's fold order (oracles.hpp:43-101)."""
    W, count = 8, 8192
    comm = comms(W)
    h = host_input(7, count, seed=9)
    got = _allreduce(comm, h, False).astype(np.float64)
    peers = [to_np(h)] + [P.payload(7, P.payload_key(1, r), 0, count) for r in range(1, W)]
    ring = P.ring_execute_allreduce(7, peers, 0).astype(np.float64)
    assert np.max(np.abs(got - ring) / np.maximum(np.abs(ring), 1.0)) <= 1e-6
    hb = h.to(torch.bfloat16)
    gotb = _allreduce(comm, hb, False)
    gotb = torch.from_numpy(gotb.view(np.int16)).view(torch.bfloat16).double().numpy()
    peersb = [hb.float().numpy()] + peers[1:]
    ringb = P.ring_execute_allreduce(7, peersb, 0).astype(np.float64)
    assert np.max(np.abs(gotb - ringb) / np.maximum(np.abs(ringb), 1.0)) <= 1e-2


# ---- full-size properties ------------------------------------------------------
@pytest.mark.parametrize("dt", [7, 9, 2])
def test_full_size_sampled_windows_and_linearity(comms, dt):
    """1 GiB allreduce at world 8: sampled windows (head, middle, tail,
    random) equal the oracle bit for bit; fold(x) - fold(0) == x for dyadic
    x (exact) -- a size-independent linearity check of every element."""
    W = 8
    comm = comms(W)
    es = torch.empty(0, dtype=TORCH[dt]).element_size()
    count = (1 << 30) // es
    gen = torch.Generator(device="cuda").manual_seed(1)
    if dt in FLOATS:
        x = (torch.randint(-128, 128, (count,), device="cuda", generator=gen).to(torch.float32) / 128).to(TORCH[dt])
    else:
        x = torch.randint(-2**31, 2**31, (count,), device="cuda", generator=gen, dtype=torch.int64).to(TORCH[dt])
    y = torch.empty_like(x)
    comm.all_reduce(x, y)
    zero = torch.zeros_like(x)
    comm.all_reduce(zero, zero)  # in place: zero <- V
    torch.cuda.synchronize()
    rng = np.random.default_rng(dt)
    starts = [0, count // 2 - 37, count - 4099] + [int(s) for s in rng.integers(0, count - 4096, 5)]
    for s in starts:
        win = slice(s, s + 4096)
        # oracle payload windows start at element s
        keys = [P.payload_key(1, r) for r in range(1, W)]
        vs = sum(P.payload(7 if dt in FLOATS else dt, k, s, 4096).astype(np.float64 if dt in FLOATS else np.uint32)
                 for k in keys)
        if dt in FLOATS:
            xs = to_np(x[win])
            xf = xs.astype(np.float32) if dt == 7 else \
                torch.from_numpy(xs.view(np.int16)).view(torch.bfloat16).float().numpy()
            want_f = (xf.astype(np.float64) + vs).astype(np.float32)
            want = want_f if dt == 7 else to_np(torch.from_numpy(want_f).to(torch.bfloat16))
        else:
            want = (to_np(x[win]).view(np.uint32) + vs.astype(np.uint32)).view(np.int32)
        assert_bit_equal(to_np(y[win]), want, f"window {s}")
    if dt == 7:  # x + V is exact in fp32 for dyadic x: every element checked
        assert torch.equal(y - zero, x)
    elif dt == 2:  # wrapping int32 is exactly linear
        assert torch.equal(y - zero, x)


@pytest.mark.parametrize("dt", [1, 2])
def test_payload_word_index_past_2_32(comms, dt):
    """Maximum sizes: a 16 GiB buffer whose payload word index crosses 2^32
    (u8: element 2^34; int32: element 2^32), where the hot kernel's per-tile
    counters take the general (high-word) form.  Windows at the crossing and
    at both ends equal the oracle bit for bit."""
    W = 8
    comm = comms(W)
    cross = 1 << 34 if dt == 1 else 1 << 32  # first element of payload word 2^32
    count = cross + (1 << 20) + 5
    x = torch.zeros(count, dtype=TORCH[dt], device="cuda")
    comm.all_reduce(x, x)  # in place: x <- the emulated peers' sum
    torch.cuda.synchronize()
    keys = [P.payload_key(1, r) for r in range(1, W)]
    for s in (0, cross - 5000, cross - 3, count - 4099):
        n = 8192 if s == cross - 5000 else 4096
        n = min(n, count - s)
        vs = sum(P.payload(dt, k, s, n).astype(np.uint64) for k in keys)
        want = (vs % (256 if dt == 1 else 1 << 32)).astype(np.uint8 if dt == 1 else np.uint32)
        got = to_np(x[s:s + n])
        assert_bit_equal(got.view(want.dtype), want, f"window {s} (crossing at {cross})")
    del x
    torch.cuda.empty_cache()


# ---- the reference-facing WorkerSession mirror -------------------------------
def test_worker_session_mirror_reference_transport_cases(cuda):
    """test_transport.cpp:129-182 through the WorkerSession mirror (zero mode)."""
    s = pb.WorkerSession(config(2, mode="zero"), 0, [pb.CollectivePlanEntry("allreduce", 32, 4)])
    buf = torch.tensor([1, 2, 3, 4, 5, 6, 7, 8], dtype=torch.int32, device="cuda").view(torch.uint8)
    s.allreduce(buf, 4)
    assert buf.view(torch.int32).cpu().tolist() == [0, 0, 0, 0, 5, 6, 7, 8]
    s.close()
    s = pb.WorkerSession(config(4, mode="zero"), 0, [pb.CollectivePlanEntry("allreduce", 64, 4)])
    buf = (torch.arange(16, dtype=torch.int32, device="cuda") + 100).view(torch.uint8)
    s.allreduce(buf, 4)
    v = buf.view(torch.int32).cpu().tolist()
    assert v == [0] * 4 + [104, 105, 106, 107] + [0] * 8
    s.close()
    s = pb.WorkerSession(config(3, mode="zero"), 0, [pb.CollectivePlanEntry("allgather", 16, 4)])
    full = torch.full((12,), -1, dtype=torch.int32, device="cuda")
    full[:4] = torch.arange(7, 11, dtype=torch.int32, device="cuda")
    s.allgather(full.view(torch.uint8), 4)
    assert full.cpu().tolist() == [7, 8, 9, 10] + [0] * 8
    s.close()


def test_worker_session_plan_and_handle_semantics(cuda):
    s = pb.WorkerSession(config(2), 0, [pb.CollectivePlanEntry("allreduce", 64, 1)])
    b1 = torch.ones(64, dtype=torch.uint8, device="cuda")
    b2 = torch.full((64,), 2, dtype=torch.uint8, device="cuda")
    h1 = s.allreduce_async(b1, 1)
    h2 = s.allreduce_async(b2, 1)
    s.wait(h2)  # reverse order (test_transport.cpp:199-216)
    s.wait(h1)
    s.wait(h1)
    assert h1.done() and h2.done()
    with pytest.raises(ValueError):
        s.wait(None)
    with pytest.raises(pb.TransportError, match="does not match the declared plan"):
        s.allgather_async(torch.zeros(128, dtype=torch.uint8, device="cuda"), 1)
    with pytest.raises(pb.TransportError, match="buffer size 32 does not match plan entry"):
        s.allreduce_async(torch.zeros(32, dtype=torch.uint8, device="cuda"), 1)
    s.close()
    with pytest.raises(pb.TransportError, match="closing"):
        s.allreduce_async(b1, 1)


def test_usage_errors_are_loud(cuda):
    comm = pb.Communicator(config(4), 0, 0)
    x = torch.zeros(16, device="cuda")
    import ctypes as C
    from paper_2405_02969_b200._capi import lib
    s = torch.cuda.current_stream().cuda_stream
    assert lib.cemuAllReduce(x.data_ptr(), x.data_ptr(), 16, 7, 2, comm._h, s) == 4  # op max
    assert b"cemuSum" in lib.cemuGetLastError(None)
    assert lib.cemuAllReduce(x.data_ptr(), x.data_ptr(), 16, 42, 0, comm._h, s) == 4  # dtype
    assert lib.cemuBroadcast(x.data_ptr(), x.data_ptr(), 16, 7, 9, comm._h, s) == 4  # root
    assert lib.cemuAllReduce(None, None, 16, 7, 0, comm._h, s) == 4
    h = C.c_void_p()
    uid = pb._capi.UniqueId()
    assert lib.cemuCommInitRankConfig(C.byref(h), config(4).encode(), uid, 2, 0) == 4  # not real
    assert b"not a real rank" in lib.cemuGetLastError(None)
    assert lib.cemuCommInitRankConfig(C.byref(h), b"world_size = x\n", uid, 0, 0) == 4
    assert b"world_size" in lib.cemuGetLastError(None)
    comm.close()


def test_group_start_end_defers_and_replays_in_order(cuda):
    from paper_2405_02969_b200._capi import lib
    comm = pb.Communicator(config(8), 0, 0)
    h = host_input(7, 4096, seed=1)
    a, b = h.cuda(), h.cuda()
    assert lib.cemuGroupStart() == 0
    comm.all_reduce(a, a)
    comm.all_reduce(a, a)  # applied twice, in order
    assert lib.cemuGroupEnd() == 0
    comm.all_reduce(b, b)
    comm.all_reduce(b, b)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    comm.close()


def test_cuda_graph_capture_and_replay(cuda):
    """Every call is a stream-ordered kernel sequence with no host sync, so it
    can be captured in a CUDA graph and replayed (launch-bound small
    collectives); results and the device delay records are per replay."""
    comm = pb.Communicator(config(8, extra="delay.inject_us = 40\n"), 0, 0)
    h = host_input(7, 4096 + 3, seed=5)
    x = h.cuda()
    ys = [torch.empty_like(x) for _ in range(4)]
    comm.all_reduce(x, ys[0])  # warm-up outside capture (occupancy queries)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for y in ys:
            comm.all_reduce(x, y)
    want = P.allreduce(7, P.PAYLOAD_HASH, 8, [0], 0, 1, [to_np(h)], x.numel())
    for _ in range(3):
        for y in ys:
            y.zero_()
        g.replay()
        torch.cuda.synchronize()
        for y in ys:
            assert_bit_equal(to_np(y), want, "graph replay")
        rec = comm.call_record()
        assert abs((rec["t_end_ns"] - rec["t_start_ns"]) / 1e3 - 40) <= 2
    comm.close()


def test_registration_on_one_real_gpu(comms):
    """cemuCommRegister / Deregister with one real GPU: bookkeeping only --
    calls on a registered tensor are unchanged, a handle can be dropped once,
    an unknown handle is an invalid argument, a null buffer registers nothing."""
    import ctypes as C
    from paper_2405_02969_b200._capi import lib
    comm = comms(8)
    x = host_input(7, 100003, seed=5)
    d = x.cuda()
    h = comm.register(d)
    assert h
    y = torch.empty_like(d)
    comm.all_reduce(d, y)
    torch.cuda.synchronize()
    assert_bit_equal(to_np(y), P.allreduce(7, P.PAYLOAD_HASH, 8, [0], 0, 1, [to_np(x)], 100003), "registered")
    comm.deregister(h)
    with pytest.raises(pb.CemuError, match="not returned by cemuCommRegister"):
        comm.deregister(h)
    out = C.c_void_p(1)
    assert lib.cemuCommRegister(comm._h, None, 0, C.byref(out)) == 0 and not out.value
