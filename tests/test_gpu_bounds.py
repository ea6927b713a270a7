"""Guard bands: no kernel writes outside the buffer it was given.

compute-sanitizer is closed on the GPU pool, so out-of-bounds writes are
checked directly: every output buffer sits inside a larger allocation whose
bytes before and after it hold a canary, and every out-of-place input is
compared byte for byte after the call.  Ragged counts (vector tails), odd
byte offsets (scalar paths), both peer-split and per-vector shapes (small vs
large counts at world 64) and all four collectives are covered; the in-range
bytes must still equal the oracle.
"""
from __future__ import annotations

import random

import pytest
import torch

import paper_2405_02969_b200 as pb
from gpu_util import TORCH, assert_bit_equal, config, host_input, to_np
from oracle import port as P

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes of canary on each side
CANARY = 0xA5


class Guarded:
    """`count` elements of dtype `dt` at byte offset GUARD + shift*esize
    inside a canary-filled byte allocation."""

    def __init__(self, dt: int, count: int, shift: int, init: torch.Tensor | None = None):
        t = TORCH[dt]
        es = torch.empty(0, dtype=t).element_size()
        self.lo = GUARD + shift * es
        self.nbytes = count * es
        self.raw = torch.full((self.lo + self.nbytes + GUARD,), CANARY, dtype=torch.uint8, device="cuda")
        self.t = self.raw[self.lo:self.lo + self.nbytes].view(t)
        if init is not None:
            self.t.copy_(init)

    def check_guards(self, what: str):
        torch.cuda.synchronize()
        raw = self.raw.cpu()
        before, after = raw[:self.lo], raw[self.lo + self.nbytes:]
        bad_b = int((before != CANARY).sum())
        bad_a = int((after != CANARY).sum())
        assert bad_b == 0 and bad_a == 0, f"{what}: {bad_b} bytes before / {bad_a} after the buffer overwritten"


COUNTS = [1, 3, 17, 255, 4099, 65536 + 5, 1 << 20 | 3]


@pytest.mark.parametrize("W", [8, 64])
@pytest.mark.parametrize("dt", [1, 2, 7, 9])
def test_collectives_stay_inside_their_buffers(cuda, W, dt):
    rng = random.Random(77 * W + dt)
    comm = pb.Communicator(config(W, (0,), "hash", 5), 0, 0)
    try:
        for count in COUNTS:
            shift = rng.choice([0, 1, 3])
            what = f"W={W} dt={dt} n={count} shift={shift}"
            # allreduce, out of place: input untouched, output exact, guards intact
            h = host_input(dt, count, seed=rng.randrange(1 << 30))
            want = P.allreduce(dt, P.PAYLOAD_HASH, W, [0], 0, 5, [to_np(h)], count)
            x = Guarded(dt, count, rng.choice([0, 2]), h)
            y = Guarded(dt, count, shift)
            comm.all_reduce(x.t, y.t)
            y.check_guards("allreduce out " + what)
            x.check_guards("allreduce in " + what)
            assert_bit_equal(to_np(x.t), to_np(h), "allreduce input modified " + what)
            assert_bit_equal(to_np(y.t), want, "allreduce " + what)
            # allreduce in place
            z = Guarded(dt, count, shift, h)
            comm.all_reduce(z.t)
            z.check_guards("allreduce in place " + what)
            assert_bit_equal(to_np(z.t), want, "allreduce in place " + what)
            # allgather (per-rank block capped so W blocks stay small)
            bc = min(count, 4099)
            hb = host_input(dt, bc, seed=rng.randrange(1 << 30))
            want = P.allgather(dt, P.PAYLOAD_HASH, W, [0], 0, 5, [to_np(hb)], bc)
            s = Guarded(dt, bc, 1, hb)
            r = Guarded(dt, W * bc, shift)
            comm.all_gather(s.t, r.t)
            r.check_guards("allgather " + what)
            s.check_guards("allgather send " + what)
            assert_bit_equal(to_np(s.t), to_np(hb), "allgather input modified " + what)
            assert_bit_equal(to_np(r.t), want, "allgather " + what)
            # reduce-scatter
            hr = host_input(dt, bc * W, seed=rng.randrange(1 << 30))
            want = P.reducescatter(dt, P.PAYLOAD_HASH, W, [0], 0, 5, [to_np(hr)], bc)
            s = Guarded(dt, bc * W, 0, hr)
            o = Guarded(dt, bc, shift)
            comm.reduce_scatter(s.t, o.t)
            o.check_guards("reducescatter " + what)
            s.check_guards("reducescatter send " + what)
            assert_bit_equal(to_np(s.t), to_np(hr), "reducescatter input modified " + what)
            assert_bit_equal(to_np(o.t), want, "reducescatter " + what)
            # broadcast from an emulated root
            want = P.broadcast(dt, P.PAYLOAD_HASH, W, [0], 0, 1, 5, None, count)
            o = Guarded(dt, count, shift)
            comm.broadcast(None, o.t, 1)
            o.check_guards("broadcast " + what)
            assert_bit_equal(to_np(o.t), want, "broadcast " + what)
    finally:
        comm.close()


@pytest.mark.parametrize("dt", [7, 9, 2])
def test_host_buffer_calls_stay_inside_their_buffers(cuda, dt, monkeypatch):
    """cemuAllReduceHost / cemuAllGatherHost: the chunked D2H copies land only
    inside the pinned output span (1 MiB chunks, so many chunks per call)."""
    monkeypatch.setenv("CEMU_HOST_CHUNK_MIB", "1")
    W = 8
    comm = pb.Communicator(config(W, (0,), "hash", 5), 0, 0)
    t = TORCH[dt]
    es = torch.empty(0, dtype=t).element_size()
    try:
        for count in (5, (3 << 20) // es + 7):
            h = host_input(dt, count, seed=count + dt)
            want = P.allreduce(dt, P.PAYLOAD_HASH, W, [0], 0, 5, [to_np(h)], count)
            raw = torch.full((2 * GUARD + count * es + es,), CANARY, dtype=torch.uint8).pin_memory()
            lo = GUARD + es  # element-aligned, not 16-byte aligned
            out = raw[lo:lo + count * es].view(t)
            src = h.pin_memory()
            comm.all_reduce_host(src, out)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(out), want, f"host allreduce dt={dt} n={count}")
            assert_bit_equal(to_np(src), to_np(h), f"host allreduce input modified dt={dt} n={count}")
            assert int((raw[:lo] != CANARY).sum()) == 0 and int((raw[lo + count * es:] != CANARY).sum()) == 0
            blk = min(count, 1 << 16)
            want = P.allgather(dt, P.PAYLOAD_HASH, W, [0], 0, 5, [to_np(h[:blk])], blk)
            raw = torch.full((2 * GUARD + W * blk * es,), CANARY, dtype=torch.uint8).pin_memory()
            out = raw[GUARD:GUARD + W * blk * es].view(t)
            comm.all_gather_host(h[:blk].contiguous().pin_memory(), out)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(out), want, f"host allgather dt={dt} blk={blk}")
            assert int((raw[:GUARD] != CANARY).sum()) == 0 and int((raw[GUARD + W * blk * es:] != CANARY).sum()) == 0
    finally:
        comm.close()
