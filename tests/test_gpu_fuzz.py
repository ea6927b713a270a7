"""Randomised parity sweep: 640 collectives with random world size, real-rank
position, seed, datatype, element count, buffer misalignment and in/out of
place, across all four collectives -- every output byte against the oracle
(NaN-free float inputs, so bit equality is the contract)."""
from __future__ import annotations

import random

import pytest
import torch

import paper_2405_02969_b200 as pb
from gpu_util import TORCH, assert_bit_equal, config, host_input, to_np
from oracle import port as P

pytestmark = pytest.mark.gpu

DTS = [0, 1, 2, 4, 6, 7, 8, 9]


def _on_device(h: torch.Tensor, shift: int) -> torch.Tensor:
    """h copied to the GPU at an element offset `shift` inside a larger
    allocation (shift > 0: not 16-byte aligned for most dtypes)."""
    big = torch.empty(h.numel() + shift + 8, dtype=h.dtype, device="cuda")
    d = big[shift:shift + h.numel()]
    d.copy_(h)
    return d


@pytest.mark.parametrize("block", range(16))
def test_random_collectives_equal_the_oracle(cuda, block):
    rng = random.Random(1000 + block)
    comms = {}
    for _ in range(40):
        W = rng.choice([2, 3, 5, 8, 16, 33, 64, 100, 257, 300])
        rank = rng.randrange(W)
        seed = rng.choice([1, 7, 0xC0FFEE])
        key = (W, rank, seed)
        if key not in comms:
            comms[key] = pb.Communicator(config(W, (rank,), "hash", seed), rank, 0)
        comm = comms[key]
        dt = rng.choice(DTS)
        coll = rng.randrange(4)
        count = rng.choice([1, 2, 3, 7, 16, 255, 1000, 4097, 65536 + rng.randrange(64), rng.randrange(1, 300000)])
        shift = rng.choice([0, 0, 1, 3])
        inplace = rng.random() < 0.4
        what = f"W={W} rank={rank} seed={seed} dt={dt} coll={coll} n={count} shift={shift} inplace={inplace}"
        if coll == 0:  # allreduce
            h = host_input(dt, count, seed=rng.randrange(1 << 30))
            want = P.allreduce(dt, P.PAYLOAD_HASH, W, [rank], rank, seed, [to_np(h)], count)
            x = _on_device(h, shift)
            y = x if inplace else _on_device(torch.zeros_like(h), rng.choice([0, 2]))
            comm.all_reduce(x, y)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(y), want, "allreduce " + what)
        elif coll == 1:  # allgather
            count = min(count, 4096)
            h = host_input(dt, count, seed=rng.randrange(1 << 30))
            want = P.allgather(dt, P.PAYLOAD_HASH, W, [rank], rank, seed, [to_np(h)], count)
            recv = _on_device(torch.zeros(W * count, dtype=TORCH[dt]), shift)
            if inplace:
                recv[rank * count:(rank + 1) * count] = h.cuda()
                comm.all_gather(recv[rank * count:(rank + 1) * count], recv)
            else:
                comm.all_gather(_on_device(h, rng.choice([0, 1])), recv)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(recv), want, "allgather " + what)
        elif coll == 2:  # reduce-scatter
            rc = max(1, min(count, 4096))
            h = host_input(dt, rc * W, seed=rng.randrange(1 << 30))
            want = P.reducescatter(dt, P.PAYLOAD_HASH, W, [rank], rank, seed, [to_np(h)], rc)
            out = _on_device(torch.zeros(rc, dtype=TORCH[dt]), shift)
            comm.reduce_scatter(_on_device(h, rng.choice([0, 1])), out)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(out), want, "reducescatter " + what)
        else:  # broadcast from the real rank or an emulated one
            root = rng.choice([rank, (rank + 1) % W])
            h = host_input(dt, count, seed=rng.randrange(1 << 30))
            want = P.broadcast(dt, P.PAYLOAD_HASH, W, [rank], rank, root, seed,
                               to_np(h) if root == rank else None, count)
            out = _on_device(torch.zeros(count, dtype=TORCH[dt]), shift)
            comm.broadcast(_on_device(h, 0) if root == rank else None, out, root)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(out), want, "broadcast " + what)
    for c in comms.values():
        c.close()


@pytest.mark.parametrize("block", range(3))
def test_random_calls_through_the_synthesis_cache(cuda, block):
    """Random sequences of >= 1 MiB allreduces / reduce-scatters whose
    element ranges overlap earlier ones -- fills, hits, partial coverage,
    buffer growth, misaligned pointers (synthesised) -- with the cache on
    for any emulated world (min peers 1): every result equals the oracle."""
    rng = random.Random(7000 + block)
    comms = {}
    for _ in range(12):
        W = rng.choice([5, 17, 64, 100, 257, 300])
        rank = rng.randrange(W)
        key = (W, rank)
        if key not in comms:
            comms[key] = pb.Communicator(config(W, (rank,), "hash", 1), rank, 0)
            comms[key].set_synth_cache(1 << 30, 1)
        comm = comms[key]
        dt = rng.choice([0, 1, 2, 6, 7, 9])
        es = torch.empty(0, dtype=TORCH[dt]).element_size()
        shift = rng.choice([0, 0, 0, 1])
        what = f"W={W} rank={rank} dt={dt} shift={shift}"
        if rng.random() < 0.6:
            count = rng.choice([1 << 20, (1 << 20) + 5, rng.randrange(1 << 18, 3 << 19)]) // max(1, es // 2)
            count = max(count, (1 << 20) // es + 1)
            h = host_input(dt, count, seed=rng.randrange(1 << 30))
            want = P.allreduce(dt, P.PAYLOAD_HASH, W, [rank], rank, 1, [to_np(h)], count)
            x = _on_device(h, shift)
            y = _on_device(torch.zeros_like(h), 0)
            comm.all_reduce(x, y)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(y), want, f"cached allreduce n={count} " + what)
        else:
            rc = ((1 << 20) // es + rng.randrange(0, 4096)) // 4 * 4
            h = host_input(dt, rc * W, seed=rng.randrange(1 << 30))
            want = P.reducescatter(dt, P.PAYLOAD_HASH, W, [rank], rank, 1, [to_np(h)], rc)
            out = _on_device(torch.zeros(rc, dtype=TORCH[dt]), shift)
            comm.reduce_scatter(_on_device(h, 0), out)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(out), want, f"cached reduce-scatter rc={rc} " + what)
    stats = [c.synth_cache_stats() for c in comms.values()]
    assert sum(s["fills"] for s in stats) > 0
    for c in comms.values():
        c.close()


@pytest.mark.parametrize("block", range(3))
def test_random_mid_size_calls_through_the_synthesis_cache(cuda, block):
    """64 KiB - 1 MiB allreduces / reduce-scatters at worlds whose ranges
    reach 2^21 peer-elements (the cache's lower bound): small enough for the
    peer-split kernels (entries filled by synth_cache_fill, then the cached
    fold), partial overlaps, misaligned pointers, every entry form (uint16,
    centred, uint32 words) -- every result equals the oracle."""
    rng = random.Random(9100 + block)
    comms = {}
    for _ in range(16):
        W = rng.choice([33, 64, 300, 1025])
        rank = rng.randrange(W)
        key = (W, rank)
        if key not in comms:
            comms[key] = pb.Communicator(config(W, (rank,), "hash", 1), rank, 0)
        comm = comms[key]
        dt = rng.choice([0, 1, 2, 6, 7, 9])
        es = torch.empty(0, dtype=TORCH[dt]).element_size()
        shift = rng.choice([0, 0, 0, 1])
        what = f"W={W} rank={rank} dt={dt} shift={shift}"
        if W >= 300 or rng.random() < 0.6:  # (reduce-scatter buffers of W chunks stay at the smaller worlds)
            count = rng.randrange((64 << 10) // es, (1 << 20) // es)
            h = host_input(dt, count, seed=rng.randrange(1 << 30))
            want = P.allreduce(dt, P.PAYLOAD_HASH, W, [rank], rank, 1, [to_np(h)], count)
            x = _on_device(h, shift)
            y = _on_device(torch.zeros_like(h), 0)
            comm.all_reduce(x, y)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(y), want, f"mid-size allreduce n={count} " + what)
        else:
            rc = rng.randrange((64 << 10) // es, (512 << 10) // es) // 4 * 4
            h = host_input(dt, rc * W, seed=rng.randrange(1 << 30))
            want = P.reducescatter(dt, P.PAYLOAD_HASH, W, [rank], rank, 1, [to_np(h)], rc)
            out = _on_device(torch.zeros(rc, dtype=TORCH[dt]), shift)
            comm.reduce_scatter(_on_device(h, 0), out)
            torch.cuda.synchronize()
            assert_bit_equal(to_np(out), want, f"mid-size reduce-scatter rc={rc} " + what)
    assert sum(c.synth_cache_stats()["fills"] for c in comms.values()) > 0
    for c in comms.values():
        c.close()
