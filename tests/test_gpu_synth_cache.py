"""GPU: the synthesis cache changes no bit.

The emulated ranks' contribution depends only on (seed, rank, element), so
a communicator folds repeat calls over an element range from a cache of the
per-element sums.  Every call here -- the one that fills the cache and the
ones that read it, every datatype, every entry form (uint16 at <= 256
emulated ranks, centred uint16 with escapes beyond, uint32 word sums), ragged tails, offsets, both streams, graph replay -- is
compared bit for bit with the CPU oracle, which never caches.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2405_02969_b200 as pb
from gpu_util import assert_bit_equal, config, host_input, to_np
from oracle import port as P

pytestmark = pytest.mark.gpu


def _comm(W, rank=0):
    return pb.Communicator(config(W, (rank,), "hash", 1), rank, 0)


def _ar(comm, h, stream=None):
    d = h.cuda()
    r = torch.empty_like(d)
    comm.all_reduce(d, r, stream=stream)
    torch.cuda.synchronize()
    return to_np(r)


@pytest.mark.parametrize("W", [64, 258, 300])
@pytest.mark.parametrize("dt", [7, 9, 6, 1, 0, 2])
def test_cached_allreduce_equals_oracle_on_fill_and_hits(cuda, W, dt):
    comm = _comm(W)
    count = (1 << 20) + 7  # >= 1 MiB for every kind, ragged tail
    for i in range(3):  # fill, hit, hit -- different inputs each time
        h = host_input(dt, count, seed=100 * W + 10 * dt + i)
        want = P.allreduce(dt, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(h)], count)
        assert_bit_equal(_ar(comm, h), want, f"cached allreduce W={W} dt={dt} call {i}")
    st = comm.synth_cache_stats()
    assert st["fills"] == 1 and st["hits"] == 2, st
    entry = 4 if dt == 2 else 2  # W = 300: centred 16-bit entries
    entries = count if dt == 2 else (count + 3) // 4 * 4  # byte kinds: whole payload words
    assert st["bytes"] == entries * entry  # one segment, exactly the range's entries
    comm.close()


def test_centred_entries_and_their_escapes():
    """257..8192 emulated ranks keep 16-bit entries centred on the byte sums'
    mean (kernels.hpp kCacheCentered16); a sum outside the 16-bit window is an
    escape the fold recomputes from the keys.  With the window's bound raised
    to 28,672 ranks, worlds of 20,001 / 20,002 ranks (even and odd peer
    counts: the u8 offset byte differs) make ~1.5% of the entries escapes --
    every result still equals the oracle (tests/c16_worker.py)."""
    import json
    import os
    import subprocess
    import sys
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c16_worker.py")
    env = dict(os.environ, CEMU_SYNTH_CACHE_C16_MAX="28672")
    r = subprocess.run([sys.executable, worker, "1024", "20001", "20002"], capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    esc = {c["world"]: c["escapes"] for c in res["cases"]}
    assert esc[1024] == 0 and esc[20001] > 100 and esc[20002] > 100, esc


def test_one_byte_cache_serves_every_byte_kind(cuda):
    """fp32, bf16, fp16 and u8 share the per-element byte sums: one fill, then
    hits for the other kinds over the same elements."""
    comm = _comm(64)
    count = 1 << 20
    for i, dt in enumerate((7, 9, 6, 1, 0)):
        h = host_input(dt, count, seed=7 + i)
        want = P.allreduce(dt, P.PAYLOAD_HASH, 64, [0], 0, 1, [to_np(h)], count)
        assert_bit_equal(_ar(comm, h), want, f"dt={dt}")
    assert comm.synth_cache_stats()["fills"] == 1
    comm.close()


def test_reduce_scatter_chunks_at_their_own_offsets(cuda):
    """Rank 5's reduce-scatter chunk starts at element 5 * rc: its entries are
    the cache's [5 rc, 6 rc); a later allreduce over [0, W rc) is a new fill
    (not covered), then hits."""
    W, rank, rc = 64, 5, (1 << 18) + 4
    comm = _comm(W, rank)
    for i in range(2):
        full = host_input(7, rc * W, seed=50 + i)
        out = torch.empty(rc, dtype=torch.float32, device="cuda")
        comm.reduce_scatter(full.cuda(), out)
        torch.cuda.synchronize()
        want = P.reducescatter(7, P.PAYLOAD_HASH, W, [rank], rank, 1, [to_np(full)], rc)
        assert_bit_equal(to_np(out), want, f"reduce-scatter call {i}")
    st = comm.synth_cache_stats()
    assert (st["fills"], st["hits"]) == (1, 1), st
    h = host_input(7, rc * W, seed=60)
    want = P.allreduce(7, P.PAYLOAD_HASH, W, [rank], rank, 1, [to_np(h)], rc * W)
    assert_bit_equal(_ar(comm, h), want, "allreduce after reduce-scatter")
    assert comm.synth_cache_stats()["fills"] == 2
    comm.close()


def test_fill_on_one_stream_hit_on_another(cuda):
    """The hit on stream B is ordered after the fill on stream A by the
    communicator's cross-stream call order."""
    comm = _comm(128)
    count = 3 << 20
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    xs = [host_input(9, count, seed=s) for s in (1, 2)]
    d = [x.cuda() for x in xs]
    r = [torch.empty_like(v) for v in d]
    torch.cuda.synchronize()
    comm.all_reduce(d[0], r[0], stream=sa)
    comm.all_reduce(d[1], r[1], stream=sb)
    torch.cuda.synchronize()
    for i in range(2):
        want = P.allreduce(9, P.PAYLOAD_HASH, 128, [0], 0, 1, [to_np(xs[i])], count)
        assert_bit_equal(to_np(r[i]), want, f"stream {i}")
    assert comm.synth_cache_stats()["hits"] == 1
    comm.close()


def test_graph_capture_reads_but_never_fills(cuda):
    """Inside a capture a covered range folds from the cache; an uncovered
    one is synthesised (no allocation or fill in a capture).  Replays equal
    the oracle."""
    comm = _comm(64)
    count = 1 << 20
    x = host_input(7, count, seed=3)
    d = x.cuda()
    r1 = torch.empty_like(d)
    comm.all_reduce(d, r1)  # fills [0, count)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        comm.all_reduce(d, r1, stream=s)   # covered: cached fold
    st0 = comm.synth_cache_stats()
    assert st0["hits"] == 1
    for i in range(3):
        d.copy_(host_input(7, count, seed=10 + i).cuda())
        g.replay()
        torch.cuda.synchronize()
        want = P.allreduce(7, P.PAYLOAD_HASH, 64, [0], 0, 1, [to_np(d.cpu())], count)
        assert_bit_equal(to_np(r1), want, f"replay {i}")
    # an uncovered range inside a capture: synthesised, nothing filled
    comm.set_synth_cache(4 << 30, 16)  # drops the entries
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        comm.all_reduce(d, r1, stream=s)
    assert comm.synth_cache_stats()["fills"] == st0["fills"]
    g2.replay()
    torch.cuda.synchronize()
    want = P.allreduce(7, P.PAYLOAD_HASH, 64, [0], 0, 1, [to_np(d.cpu())], count)
    assert_bit_equal(to_np(r1), want, "uncached replay")
    comm.close()


def test_cache_off_and_host_pipeline(cuda):
    """capBytes = 0: nothing is cached.  The host-buffer pipeline's chunks
    (32 MiB each, offsets e0 = i * chunk) fill and then hit per chunk."""
    comm = _comm(64)
    comm.set_synth_cache(0, 16)
    count = 1 << 20
    h = host_input(7, count, seed=9)
    want = P.allreduce(7, P.PAYLOAD_HASH, 64, [0], 0, 1, [to_np(h)], count)
    assert_bit_equal(_ar(comm, h), want, "cache off")
    assert comm.synth_cache_stats()["fills"] == 0
    comm.set_synth_cache(4 << 30, 16)
    count = (20 << 20) + 5  # 80 MiB fp32: three pipeline chunks
    for i in range(2):
        hin = host_input(7, count, seed=20 + i).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        comm.all_reduce_host(hin, hout)
        torch.cuda.synchronize()
        want = P.allreduce(7, P.PAYLOAD_HASH, 64, [0], 0, 1, [hin.numpy()], count)
        assert np.array_equal(hout.numpy().view(np.uint32), want.view(np.uint32)), i
    st = comm.synth_cache_stats()
    assert st["fills"] == 3 and st["hits"] == 3, st
    comm.close()
