"""The N>1 host-side logic on CPU: world_size-2 gloo processes.

Each process is one real GPU of a job with real ranks {0, 1} in a world of
16.  The product's decomposition (cemuPlanShards: the same function
comm.cpp's multi-GPU allreduce uses) is executed with gloo standing in for
NCCL and the oracle standing in for the synthesis kernel; the reassembled
result must equal the oracle's whole-world allreduce, and the shards must
tile the buffer exactly once.  Also covers the unique-id exchange and the
max-over-ranks timing that bench.py uses.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

W, REAL, SEED = 16, [0, 1], 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, results):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import port as P
    from paper_2405_02969_b200 import get_unique_id
    from paper_2405_02969_b200.schedule import plan_shards
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        # unique id exchange, as bench.py does it
        obj = [get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
        # dyadic real inputs: NCCL's real sum is then exact in any order
        for count in (1, 2, 1001, 4096, 4099):
            rng = np.random.default_rng(count)
            sends = [(rng.integers(-512, 512, size=count) / 64).astype(np.float32) for _ in REAL]
            mine = torch.from_numpy(sends[rank].copy())
            plan = plan_shards(count, len(REAL), rank)
            (so, sc), (to, tc) = plan["shard"], plan["tail"]
            # "NCCL reduce-scatter" of the real part (+ the tail all-reduce)
            real_sum = mine.clone()
            dist.all_reduce(real_sum)
            out = torch.zeros(count)
            for off, n in ((so, sc), (to, tc)):
                if n:
                    seg = real_sum[off:off + n].numpy()
                    # emulated part on the own shard only: x + payloads of
                    # the emulated ranks at global element offsets off..off+n
                    keys = [P.payload_key(SEED, r) for r in range(W) if r not in REAL]
                    S = sum(P.payload(7, k, off, n).astype(np.float64) for k in keys)
                    out[off:off + n] = torch.from_numpy((seg.astype(np.float64) + S).astype(np.float32))
            # "NCCL allgather" of the shards
            owned = torch.zeros(count)
            owned[so:so + sc] = 1
            if tc:
                owned[to:to + tc] = 1
            dist.all_reduce(out.mul_(torch.where(torch.arange(count) >= to, 0.5, 1.0)))
            dist.all_reduce(owned)
            want = P.allreduce(7, P.PAYLOAD_HASH, W, REAL, rank, SEED, sends, count)
            ok = np.array_equal(out.numpy().view(np.uint32), want.view(np.uint32))
            tiles = bool(torch.all(owned[:to] == 1)) and bool(torch.all(owned[to:] == 2))
            results.put((rank, count, ok, tiles, uid == obj[0]))
        # max over ranks (bench.py's timing rule)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        results.put((rank, "max", float(t.item()) == 2.0, True, True))
    finally:
        dist.destroy_process_group()


def test_two_process_decomposition_equals_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = [q.get(timeout=5) for _ in range(2 * 6)]
    assert len(res) == 12
    for rank, count, ok, tiles, same_uid in res:
        assert ok and tiles and same_uid, (rank, count)


def test_plan_shards_properties():
    from paper_2405_02969_b200.schedule import plan_shards
    for count in (0, 1, 7, 8, 1 << 20, (1 << 20) + 3):
        for k in (1, 2, 3, 4, 8):
            cover = np.zeros(count, dtype=np.int64)
            for li in range(k):
                p = plan_shards(count, k, li)
                so, sc = p["shard"]
                to, tc = p["tail"]
                cover[so:so + sc] += 1
                assert tc < k and to + tc == count
            assert np.all(cover[: count - (count % k)] == 1) and np.all(cover[count - (count % k):] == 0)
