"""One rank of the round-2 multi-GPU soak (run by test_gpu_multigpu.py with a
short count; `SOAK_ITERS=20000 torchrun --nproc-per-node N tests/soak_worker.py`
for a long run).

A random sequence of collectives over one communicator, each on one of two
streams chosen at random: allreduces on registered caller memory
(cemuCommRegister), on cemuMemAlloc memory (512 MiB: the copy-engine
pipeline at two GPUs) and on plain buffers (the NCCL path), reduce-scatters
and all-gathers on symmetric memory, broadcasts from an emulated root -- with
the synthesis cache on for every call over 1 MiB.  Each case alternates
between two input sets whose oracle results were computed up front; every
result is compared bit for bit on the device, on its own stream, right
after the call.  Exercises the per-communicator ordering, cache fills and
hits, the fused / copy-engine / NCCL paths and registration together.
"""
from __future__ import annotations

import json
import os
import random
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2405_02969_b200 as pb  # noqa: E402
from gpu_util import TORCH, to_np  # noqa: E402
from oracle import port as P  # noqa: E402


def main():
    limit = float(os.environ.get("MGPU_WATCHDOG_S", "900"))
    threading.Timer(limit, lambda: (print(f"watchdog: {limit}s", file=sys.stderr, flush=True), os._exit(3))).start()
    try:
        run()
    except BaseException as e:  # noqa: BLE001
        print(f"[{os.environ.get('LOCAL_RANK')}] FAILED: {e!r}", file=sys.stderr, flush=True)
        os._exit(1)
    sys.stdout.flush()
    os._exit(0)


def bits(t):
    return t.view(torch.int16) if t.element_size() == 2 else t.view(torch.int32)


def dev(arr, dt):
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return (t.view(torch.int16).view(torch.bfloat16) if dt == 9 else t).cuda()


def run():
    local, n = int(os.environ["LOCAL_RANK"]), int(os.environ["WORLD_SIZE"])
    iters = int(os.environ.get("SOAK_ITERS", "400"))
    big = int(os.environ.get("SOAK_BIG_MIB", "512"))
    os.environ.setdefault("CEMU_SYNTH_CACHE_MIN_PEERS", "4")  # the cache on at this world size
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    W, real = 8 * n, list(range(n))
    obj = [pb.get_unique_id() if local == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = pb.Communicator(f"world_size = {W}\nreal_ranks = {','.join(map(str, real))}\nbucket_bytes = 1\n",
                           local, local, obj[0])

    def inputs(dt, count, tag):
        out = []
        for r in range(n):
            g = np.random.default_rng(1_000_003 * tag + 7919 * r + count)
            if dt == 2:
                out.append(torch.from_numpy(g.integers(-2**31, 2**31, size=count).astype(np.int64)).to(torch.int32))
            else:  # dyadic: the NCCL path's fold order cannot matter
                out.append(torch.from_numpy((g.integers(-64, 64, size=count) / 8).astype(np.float32)).to(TORCH[dt]))
        return out

    # (name, fn(stream, stream index, j) -> result tensor, [expected_j for j in 0, 1]).  Every case
    # writes a separate output per stream: the library orders its own calls
    # across streams (NCCL semantics), not the user's kernels that read a
    # result -- two streams sharing an output would race the check on one
    # stream against the next call on the other.
    cases = []

    def add_allreduce(name, dt, count, kind, tag):
        sends, recv, want = [], None, []
        for j in range(2):
            s = inputs(dt, count, tag + j)
            if kind == "plain":
                x = s[local].cuda()
            else:
                x = comm.alloc(count, TORCH[dt]) if kind == "alloc" else torch.empty(count, dtype=TORCH[dt],
                                                                                      device="cuda")
                x.copy_(s[local])
            sends.append(x)
            want.append(dev(P.allreduce(dt, P.PAYLOAD_HASH, W, real, local, 1, [to_np(v) for v in s], count), dt))
        if kind == "alloc":
            recv = [comm.alloc(count, TORCH[dt]) for _ in range(2)]
        else:
            recv = [torch.empty(count, dtype=TORCH[dt], device="cuda") for _ in range(2)]
        if kind == "register":  # collective: every rank registers the same buffers in the same order
            for t in sends + recv:
                comm.register(t)
        cases.append((name, lambda st, si, j: comm.all_reduce(sends[j], recv[si], stream=st), want))

    add_allreduce("allreduce fp32 registered", 7, (1 << 20) + 8, "register", 10)
    add_allreduce("allreduce bf16 cemuMemAlloc", 9, 4 << 20, "alloc", 20)
    add_allreduce("allreduce int32 plain (NCCL path)", 2, (1 << 18) + 5, "plain", 30)
    add_allreduce(f"allreduce fp32 {big} MiB cemuMemAlloc", 7, big << 18, "alloc", 40)
    # reduce-scatter and all-gather on symmetric memory
    rc = 1 << 19
    rs_send, rs_want = [], []
    for j in range(2):
        s = inputs(9, rc * W, 50 + j)
        t = comm.alloc(rc * W, torch.bfloat16)
        t.copy_(s[local])
        rs_send.append(t)
        rs_want.append(dev(P.reducescatter(9, P.PAYLOAD_HASH, W, real, local, 1, [to_np(v) for v in s], rc), 9))
    rs_out = [comm.alloc(rc, torch.bfloat16) for _ in range(2)]
    cases.append(("reduce-scatter bf16", lambda st, si, j: comm.reduce_scatter(rs_send[j], rs_out[si], stream=st),
                  rs_want))
    blk = 1 << 16
    ag_send, ag_want = [], []
    for j in range(2):
        s = inputs(7, blk, 60 + j)
        t = comm.alloc(blk, torch.float32)
        t.copy_(s[local])
        ag_send.append(t)
        ag_want.append(dev(P.allgather(7, P.PAYLOAD_HASH, W, real, local, 1, [to_np(v) for v in s], blk), 7))
    ag_out = [comm.alloc(blk * W, torch.float32) for _ in range(2)]
    cases.append(("all-gather fp32", lambda st, si, j: comm.all_gather(ag_send[j], ag_out[si], stream=st), ag_want))
    root = n  # an emulated rank
    bc_out = [torch.empty(1 << 20, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    bc_want = dev(P.broadcast(9, P.PAYLOAD_HASH, W, real, local, root, 1, None, 1 << 20), 9)
    cases.append(("broadcast from an emulated root",
                  lambda st, si, j: comm.broadcast(None, bc_out[si], root, stream=st), [bc_want, bc_want]))
    torch.cuda.synchronize()
    dist.barrier()

    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    bad = {c[0]: torch.zeros((), dtype=torch.int64, device="cuda") for c in cases}
    counts = {c[0]: 0 for c in cases}
    rng = random.Random(12345)  # the same sequence on every rank
    weights = [1.0 if "MiB" not in c[0] else 0.05 for c in cases]
    t0 = time.time()
    for i in range(iters):
        name, fn, want = rng.choices(cases, weights)[0]
        si = rng.randrange(2)
        st = streams[si]
        j = counts[name] % 2
        with torch.cuda.stream(st):
            out = fn(st, si, j)
            bad[name] += (bits(out) != bits(want[j])).sum()
        counts[name] += 1
    torch.cuda.synchronize()
    res = {"rank": local, "n": n, "iters": iters, "seconds": round(time.time() - t0, 1),
           "bad": {k: int(v) for k, v in bad.items()}, "calls": counts, "async_error": comm.async_error(),
           "cache": comm.synth_cache_stats()}
    print("SOAK " + json.dumps(res), flush=True)
    dist.barrier()
    comm.close()


if __name__ == "__main__":
    main()
