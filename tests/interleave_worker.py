"""One rank of the two-stream interleave check (launched by
test_gpu_multigpu.py under torch.distributed.run).

One communicator, two streams: stream A runs fused all-gathers, stream B
alternates fused reduce-scatters and allreduces -- the FSDP pattern of an
all-gather stream beside a reduce-scatter stream over one communicator.
Inputs alternate between two sets, so a call that read a peer's buffer
before the peer's previous call finished (or took another call's barrier
flags) produces a detectable mismatch.  Every result is compared bit for
bit, on its own stream right after the call, with the oracle's result for
that input set; mismatching elements are counted on the device.

CEMU_ORDER=0 (diagnostic only) removes the communicator's cross-stream
ordering: the fused calls then share the signal area's epoch and counter.
"""
from __future__ import annotations

import json
import os
import sys
import threading

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2405_02969_b200 as pb  # noqa: E402
from gpu_util import TORCH, to_np  # noqa: E402
from oracle import port as P  # noqa: E402


def bits(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.int16) if t.element_size() == 2 else t.view(torch.int32)


def expected(arr: np.ndarray, dt: int) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if dt == 9:
        t = t.view(torch.int16).view(torch.bfloat16)
    return t.cuda()


def main():
    limit = float(os.environ.get("MGPU_WATCHDOG_S", "300"))
    threading.Timer(limit, lambda: (print(f"watchdog: {limit}s", file=sys.stderr, flush=True), os._exit(3))).start()
    try:
        run()
    except BaseException as e:  # noqa: BLE001
        print(f"[{os.environ.get('LOCAL_RANK')}] FAILED: {e!r}", file=sys.stderr, flush=True)
        os._exit(1)
    sys.stdout.flush()
    os._exit(0)


def run():
    local = int(os.environ["LOCAL_RANK"])
    n = int(os.environ["WORLD_SIZE"])
    iters = int(os.environ.get("INTERLEAVE_ITERS", "1000"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    W = 8 * n
    real = list(range(n))
    obj = [pb.get_unique_id() if local == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = pb.Communicator(f"world_size = {W}\nreal_ranks = {','.join(map(str, real))}\nbucket_bytes = 1\n",
                           local, local, obj[0])

    def inputs(dt, count, tag):
        out = []
        for r in range(n):
            g = np.random.default_rng(7919 * tag + 31 * r + count)
            if dt == 2:
                v = torch.from_numpy(g.integers(-2**31, 2**31, size=count).astype(np.int64)).to(torch.int32)
            else:
                v = torch.from_numpy((g.standard_normal(count) * 3).astype(np.float32)).to(TORCH[dt])
            out.append(v)
        return out

    # all-gather (fp32, 64 Ki elements per block), reduce-scatter (bf16,
    # 512 Ki elements per chunk), allreduce (int32, 256 Ki elements): the
    # last two are >= 1 MiB, so the synthesis cache serves them when on
    blk, rc, ar = 1 << 16, 1 << 19, 1 << 18
    ag_send, ag_want, rs_send, rs_want, ar_send, ar_want = [], [], [], [], [], []
    for tag in range(2):
        s = inputs(7, blk, tag)
        t = comm.alloc(blk, torch.float32)
        t.copy_(s[local])
        ag_send.append(t)
        ag_want.append(expected(P.allgather(7, P.PAYLOAD_HASH, W, real, local, 1, [to_np(x) for x in s], blk), 7))
        s = inputs(9, rc * W, 10 + tag)
        t = comm.alloc(rc * W, torch.bfloat16)
        t.copy_(s[local])
        rs_send.append(t)
        rs_want.append(expected(P.reducescatter(9, P.PAYLOAD_HASH, W, real, local, 1, [to_np(x) for x in s], rc), 9))
        s = inputs(2, ar, 20 + tag)
        t = comm.alloc(ar, torch.int32)
        t.copy_(s[local])
        ar_send.append(t)
        ar_want.append(expected(P.allreduce(2, P.PAYLOAD_HASH, W, real, local, 1, [to_np(x) for x in s], ar), 2))
    ag_recv = comm.alloc(blk * W, torch.float32)
    rs_recv = comm.alloc(rc, torch.bfloat16)
    ar_recv = comm.alloc(ar, torch.int32)
    torch.cuda.synchronize()
    dist.barrier()

    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    bad_a = torch.zeros((), dtype=torch.int64, device="cuda")
    bad_b = torch.zeros((), dtype=torch.int64, device="cuda")
    launches0 = comm.kernel_launches
    for i in range(iters):
        j = i % 2
        with torch.cuda.stream(sa):
            comm.all_gather(ag_send[j], ag_recv, stream=sa)
            bad_a += (bits(ag_recv) != bits(ag_want[j])).sum()
        with torch.cuda.stream(sb):
            if i % 2 == 0:
                comm.reduce_scatter(rs_send[(i // 2) % 2], rs_recv, stream=sb)
                bad_b += (bits(rs_recv) != bits(rs_want[(i // 2) % 2])).sum()
            else:
                comm.all_reduce(ar_send[(i // 2) % 2], ar_recv, stream=sb)
                bad_b += (bits(ar_recv) != bits(ar_want[(i // 2) % 2])).sum()
    torch.cuda.synchronize()
    res = {"rank": local, "n": n, "iters": iters, "bad_allgather": int(bad_a), "bad_rs_ar": int(bad_b),
           "async_error": comm.async_error(), "launches": comm.kernel_launches - launches0,
           "order": os.environ.get("CEMU_ORDER", "1")}
    print(json.dumps(res), flush=True)
    dist.barrier()
    comm.close()


if __name__ == "__main__":
    main()
