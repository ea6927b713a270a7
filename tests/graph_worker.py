"""One rank of the multi-GPU graph-capture check (launched by
test_gpu_multigpu.py under torch.distributed.run).

A 512 MiB fp32 allreduce between symmetric buffers -- at two real GPUs the
copy-engine pipeline (CE pulls / fold-only kernels / CE pushes between peer
barriers), at four the fused kernel -- with a delay-model plugin active, is
captured into a CUDA graph and replayed on fresh inputs.  Nothing on the
enqueue path may block the host or allocate (the copy-engine staging was
sized by the eager warm-up; the plugin's offsets travel in the spin kernel's
parameters), so the capture must succeed; every replay must equal the
eager call on the same inputs bit for bit, the first 1 Mi elements must
equal the oracle, and the replayed delay must follow the plugin's floors.
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
from oracle import port as P  # noqa: E402


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


def plugin(coll, n, nbytes, k):
    return [3000.0 * (j + 1) / k for j in range(k)]


def run():
    local = int(os.environ["LOCAL_RANK"])
    n = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    W = 8 * n
    real = list(range(n))
    obj = [pb.get_unique_id() if local == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    os.environ["CEMU_CE"] = "1"  # two GPUs: the copy-engine pipeline, the path with the most moving parts
    comm = pb.Communicator(f"world_size = {W}\nreal_ranks = {','.join(map(str, real))}\nbucket_bytes = 1\n",
                           local, local, obj[0])
    comm.set_delay_model(plugin)
    count = 128 << 20  # 512 MiB fp32: the copy-engine pipeline's size at two GPUs
    x, y = comm.alloc(count, torch.float32), comm.alloc(count, torch.float32)
    base = ((torch.arange(count, device="cuda", dtype=torch.int64) % 61) - 30).float() / 8

    def fill(step):
        x.copy_(base + (local + step))
    fill(0)
    torch.cuda.synchronize()
    dist.barrier()
    comm.all_reduce(x, y)  # eager warm-up: sizes the copy-engine staging
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    l0 = comm.kernel_launches
    dist.barrier()
    with torch.cuda.graph(g, stream=s):
        comm.all_reduce(x, y, stream=s)
    captured_launches = comm.kernel_launches - l0
    captured_id = comm.last_call_id
    res = {"rank": local, "n": n, "captured_launches": captured_launches, "replays": []}
    for step in range(1, 4):
        fill(step)
        torch.cuda.synchronize()
        dist.barrier()
        g.replay()
        torch.cuda.synchronize()
        rec = comm.call_record(captured_id)
        got = y.clone()
        dist.barrier()
        comm.all_reduce(x, y)  # eager, same inputs
        torch.cuda.synchronize()
        eq = bool(torch.equal(got.view(torch.int32), y.view(torch.int32)))
        sub = 1 << 20
        sends = [((np.arange(sub) % 61) - 30).astype(np.float32) / 8 + (r + step) for r in range(n)]
        want = P.allreduce(7, P.PAYLOAD_HASH, W, real, local, 1, sends, sub)
        oracle_eq = bool(np.array_equal(got[:sub].cpu().numpy().view(np.uint32), want.view(np.uint32)))
        k = rec["steps"]
        floors_ok = rec["floors_us"].tolist() == [int(np.floor(3000.0 * (j + 1) / k + 0.5)) for j in range(k)]
        res["replays"].append({"equal_eager": eq, "equal_oracle_1Mi": oracle_eq, "floors_ok": floors_ok,
                               "delay_us": round((rec["t_end_ns"] - rec["t_start_ns"]) / 1e3, 2),
                               "late_us": round(rec["late_ns"] / 1e3, 2),
                               "overshoot_us": round(rec["overshoot_ns"] / 1e3, 2),
                               "pause_us": round(rec["stall_ns"] / 1e3, 2) if rec["stall_ns"] > 20_000 else 0.0})
    res["async_error"] = comm.async_error()
    print(json.dumps(res), flush=True)
    dist.barrier()
    comm.free(x)
    comm.free(y)
    comm.close()


if __name__ == "__main__":
    main()
