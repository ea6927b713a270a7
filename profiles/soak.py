"""Soak: mixed collectives for SECONDS, every 50th result checked against the
oracle; device memory and the async-error state checked at the end."""
import os, sys, time, random, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2405_02969_b200 as pb
from gpu_util import TORCH, host_input, to_np, assert_bit_equal
from oracle import port as P
SECONDS = float(os.environ.get("SOAK_S", "60"))
n = int(os.environ.get("WORLD_SIZE", "1")); local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
uid = None
if n > 1:
    import torch.distributed as dist
    dist.init_process_group("gloo")
    obj = [pb.get_unique_id() if local == 0 else None]; dist.broadcast_object_list(obj, src=0); uid = obj[0]
W = 8 * n
real = list(range(n))
comm = pb.Communicator(f"world_size = {W}\nreal_ranks = {','.join(map(str, real))}\nbucket_bytes = 1\n", local, local, uid)
rng = random.Random(42)  # same sequence on every rank (collective calls must match)
torch.cuda.empty_cache()
free0 = torch.cuda.mem_get_info()[0]
calls = checks = 0
t_end = time.time() + SECONDS
bufs = {}
while True:
    if n > 1:
        flag = torch.tensor([1 if time.time() < t_end else 0])
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not flag.item(): break
    elif time.time() >= t_end:
        break
    dt = rng.choice([7, 9, 2, 1]); count = rng.choice([17, 4099, 65536, 1 << 20]); coll = rng.randrange(3)
    sym = n > 1 and rng.random() < 0.5
    for _ in range(49):
        calls += 1
        if coll == 0:
            x = (comm.alloc(count, TORCH[dt]) if sym else torch.zeros(count, dtype=TORCH[dt], device="cuda"))
            comm.all_reduce(x, x)
            if sym: torch.cuda.synchronize(); comm.free(x)
        elif coll == 1:
            r = torch.empty(count * W, dtype=TORCH[dt], device="cuda")
            comm.all_gather(r[local * count:(local + 1) * count], r)
        else:
            s_ = torch.zeros(count * W, dtype=TORCH[dt], device="cuda"); o = torch.empty(count, dtype=TORCH[dt], device="cuda")
            comm.reduce_scatter(s_, o)
    # one checked call
    if dt in (7, 9) and n > 1:  # dyadic (<= 5 significant bits): any real-part order sums exactly
        sends = [torch.from_numpy((np.random.default_rng(calls + i).integers(-16, 16, size=count) / 8)
                                  .astype(np.float32)).to(TORCH[dt]) for i in range(n)]
    else:
        sends = [host_input(dt, count, seed=calls + i) for i in range(n)]
    y = torch.empty(count, dtype=TORCH[dt], device="cuda")
    comm.all_reduce(sends[local].cuda(), y)
    torch.cuda.synchronize()
    want = P.allreduce(dt, P.PAYLOAD_HASH, W, real, local, 1, [to_np(s) for s in sends], count)
    assert_bit_equal(to_np(y), want, f"soak call {calls}")
    checks += 1; calls += 1
torch.cuda.synchronize()
assert comm.async_error() is None
torch.cuda.empty_cache()  # torch's caching allocator holds the loop's tensors
free1 = torch.cuda.mem_get_info()[0]
comm.close()
if local == 0:
    print(json.dumps({"gpus": n, "seconds": SECONDS, "calls": calls, "checked": checks,
                      "device_free_delta_MiB": round((free0 - free1) / 2**20, 1)}))
