import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
from paper_2405_02969_b200 import fidelity as F
from paper_2405_02969_b200 import ddp as D
from paper_2405_02969_b200.comm import Communicator
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
host = dist.new_group(backend="gloo")
k = dist.get_world_size()
sizes = F.SIZES[:12]

def loaded_sweep(sizes, reps):
    """NCCL per-call latency while bf16 GEMMs run on another stream."""
    a = torch.randn(8192, 4096, device="cuda", dtype=torch.bfloat16); w = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    side = torch.cuda.Stream()
    out = []
    for size in sizes:
        x = torch.ones(size // 4, device="cuda")
        dist.barrier()
        s = torch.cuda.Stream()
        for _ in range(3): F.NcclAllReduce().all_reduce(x, stream=s)
        torch.cuda.synchronize(); dist.barrier()
        with torch.cuda.stream(side):
            for _ in range(60): a = (a @ w) * 0.001
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            for _ in range(reps): F.NcclAllReduce().all_reduce(x, stream=s)
            e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3 / reps)
    return out

idle = [u for u, _ in F.baseline_sweep(sizes, 100)]
loaded = loaded_sweep(sizes, 20)
res = {"idle": idle, "loaded": loaded}
iters = 60
class Timed(D.EmulatedDDP):
    def __init__(s, *a, **kw):
        super().__init__(*a, **kw); s.lat = []; s.rdy = [torch.cuda.Event(enable_timing=True) for _ in s.buckets]; s.dn = [torch.cuda.Event(enable_timing=True) for _ in s.buckets]; s.cur = []
    def _hook(s, p):
        bi, off = s.where[p]
        s.flat[bi][off:off + p.numel()].copy_(p.grad.view(-1), non_blocking=True)
        s.pending[bi] += 1
        if s.pending[bi] == len(s.buckets[bi]):
            s.rdy[bi].record(); s.comm_stream.wait_event(s.rdy[bi])
            s.comm.all_reduce(s.flat[bi], stream=s.comm_stream)
            s.done[bi].record(s.comm_stream); s.dn[bi].record(s.comm_stream)
    def finish(s):
        super().finish()
orig = D.EmulatedDDP
D.EmulatedDDP = Timed
def run(coll, sync=True):
    if sync: dist.barrier(group=host)
    t = F.mlp_loop(coll, iters, 3)
    return [float(np.mean(t)), float(np.std(t))]
res["nccl"] = run(F.NcclAllReduce())
import subprocess

dist.barrier(group=host)
if local == 0:
    for tag, tab in (("idle", idle), ("loaded", loaded)):
        for fp, smem in (((0, 0), (32, 100000)) if tag == "idle" else ((0, 0), (32, 100000), (32, 150000), (64, 100000))):
            comm = Communicator(f"world_size = {k}\nreal_ranks = 0\nbucket_bytes = 1\n", 0, local)
            comm.set_delay_model(F.table_plugin(sizes, tab)); comm.set_queue_chaining(10); comm.set_delay_footprint(fp, smem)
            res[f"emulated_{tag}_fp{fp}_smem{smem}"] = run(comm, False); comm.close()
dist.barrier(group=host)
if local == 0: print("RESULT " + json.dumps(res), flush=True)
dist.barrier(group=host)
