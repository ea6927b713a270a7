import os, sys, json
import torch, torch.distributed as dist
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("gloo")
n = 1 << 28
hi = torch.randn(n).pin_memory(); ho = torch.empty(n).pin_memory()
d1 = torch.empty(n, device="cuda"); d2 = torch.randn(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1): d1.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(d2, non_blocking=True)
def h2d():
    d1.copy_(hi, non_blocking=True)
res = {}
for name, f in (("h2d", h2d), ("bidir", both)):
    f(); torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): f()
    torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 5
print(json.dumps({"rank": local, **{k: round(v, 2) for k, v in res.items()}}))
os.system(f"nvidia-smi topo -m > gpurun_out/topo.txt 2>&1") if local == 0 else None
