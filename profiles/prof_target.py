"""The command profiled with ncu: the bench workload's hot kernel.

Emulated 1 GiB fp32 allreduce, world 8 (1 real + 7 emulated ranks), out of
place, through the C-ABI -- exactly bench.py's timed step.  Usage:
    python profiles/prof_target.py [--world 8] [--mib 1024] [--dtype fp32] [--iters 5]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_02969_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--mib", type=int, default=1024)
ap.add_argument("--dtype", default="fp32")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--cache", type=int, default=1, help="0: synthesis cache off (every call synthesises)")
a = ap.parse_args()
dt = {"fp32": torch.float32, "bf16": torch.bfloat16}[a.dtype]
comm = pb.Communicator(f"world_size = {a.world}\nreal_ranks = 0\nbucket_bytes = 1\n", 0, 0)
if not a.cache:
    comm.set_synth_cache(0, 16)
n = (a.mib << 20) // torch.empty(0, dtype=dt).element_size()
x = torch.randn(n, device="cuda").to(dt)
y = torch.empty_like(x)
for i in range(a.iters):
    comm.all_reduce(x, y)
    if i == 0:  # the fill has run: a centred range's escape count is known to the next calls
        torch.cuda.synchronize()
torch.cuda.synchronize()
print("ok", a.world, a.mib, a.dtype)
