"""DDP what-if with REAL compute ("issue the real compute on
one stream and the emulated allreduce plus spin on a comm stream").

The reference's harness emulates a training step with busy-wait compute
(proj/src/harness.cpp:191-254, clock.hpp:29-37); whatif.py restates that
with %globaltimer spin kernels.  Here the step is a genuine bf16 model on the
B200 -- an MLP stack whose GEMMs run on the tensor cores -- and data-parallel
training is emulated around it exactly as NeuronaBox intends: gradients are
bucketed in reverse layer order (bucketize's rule, harness.cpp:152-175) as
autograd produces them, each full bucket is all-reduced by the emulated
collective on a separate comm stream (synthesised peers + the injected
network delay), and the optimizer waits for the last bucket.  Sweeping the
injected delay gives the latency-vs-iteration-time curve of the real job:
below the knee the stall hides behind backward compute, above it every
bucket's stall is exposed (tail slope ~ bucket count).

    python -m paper_2405_02969_b200.ddp --layers 8 --width 4096 --tokens 8192 \\
        --bucket-mib 25 --delays-us 0 1000 2000 4000 8000
"""
from __future__ import annotations

import argparse
import json

import numpy as np
import torch

from .comm import Communicator


def build_model(layers: int, width: int, device) -> torch.nn.Module:
    mods = []
    for _ in range(layers):
        mods += [torch.nn.Linear(width, width, bias=False), torch.nn.GELU()]
    return torch.nn.Sequential(*mods).to(device=device, dtype=torch.bfloat16)


class EmulatedDDP:
    """Gradient bucketing + emulated allreduce on a comm stream.  Buckets fill
    in the order autograd finishes parameters (reverse layer order); a bucket
    is flushed when it reaches `bucket_bytes` or the last parameter arrives."""

    def __init__(self, model: torch.nn.Module, comm: Communicator, bucket_bytes: int):
        self.comm = comm
        self.params = [p for p in model.parameters() if p.requires_grad]
        self.comm_stream = torch.cuda.Stream()
        # static buckets, reverse parameter order (bucketize, harness.cpp:152-175)
        self.buckets, cur, size = [], [], 0
        for p in reversed(self.params):
            nbytes = p.numel() * p.element_size()
            if cur and size + nbytes > bucket_bytes:
                self.buckets.append(cur)
                cur, size = [], 0
            cur.append(p)
            size += nbytes
        if cur:
            self.buckets.append(cur)
        self.flat = [torch.empty(sum(p.numel() for p in b), dtype=self.params[0].dtype, device=self.params[0].device)
                     for b in self.buckets]
        self.where = {}
        for bi, b in enumerate(self.buckets):
            off = 0
            for p in b:
                self.where[p] = (bi, off)
                off += p.numel()
        self.pending = [0] * len(self.buckets)
        self.done = [torch.cuda.Event() for _ in self.buckets]
        self.handles = [p.register_post_accumulate_grad_hook(self._hook) for p in self.params]

    def close(self):
        for h in self.handles:
            h.remove()

    def _hook(self, p):
        bi, off = self.where[p]
        self.flat[bi][off:off + p.numel()].copy_(p.grad.view(-1), non_blocking=True)
        self.pending[bi] += 1
        if self.pending[bi] == len(self.buckets[bi]):  # bucket complete: all-reduce it
            ready = torch.cuda.Event()
            ready.record()
            self.comm_stream.wait_event(ready)
            self.comm.all_reduce(self.flat[bi], stream=self.comm_stream)
            self.done[bi].record(self.comm_stream)

    def finish(self):
        """Compute stream waits for every bucket; gradients get the sums."""
        for bi, b in enumerate(self.buckets):
            torch.cuda.current_stream().wait_event(self.done[bi])
            off = 0
            for p in b:
                p.grad.view(-1).copy_(self.flat[bi][off:off + p.numel()], non_blocking=True)
                off += p.numel()
        self.pending = [0] * len(self.buckets)


def run(layers=8, width=4096, tokens=8192, bucket_mib=25, world=8, delays_us=(0, 1000, 2000, 4000, 8000),
        iterations=12, warmup=3, device=0):
    torch.cuda.set_device(device)
    torch.manual_seed(0)
    model = build_model(layers, width, "cuda")
    x = torch.randn(tokens, width, device="cuda", dtype=torch.bfloat16)
    opt = torch.optim.SGD(model.parameters(), lr=1e-6)

    def step(ddp):
        opt.zero_grad(set_to_none=False)
        loss = model(x).float().pow(2).mean()
        loss.backward()
        if ddp is not None:
            ddp.finish()
        opt.step()

    def timed(ddp):
        for _ in range(warmup):
            step(ddp)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(iterations + 1)]
        ev[0].record()
        for i in range(iterations):
            step(ddp)
            ev[i + 1].record()
        torch.cuda.synchronize()
        return [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(iterations)]

    compute_only = float(np.mean(timed(None)))
    points, buckets = [], None
    for d in sorted(delays_us):
        cfg = f"world_size = {world}\nreal_ranks = 0\nbucket_bytes = {bucket_mib << 20}\ndelay.inject_us = {float(d)!r}\n"
        comm = Communicator(cfg, 0, device)
        ddp = EmulatedDDP(model, comm, bucket_mib << 20)
        buckets = len(ddp.buckets)
        t = timed(ddp)
        points.append({"inject_us": float(d), "mean_us": float(np.mean(t)), "stddev_us": float(np.std(t, ddof=1))})
        ddp.close()
        comm.close()
    hi = [(p["inject_us"], p["mean_us"]) for p in points if p["inject_us"] >= 4000]
    slope = None
    if len(hi) >= 2:
        xs, ys = np.array(hi).T
        slope = float(np.polyfit(xs, ys, 1)[0])
    return {"layers": layers, "width": width, "tokens": tokens, "world": world, "bucket_mib": bucket_mib,
            "buckets": buckets, "compute_only_us": compute_only,
            "emulation_overhead_at_0_delay_pct": 100.0 * (points[0]["mean_us"] / compute_only - 1.0) if points else None,
            "tail_slope": slope, "points": points}


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--width", type=int, default=4096)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--bucket-mib", type=int, default=25)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--delays-us", type=float, nargs="+", default=[0, 1000, 2000, 4000, 8000])
    a = ap.parse_args()
    print(json.dumps(run(a.layers, a.width, a.tokens, a.bucket_mib, a.world, a.delays_us), indent=1))


if __name__ == "__main__":
    main()
