"""BASELINE config 3 on this box: a bf16 allreduce in a 128-rank world laid
out as 16 nodes x 8 GPUs, whose real ranks are THIS node's GPUs (ranks
0..k-1, k = 1, 2 or 4 under torchrun) and whose other 15 nodes (plus the
node's remaining 8-k GPUs) are emulated.
"hierarchical ring".

Two measurements, each the max over ranks:

  throughput  delay off: bf16 allreduce of `--mib` MiB per GPU from symmetric
              buffers (k > 1: one fused kernel over NVLink peer memory; k = 1:
              one synthesis kernel), algorithmic HBM GB/s = 2 S per GPU per
              call, and NVLink GB/s per direction = 2 (k-1)/k S per GPU.
  delay       collective_algo = hierarchical with the FSDP module's network
              (alpha 5 us / 50 GB/s between nodes, 2 us / 770 GB/s NVLink
              inside one; fsdp.NET): per size, the device-measured call
              latency (%globaltimer, call start to last release) against the
              model's, error = |measured - model| <= max(1%, 2 us).

    python -m paper_2405_02969_b200.c3 --mib 1024
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        -m paper_2405_02969_b200.c3 --mib 1024
"""
from __future__ import annotations

import argparse
import json
import os

import torch

from .comm import Communicator, get_unique_id
from .fsdp import NET

WORLD, GPN = 128, 8


def config(k: int, delay: bool) -> str:
    lines = [f"world_size = {WORLD}", f"real_ranks = {','.join(str(r) for r in range(k))}", "bucket_bytes = 1",
             "collective_algo = hierarchical", f"topology.gpus_per_node = {GPN}"]
    if delay:
        lines += ["delay.kind = alpha_beta", f"link.alpha_us = {NET['alpha_inter_us']!r}",
                  f"link.beta_us_per_byte = {NET['beta_inter_us_per_byte']!r}",
                  f"link.gamma_us_per_byte = {NET['gamma_us_per_byte']!r}",
                  f"link.intra.alpha_us = {NET['alpha_intra_us']!r}",
                  f"link.intra.beta_us_per_byte = {NET['beta_intra_us_per_byte']!r}"]
    return "\n".join(lines) + "\n"


def run(mib: int = 1024, steps: int = 50, warmup: int = 5, delay_sizes_mib=(1, 64, 256)):
    import torch.distributed as dist
    k = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    if k > 1:
        dist.init_process_group("gloo")

    def new_uid():  # one NCCL unique id per communicator (an id is consumed by its init)
        if k == 1:
            return None
        obj = [get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def max_over_ranks(v: float) -> float:
        if k == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        torch.cuda.synchronize()
        if k > 1:
            dist.barrier()

    out = {"config": "C3", "world": WORLD, "gpus_per_node": GPN, "real_gpus": k,
           "emulated_ranks": WORLD - k, "dtype": "bf16", "collective_algo": "hierarchical"}
    # -- throughput, delay off -------------------------------------------------
    comm = Communicator(config(k, False), rank, dev, new_uid())
    nbytes = mib << 20
    count = nbytes // 2
    x, y = comm.alloc(count, torch.bfloat16), comm.alloc(count, torch.bfloat16)
    x.copy_(torch.randn(count, device="cuda", generator=torch.Generator("cuda").manual_seed(rank)))
    for _ in range(warmup):
        comm.all_reduce(x, y)
    barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    l0 = comm.kernel_launches
    evs[0].record()
    for _ in range(steps):
        comm.all_reduce(x, y)
    evs[1].record()
    barrier()
    ms = max_over_ranks(evs[0].elapsed_time(evs[1]) / steps)
    out["throughput"] = {
        "bytes_per_gpu": nbytes, "steps": steps, "ms_per_call": round(ms, 5),
        "hbm_algorithmic_gbs_aggregate": round(k * 2 * nbytes / (ms * 1e-3) / 1e9, 1),
        "nvlink_gbs_per_direction_per_gpu": (round(2 * (k - 1) / k * nbytes / (ms * 1e-3) / 1e9, 1)
                                             if k > 1 else None),
        "kernel_launches_per_call": (comm.kernel_launches - l0) / steps,
        "path": "fused NVLink kernel (symmetric buffers)" if k > 1 else "one synthesis kernel"}
    del x, y
    comm.close()
    # -- hierarchical delay ------------------------------------------------------
    comm = Communicator(config(k, True), rank, dev, new_uid())
    pts = []
    for smib in delay_sizes_mib:
        n = (smib << 20) // 2
        x, y = comm.alloc(n, torch.bfloat16), comm.alloc(n, torch.bfloat16)
        x.zero_()
        errs, model = [], None
        for _ in range(4):
            barrier()
            comm.all_reduce(x, y)
            torch.cuda.synchronize()
            rec = comm.call_record()
            measured = (rec["t_end_ns"] - rec["t_start_ns"]) / 1e3
            model = rec["model_latency_us"]
            errs.append(abs(measured - model))
        err = max_over_ranks(max(errs[1:]))
        pts.append({"bytes": smib << 20, "model_us": model, "max_err_us": round(err, 3),
                    "tolerance_us": round(max(0.01 * model, 2.0), 3), "ok": err <= max(0.01 * model, 2.0)})
        del x, y
    comm.close()
    out["delay"] = pts
    if k > 1:
        dist.destroy_process_group()
    return out if rank == 0 else None


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--mib", type=int, default=1024, help="allreduce bytes per GPU (MiB)")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--delay-mib", type=int, nargs="+", default=[1, 64, 256])
    a = ap.parse_args()
    r = run(a.mib, a.steps, a.warmup, a.delay_mib)
    if r is not None:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
