"""Synthesis-cache probe: per-call device time of 1 GiB emulated allreduces
at the many-peer shapes (config 2: world 64 fp32 / bf16 / int32; config 3
at k = 1: world 128 bf16; world 1024 bf16), with the cache off, on its
filling call and on warm calls.  Prints one JSON line per shape.

  python profiles/cache_probe.py [--mib 1024] [--reps 10] [--shapes 1024:bf16,1024:fp32]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_02969_b200 as pb  # noqa: E402

PEAK = 6550.4


def timed(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--shapes", default="", help="W:dtype,... (fp32, bf16, int32); default: the six below")
    args = ap.parse_args()
    names = {"fp32": torch.float32, "bf16": torch.bfloat16, "int32": torch.int32}
    shapes = [(int(w), names[d]) for w, d in (x.split(":") for x in args.shapes.split(",") if x)] or \
        [(64, torch.float32), (64, torch.bfloat16), (64, torch.int32), (128, torch.bfloat16),
         (16, torch.float32), (1024, torch.bfloat16)]
    torch.cuda.set_device(0)
    S = args.mib << 20
    for W, dtype in shapes:
        comm = pb.Communicator(f"world_size = {W}\nreal_ranks = 0\nbucket_bytes = 1\n", 0, 0)
        n = S // torch.empty(0, dtype=dtype).element_size()
        x = torch.ones(n, dtype=dtype, device="cuda") if dtype != torch.int32 else \
            torch.arange(n, dtype=torch.int32, device="cuda")
        y = torch.empty_like(x)
        comm.set_synth_cache(0, 16)
        comm.all_reduce(x, y)
        off = timed(lambda: comm.all_reduce(x, y), args.reps)
        comm.set_synth_cache(4 << 30, 16)
        fill = timed(lambda: comm.all_reduce(x, y), 1)
        warm = timed(lambda: comm.all_reduce(x, y), args.reps)
        st = comm.synth_cache_stats()
        res = {"world": W, "dtype": str(dtype).split(".")[-1], "bytes": S, "ms_uncached": round(off, 4),
               "ms_fill": round(fill, 4), "ms_cached": round(warm, 4),
               "hbm_frac_uncached": round(2 * S / off / 1e6 / PEAK, 3),
               "hbm_frac_cached": round(2 * S / warm / 1e6 / PEAK, 3), "stats": st}
        print(json.dumps(res), flush=True)
        comm.close()
        del x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
