"""Collective exerciser on the B200 path -- the counterpart of the reference's
`cemu-coll` (proj/tools/cemu_coll.cpp): every real rank runs the same call
sequence.

  timing  per-call latency on rank 0 over a list of sizes (warm-up, then
          repetitions), each call synchronous as the reference measures it
          (cemu_coll.cpp:107-163); prints one line per size
            RESULT op=allreduce bytes=B reps=R mean_us=M stddev_us=S
          and optionally writes the same columns as CSV
            op,size_bytes,repetitions,mean_us,stddev_us
  verify  checks every element against an expectation recomputed on the
          host (cemu_coll.cpp:41-105): the real ranks' seeded trial vectors
          plus, for every emulated rank, its payload words (the hash spec of
          DESIGN.md, computed here in numpy and self-checked against the
          C-ABI's cemuPayloadWord); int32 lanes, wrapping, as the reference's
          elem_size 4.  Prints  VERIFY ok op=allreduce n=W trials=T

Several real ranks: launch under torchrun (one process per GPU; rank 0's
NCCL unique id is broadcast over gloo).

    python -m paper_2405_02969_b200.coll --config job.cfg --mode timing \\
        --op allreduce --sizes 4096 1048576 67108864 --reps 20 --warmup 3
    python -m paper_2405_02969_b200.coll --config job.cfg --mode verify --trials 8
"""
from __future__ import annotations

import argparse
import csv
import os
import statistics
import sys
import time

import numpy as np
import torch

from . import schedule as S
from .comm import Communicator, get_unique_id

_WEYL, _WEYL_HI, _MUL1 = 0x9E3779B9, 0x85EBCA77, 0x7FEB352D


def payload_words(key: int, j0: int, n: int) -> np.ndarray:
    """word_key(j) for j in [j0, j0 + n) (payload.cuh), vectorised."""
    j = np.arange(j0, j0 + n, dtype=np.uint64)
    lo = (j & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    hi = (j >> np.uint64(32)).astype(np.uint32)
    with np.errstate(over="ignore"):
        c1 = ((lo * np.uint32(_WEYL)) ^ (hi * np.uint32(_WEYL_HI))) * np.uint32(_MUL1)
        x = np.uint32((key * _MUL1) & 0xFFFFFFFF) + c1
        x ^= x >> np.uint32(15)
        x *= np.uint32(key | 1)
        x += x >> np.uint32(16)
    return x


def _mix(seed: int, trial: int, rank: int) -> int:
    """cemu_coll.cpp:22-31 (splitmix64 finalizer of the three inputs)."""
    m = (1 << 64) - 1
    h = (seed ^ (trial * 0x9E3779B97F4A7C15) ^ (rank * 0xBF58476D1CE4E5B9)) & m
    h ^= h >> 30
    h = (h * 0xBF58476D1CE4E5B9) & m
    h ^= h >> 27
    h = (h * 0x94D049BB133111EB) & m
    h ^= h >> 31
    return h


def trial_vector(seed: int, trial: int, rank: int, elems: int) -> np.ndarray:
    """A real rank's seeded int32 input (the reference draws mt19937_64 from
    the same mixed seed, cemu_coll.cpp:33-39; numpy's generator here)."""
    g = np.random.default_rng(_mix(seed, trial, rank))
    return g.integers(-2**31, 2**31, size=elems, dtype=np.int64).astype(np.int32)


def _setup(config_text: str):
    n_local = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    from .comm import JobConfig
    real = JobConfig.parse(config_text).real_ranks
    if len(real) != n_local:
        raise SystemExit(f"the config has {len(real)} real ranks but {n_local} process(es) were launched")
    uid = None
    if n_local > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("gloo")
        obj = [get_unique_id() if local == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    return Communicator(config_text, real[local], local, uid), real, local


def _payload(config_text: str) -> tuple[str, int]:
    mode, pseed = "hash", 1
    for line in config_text.splitlines():
        k, _, v = line.partition("=")
        if k.strip() == "payload.mode":
            mode = v.strip()
        elif k.strip() == "payload.seed":
            pseed = int(v.strip())
    return mode, pseed


def run_verify(config_text: str, op: str, trials: int, seed: int) -> int:
    mode, pseed = _payload(config_text)
    if mode != "hash":
        raise SystemExit("verify recomputes the hash payload; payload.mode = zero is checked by the tests")
    comm, real, local = _setup(config_text)
    W = comm.world_size
    me = real[local]
    # self-check of the host hash against the library's own spec
    for key in (S.payload_key(pseed, 1), 0xDEADBEEF):
        for j in (0, 1, 12345, (1 << 32) + 7):
            assert int(payload_words(key, j, 1)[0]) == S.payload_word(key, j)
    size_rng = np.random.default_rng(_mix(seed, 0xA11, 0))
    sizes = [W + int(size_rng.integers(0, 1024)) for _ in range(trials)]
    emulated = [r for r in range(W) if r not in real]
    keys = [S.payload_key(pseed, r) for r in emulated]
    for t, elems in enumerate(sizes):
        if op == "allreduce":
            buf = torch.from_numpy(trial_vector(seed, t, me, elems)).cuda()
            comm.all_reduce(buf)
            torch.cuda.synchronize()
            want = np.zeros(elems, dtype=np.uint32)
            with np.errstate(over="ignore"):
                for r in real:
                    want += trial_vector(seed, t, r, elems).view(np.uint32)
                for k in keys:
                    want += payload_words(k, 0, elems)
            if not np.array_equal(buf.cpu().numpy().view(np.uint32), want):
                print(f"rank {me} trial {t}: allreduce result mismatch", file=sys.stderr)
                return 1
        else:
            full = torch.zeros(elems * W, dtype=torch.int32, device="cuda")
            own = torch.from_numpy(trial_vector(seed, t, me, elems)).cuda()
            comm.all_gather(own, full)
            torch.cuda.synchronize()
            got = full.cpu().numpy().view(np.uint32).reshape(W, elems)
            for r in range(W):
                want = (trial_vector(seed, t, r, elems).view(np.uint32) if r in real else
                        payload_words(S.payload_key(pseed, r), 0, elems))
                if not np.array_equal(got[r], want):
                    print(f"rank {me} trial {t}: allgather block {r} mismatch", file=sys.stderr)
                    return 1
    comm.close()
    if local == 0:
        print(f"VERIFY ok op={op} n={W} trials={trials}")
    return 0


def run_timing(config_text: str, op: str, sizes: list[int], reps: int, warmup: int, csv_path: str | None,
               host: bool) -> int:
    comm, real, local = _setup(config_text)
    W = comm.world_size
    rows = []
    for nbytes in sizes:
        aligned = nbytes - nbytes % 4
        count = aligned // 4
        shape = count * W if op == "allgather" else count
        if host:
            buf = torch.zeros(shape, dtype=torch.int32).pin_memory()
        else:
            buf = torch.zeros(shape, dtype=torch.int32, device="cuda")
        own = buf[me_block(local, real, count)] if op == "allgather" else None
        us = []
        for i in range(warmup + reps):
            t0 = time.perf_counter()
            if op == "allreduce":
                (comm.all_reduce_host if host else comm.all_reduce)(buf)
            else:
                (comm.all_gather_host if host else comm.all_gather)(own, buf)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            if i >= warmup:
                us.append((t1 - t0) * 1e6)
        if local == 0:
            m = statistics.fmean(us)
            sd = statistics.stdev(us) if len(us) > 1 else 0.0
            print(f"RESULT op={op} bytes={aligned} reps={reps} mean_us={m:.3f} stddev_us={sd:.3f}", flush=True)
            rows.append([op, aligned, reps, f"{m:.6f}", f"{sd:.6f}"])
    comm.close()
    if local == 0 and csv_path:
        with open(csv_path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["op", "size_bytes", "repetitions", "mean_us", "stddev_us"])
            w.writerows(rows)
    return 0


def me_block(local: int, real: list[int], count: int) -> slice:
    r = real[local]
    return slice(r * count, (r + 1) * count)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--config", required=True, help="job config file (reference format)")
    ap.add_argument("--mode", choices=("timing", "verify"), default="timing")
    ap.add_argument("--op", choices=("allreduce", "allgather"), default="allreduce")
    ap.add_argument("--sizes", type=int, nargs="+", default=[4096, 65536, 1 << 20, 16 << 20])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--csv", default=None)
    ap.add_argument("--host-buffers", action="store_true", help="time cemuAllReduceHost / AllGatherHost")
    ap.add_argument("--trials", type=int, default=8)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args(argv)
    text = open(a.config).read()
    if a.mode == "verify":
        return run_verify(text, a.op, a.trials, a.seed)
    return run_timing(text, a.op, a.sizes, a.reps, a.warmup, a.csv, a.host_buffers)


if __name__ == "__main__":
    sys.exit(main())
