"""ncu evidence for the fused NVLink kernels of an unmodified multi-process
NCCL job (tests/apps/nccl_mp_app in `window` mode: ncclMemAlloc +
ncclCommWindowRegister, so every allreduce is fused_allreduce_vec).

Rank 0 runs under ncu; ranks 1..N-1 run unprofiled.  Metrics are limited to
ones that need a single pass -- a replayed fused kernel would wait at its
start barrier for peers that never run the same call again.  The ncu
wrapper on the GPU box first runs the profiled command once without ncu, so
the unprofiled peers are respawned for every rank-0 process: rank 0 writes
the unique id file, this launcher hands a copy to each peer.

  python profiles/ncu_fused_launch.py N COUNT ITERS OUT.csv METRICS [MODE [KERNEL_REGEX]]

MODE plain profiles the NCCL reduce-scatter / allgather path instead (the
real NCCL kernels' launch footprint, e.g. with KERNEL_REGEX nccl).
"""
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    n, count, iters, out_csv, metrics = int(sys.argv[1]), sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5]
    mode = sys.argv[6] if len(sys.argv) > 6 else "window"
    kregex = sys.argv[7] if len(sys.argv) > 7 else "fused|synth|barrier|delay"
    d = tempfile.mkdtemp()
    cfg = os.path.join(d, "job.cfg")
    with open(cfg, "w") as f:
        f.write(f"world_size = {8 * n}\nreal_ranks = {','.join(map(str, range(n)))}\nbucket_bytes = 1\n")
    env = dict(os.environ, CEMU_CONFIG=cfg, LD_PRELOAD=os.path.join(ROOT, "paper_2405_02969_b200", "libnccl_cemu.so"))
    app = os.path.join(ROOT, "tests", "apps", "nccl_mp_app")
    idf = os.path.join(d, "id")
    r0 = subprocess.Popen(["ncu", "--metrics", metrics, "--clock-control", "none", "--csv", "--log-file", out_csv,
                           "-k", f"regex:{kregex}",
                           app, str(8 * n), "0", "0", count, mode, idf, os.path.join(d, "o0"), iters], env=env)
    rounds = 0
    while r0.poll() is None and rounds < 4:
        if not os.path.exists(idf):
            time.sleep(0.05)
            continue
        time.sleep(0.2)  # the rename is atomic; give rank 0 a moment
        data = open(idf, "rb").read()
        os.unlink(idf)
        peers = []
        for r in range(1, n):
            pf = os.path.join(d, f"id_{rounds}_{r}")
            with open(pf, "wb") as f:
                f.write(data)
            peers.append(subprocess.Popen([app, str(8 * n), str(r), str(r), count, mode, pf,
                                           os.path.join(d, f"o{r}"), iters], env=env))
        for p in peers:
            p.wait(timeout=600)
        rounds += 1
    rc = r0.wait(timeout=900)
    print(f"ncu_fused_launch: rank-0 exit {rc}, peer rounds {rounds}", flush=True)
    sys.exit(rc)


if __name__ == "__main__":
    main()
