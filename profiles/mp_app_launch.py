"""Starts tests/apps/nccl_mp_app (an unmodified multi-process NCCL program)
on GPUs 0..N-1 under the interposer -- one process per GPU, real ranks
0..N-1 of a world of 8N -- and prints each rank's line.  Used to capture an
ncu launch list of the whole job:
  ncu --target-processes all --metrics gpu__time_duration.sum ... \\
      python profiles/mp_app_launch.py N MODE COUNT ITERS
MODE: plain | register | window (see nccl_mp_app.c)."""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    n, mode, count, iters = int(sys.argv[1]), sys.argv[2], sys.argv[3], sys.argv[4]
    d = tempfile.mkdtemp()
    cfg = os.path.join(d, "job.cfg")
    with open(cfg, "w") as f:
        f.write(f"world_size = {8 * n}\nreal_ranks = {','.join(map(str, range(n)))}\nbucket_bytes = 1\n")
    env = dict(os.environ, CEMU_CONFIG=cfg, CEMU_DEBUG="INFO",
               LD_PRELOAD=os.path.join(ROOT, "paper_2405_02969_b200", "libnccl_cemu.so"))
    app = os.path.join(ROOT, "tests", "apps", "nccl_mp_app")
    idf = os.path.join(d, "id")
    procs = [subprocess.Popen([app, str(8 * n), str(r), str(r), count, mode, idf, os.path.join(d, f"o{r}"), iters],
                              env=env) for r in range(n)]
    rcs = [p.wait(timeout=900) for p in procs]
    sys.exit(max(rcs))


if __name__ == "__main__":
    main()
