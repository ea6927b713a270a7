"""One reference emulated-allreduce session in its own process (bench.py's
reference arm / cpu_baseline).  TEST INFRASTRUCTURE ONLY: it times the
reference (oracle/_ref) and is never on the product path.

Each session is a separate process -- the way the reference deploys a real
rank (proj/tools/cemu_coll.cpp) -- so the parent can bound it: the
reference's loopback transport occasionally stalls for minutes with both
peers' 8 MiB DATA frames in flight (sender blocked in sendmsg, receiver idle;
its own 30 s await does not end the call), and a thread stuck inside a C
call cannot be killed, a process can.

    python -m oracle.ref_session WORLD WARMUP STEPS SEED SAMPLE_BYTES

prints "ready" once the buffer is built, waits for one line on stdin (the
parent releases all sessions together), then prints the timed calls' wall
times (us) as one JSON list.
"""
from __future__ import annotations

import json
import sys

import numpy as np

from oracle import ref


def main(argv):
    world, warmup, steps, seed, sample = (int(a) for a in argv[1:6])
    buf = np.random.default_rng(seed).integers(0, 2**31, size=sample // 4, dtype=np.int64).astype(np.int32)
    ref.lib()
    print("ready", flush=True)
    sys.stdin.readline()
    last = None
    for _ in range(3):  # a loopback port picked by bind(0) can be taken in between: retry
        try:
            times = ref.emulated_collective(world, 0, buf, sample, 4, kind=0, warmup=warmup, reps=steps)
            print(json.dumps([float(t) for t in times]), flush=True)
            return 0
        except ref.RefError as e:
            last = e
    print(json.dumps({"error": str(last)}), flush=True)
    return 1


if __name__ == "__main__":
    sys.exit(main(sys.argv))
