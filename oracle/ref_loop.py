"""The reference's run_training_loop in its own process (bench.py's what-if
comparison arm).  TEST INFRASTRUCTURE ONLY: it times the reference
(oracle/_ref) and is never on the product path.

A separate process so the caller can bound it: the reference's loopback
transport occasionally stalls (oracle/ref_session.py), and a thread stuck
inside a C call cannot be killed, a process can.

    echo '{"text": ..., "world": 8, "bucket_bytes": 26214400, "inject": 0}' | python -m oracle.ref_loop

prints the per-iteration wall times (us) as one JSON list, or exits 1 with
the reference's error on stderr.
"""
from __future__ import annotations

import json
import sys

from oracle import ref


def main() -> int:
    a = json.loads(sys.stdin.read())
    try:
        it = ref.run_training_loop(a["text"], int(a["world"]), int(a["bucket_bytes"]), inject=float(a["inject"]))
    except ref.RefError as e:
        print(str(e), file=sys.stderr, flush=True)
        return 1
    print(json.dumps([float(t) for t in it]), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
