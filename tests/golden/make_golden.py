"""Generates tests/golden/*.json from the REFERENCE itself (oracle/_ref).

Run here, where /root/reference exists and `make -C oracle ref` built
oracle/_ref/libcemu_ref.so:

    python tests/golden/make_golden.py

Every fixture is an output of the reference's own code (cemu_core compiled
from /root/reference/proj/src): config render/digest, chunking, DAG and
boundary dumps (checked against the reference's own golden files
proj/tests/data/*.txt), delay offsets/floors, OpState-driven call latency,
the emulator's zero-payload results (WorkerSession + EmulatorServer over
loopback) and all-real TCP ring results fed the hash payload.  The fixtures
travel to the GPU box; /root/reference does not.
"""
from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import port as P  # noqa: E402
from oracle import ref as R  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
REF_DATA = "/root/reference/proj/tests/data"
REF_CONFIGS = "/root/reference/proj/configs"


def dump(name, obj):
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, indent=1, sort_keys=True)
    print("wrote", name)


def f64hex(x):
    return np.float64(x).view(np.uint64).item()


def configs():
    out = {"shipped": {}, "random": [], "errors": []}
    for fn in sorted(os.listdir(REF_CONFIGS)):
        text = open(os.path.join(REF_CONFIGS, fn)).read()
        render, digest = R.config_render(text)
        out["shipped"][fn] = {"text": text, "render": render, "digest": digest}
    rng = random.Random(3)  # the shape of test_config.cpp:23-42's random_config
    for _ in range(60):
        n = 2 + rng.randrange(7)
        real = [0] + ([1] if n > 2 and rng.randrange(2) else [])
        lines = [f"world_size = {n}", "real_ranks = " + ",".join(map(str, real)),
                 f"bucket_bytes = {1 + rng.randrange(1 << 20)}",
                 f"link.alpha_us = {rng.randrange(1000) / 7.0!r}",
                 f"link.beta_us_per_byte = {rng.randrange(1000) / 1e6!r}",
                 f"link.gamma_us_per_byte = {rng.randrange(1000) / 1e7!r}",
                 "delay.kind = " + ["none", "alpha_beta", "fixed"][rng.randrange(3)],
                 f"delay.fixed_us = {rng.randrange(10000) / 3.0!r}",
                 f"delay.inject_us = {rng.randrange(10000) / 3.0!r}",
                 f"poll_period_us = {1 + rng.randrange(100)}",
                 "node_class = class-a"]
        lines += [f"endpoint.{r} = 127.0.0.1:{20000 + r}" for r in range(n)]
        rng.shuffle(lines)
        text = "# random\n" + "\n".join(lines) + "\n"
        render, digest = R.config_render(text)
        out["random"].append({"text": text, "render": render, "digest": digest})
    bad = [
        "world_size = banana\n",
        "world_size = 1\nreal_ranks = 0\nbucket_bytes = 1\nendpoint.0 = 127.0.0.1:29500\n",
        "world_size = 2\nreal_ranks = 0,1\nbucket_bytes = 1024\nendpoint.0 = 127.0.0.1:29500\nendpoint.1 = 127.0.0.1:29501\n",
        "world_size = 3\nreal_ranks = 0\nbucket_bytes = 1024\nendpoint.0 = 127.0.0.1:29500\nendpoint.1 = 127.0.0.1:29501\nendpoint.2 = 127.0.0.1:29502\nnode_class.0 = a\nnode_class.1 = b\n",
        "world_size = 2\nreal_ranks = 0\nbucket_bytes = 1024\nendpoint.0 = 127.0.0.1:29500\nendpoint.1 = 127.0.0.1:29501\nbogus_key = 1\n",
        "world_size = 2\nreal_ranks = 0\nbucket_bytes = 8\nendpoint.0 = 127.0.0.1:1\n",
        "world_size = 3\nreal_ranks = 0\nbucket_bytes = 8\nendpoint.0 = 127.0.0.1:2000\nendpoint.1 = 127.0.0.1:2000\nendpoint.2 = 127.0.0.1:3000\n",
        "world_size = 2\nreal_ranks = 0\nbucket_bytes = 0\nendpoint.0 = 127.0.0.1:1\nendpoint.1 = 127.0.0.1:2\n",
        "world_size = 2\nreal_ranks = 5\nbucket_bytes = 8\nendpoint.0 = 127.0.0.1:1\nendpoint.1 = 127.0.0.1:2\n",
        "world_size = 2\nreal_ranks = 0\nbucket_bytes = 8\ndelay.kind = banana\nendpoint.0 = 127.0.0.1:1\nendpoint.1 = 127.0.0.1:2\n",
        "world_size = 2\nreal_ranks = 0\nbucket_bytes = 8\nlink.alpha_us = -1\nendpoint.0 = 127.0.0.1:1\nendpoint.1 = 127.0.0.1:2\n",
        "world_size = 2\nreal_ranks = 0\nbucket_bytes = 8\nworld_size = 3\n",
        "world_size = 2\nreal_ranks = 0\nbucket_bytes = 8\nendpoint.0 = 127.0.0.1:1\nendpoint.1 = 127.0.0.1:99999\n",
        "world_size = 2\nreal_ranks = 0\nbucket_bytes = 8\njunk line\n",
        "world_size = 2\nreal_ranks = 0\nbucket_bytes = 8\ncollective_algo = mesh\nendpoint.0 = 127.0.0.1:1\nendpoint.1 = 127.0.0.1:2\n",
    ]
    for text in bad:
        try:
            R.config_render(text)
            raise SystemExit(f"expected the reference to reject: {text!r}")
        except R.RefError as e:
            out["errors"].append({"text": text, "error": str(e)})
    dump("configs.json", out)


def schedule():
    out = {"chunks": [], "dag_dumps": [], "boundary_dumps": []}
    rng = random.Random(7)
    cases = [(4, 1003, 1, c) for c in range(4)] + [(3, 40, 4, c) for c in range(3)]
    for _ in range(300):
        n = rng.randint(2, 1024)
        elem = rng.choice([1, 2, 4, 8])
        total = rng.randint(0, 1 << 34) // elem * elem
        cases.append((n, total, elem, rng.randrange(n)))
    for n, total, elem, c in cases:
        out["chunks"].append([n, total, elem, c, R.chunk_bytes(n, total, elem, c),
                              R.chunk_offset_bytes(n, total, elem, c)])
    full = R.dump_dag(0, 2, 64)
    assert full == open(os.path.join(REF_DATA, "full-allreduce-n2.txt")).read()
    bd = R.dump_boundary(0, 4, 4096)
    assert bd == open(os.path.join(REF_DATA, "boundary-allreduce-n4-real0.txt")).read()
    out["dag_dumps"].append({"coll": 0, "n": 2, "bytes": 64, "elem": 1, "text": full})
    for n in list(range(2, 13)) + [16, 31, 64]:
        for coll in (0, 1):
            for real in sorted({0, 1, n // 2, n - 1}):
                nbytes = 4096 * n + (12 if coll == 0 else 0)
                out["boundary_dumps"].append({
                    "coll": coll, "n": n, "bytes": nbytes, "elem": 4, "real": real,
                    "text": R.dump_boundary(coll, n, nbytes, 4, (real,))})
    dump("schedule.json", out)


def delay():
    out = {"cases": []}
    rng = random.Random(11)
    kat = [  # test_delay.cpp:10-30, 88-132 and the config-1 shape
        (0, 4, 4096, 1, 10.0, 0.01, 0.001, 0.0, 0.0),
        (1, 4, 1024, 1, 5.0, 0.02, 0.0, 0.0, 0.0),
        (0, 2, 64, 0, 0.0, 0.0, 0.0, 0.0, 2500.0),
        (0, 2, 64, 2, 0.0, 0.0, 0.0, 10.0, 2500.0),
        (0, 4, 4096, 2, 0.0, 0.0, 0.0, 100.0, 0.0),
        (0, 8, 64 << 20, 1, 10.0, 0.001, 0.0001, 0.0, 0.0),
    ]
    for _ in range(200):
        coll = rng.randrange(2)
        n = rng.randint(2, 64)
        nbytes = rng.randint(n, 1 << 30) // 4 * 4
        kat.append((coll, n, nbytes, rng.randrange(3), rng.randrange(10000) / 13.0,
                    rng.randrange(10000) / 777777.0, rng.randrange(10000) / 3333333.0,
                    rng.randrange(10000) / 3.0, rng.choice([0.0, rng.randrange(10000) / 7.0])))
    for coll, n, nbytes, kind, a, b, g, fx, inj in kat:
        offs = R.release_offsets(coll, n, nbytes, 4, (0,), kind, a, b, g, fx, inj)
        floors = R.opstate_floors(coll, n, nbytes, 4, (0,), kind, a, b, g, fx, inj, now=1000)
        lat, rel = R.simulated_call_latency_us(coll, n, nbytes, 4, kind, a, b, g, fx, inj)
        total = (R.ring_allreduce_delay_us(n, nbytes, a, b, g) if coll == 0
                 else R.ring_allgather_delay_us(n, nbytes, a, b))
        out["cases"].append({
            "coll": coll, "n": n, "bytes": nbytes, "kind": kind, "alpha": a, "beta": b,
            "gamma": g, "fixed": fx, "inject": inj, "total_bits": f64hex(total),
            "offsets_bits": [f64hex(o) for o in offs], "floors_now1000": [int(x) for x in floors],
            "latency_us": int(lat), "release_us": [int(x) for x in rel]})
    # multi-real K counts (BoundaryDag::count(kToReal))
    out["to_real_counts"] = []
    for n in range(3, 12):
        for real in ([0, 1], [0, 2], [1, 3, 4], [0, 1, 2, 3], [2, 5, 7]):
            real = [r for r in real if r < n]
            if len(real) >= n:
                continue
            for coll in (0, 1):
                out["to_real_counts"].append([coll, n, real, len(R.release_offsets(coll, n, 64 * n, 1, real))])
    dump("delay.json", out)


def emulated_zero():
    """The reference emulator's actual outputs (dummy zero payloads)."""
    out = {"allreduce": [], "allgather": []}
    rng = np.random.default_rng(5)
    for n in (2, 3, 4, 5, 8):
        for elem, count in ((4, 8), (4, 37), (4, 1000), (1, 100), (1, 1001)):
            count = max(count, n)
            dt = np.int32 if elem == 4 else np.uint8
            buf = rng.integers(-2**31 if elem == 4 else 0, 2**31 if elem == 4 else 256,
                               size=count, dtype=np.int64).astype(dt)
            inp = buf.copy()
            R.emulated_collective(n, 0, buf, count * elem, elem)
            out["allreduce"].append({"n": n, "elem": elem, "input": inp.tolist(), "output": buf.tolist()})
        for elem, block in ((4, 4), (4, 33), (1, 50)):
            dt = np.int32 if elem == 4 else np.uint8
            full = np.full(block * n, 7, dtype=dt)
            full[:block] = np.arange(block, dtype=dt) + 1
            inp = full.copy()
            R.emulated_collective(n, 1, full, block * elem, elem)
            out["allgather"].append({"n": n, "elem": elem, "input": inp.tolist(), "output": full.tolist()})
    dump("emulated_zero.json", out)


def real_ring_hash():
    """All-real reference TCP rings fed this build's hash payload (rank r's
    input = payload of rank r, seed 1): pins the integer hash-mode results."""
    out = {"allreduce": [], "allgather": []}
    seed = 1
    for n in (2, 3, 4, 6, 8):
        for dtype, elem, count in ((2, 4, 64), (2, 4, 1031), (1, 1, 515)):
            bufs = [P.payload(dtype, P.payload_key(seed, r), 0, count).copy() for r in range(n)]
            R.real_ring(n, 0, bufs, count * elem, elem)
            for r in range(1, n):
                assert np.array_equal(bufs[r], bufs[0])
            out["allreduce"].append({"n": n, "dtype": dtype, "count": count, "seed": seed,
                                     "output": bufs[0].tolist()})
        for dtype, elem, block in ((2, 4, 40), (1, 1, 77)):
            fulls = []
            for r in range(n):
                f = np.zeros(block * n, dtype=P.DTYPES[dtype])
                f[r * block:(r + 1) * block] = P.payload(dtype, P.payload_key(seed, r), 0, block)
                fulls.append(f)
            R.real_ring(n, 1, fulls, block * elem, elem)
            out["allgather"].append({"n": n, "dtype": dtype, "block": block, "seed": seed,
                                     "output": fulls[0].tolist()})
    dump("real_ring_hash.json", out)


def eventlog():
    """The reference emulator's own EventLog of delayed calls: the emulator-side
    events (register, recv from_real, send to_real, complete) in log order."""
    import tempfile
    out = {"cases": []}
    path = tempfile.mktemp(suffix=".trace")
    R.trace_open(path)
    cases = [(4, 0, 64 << 10, 4, 1, 10.0, 0.001, 0.0001, 0.0, 0.0),
             (3, 1, 4096, 4, 2, 0.0, 0.0, 0.0, 300.0, 0.0),
             (8, 0, 1 << 20, 4, 1, 5.0, 0.0005, 0.0, 0.0, 1000.0)]
    for n, coll, plan_bytes, elem, kind, a, b, g, fx, inj in cases:
        start = sum(1 for _ in open(path)) if os.path.exists(path) else 0
        buf = np.zeros((plan_bytes * (n if coll == 1 else 1)) // 4, dtype=np.int32)
        R.emulated_collective(n, coll, buf, plan_bytes, elem, kind, a, b, g, fx, inj, warmup=0, reps=1)
        lines = open(path).read().splitlines()[start:]
        ev = []
        for ln in lines:
            f = ln.split()
            if len(f) == 6 and f[3] in ("to_real", "from_real", "-") and f[2] in ("register", "send", "recv", "complete"):
                ev.append(f[2:])
        out["cases"].append({"n": n, "coll": coll, "bytes": plan_bytes, "elem": elem, "kind": kind, "alpha": a,
                             "beta": b, "gamma": g, "fixed": fx, "inject": inj, "events": ev})
    dump("eventlog.json", out)


def payload_vectors():
    """Self-pinned regression vectors of the (new) payload spec."""
    out = {"keys": [], "words": []}
    for seed in (1, 2, 0xDEADBEEF):
        for rank in (0, 1, 7, 63, 1023):
            key = P.payload_key(seed, rank)
            out["keys"].append([seed, rank, key])
            for j in (0, 1, 2, 3, 1000, (1 << 28) + 5, (1 << 33) + 1):
                out["words"].append([key, j, P.payload_word(key, j)])
    dump("payload.json", out)


if __name__ == "__main__":
    if not R.available():
        raise SystemExit("build the reference first: make -C oracle ref")
    configs()
    schedule()
    delay()
    emulated_zero()
    real_ring_hash()
    eventlog()
    payload_vectors()
