"""The oracle is pinned before it is trusted (CPU only).

Every check compares the C restatement (oracle/cemu_oracle.c) with outputs
of the REFERENCE itself: the committed fixtures in tests/golden/ (made by
tests/golden/make_golden.py from oracle/_ref) and, where the reference was
built here, live calls into oracle/_ref/libcemu_ref.so.
"""
from __future__ import annotations

import random

import numpy as np
import pytest

from conftest import golden
from oracle import port as P
from oracle import ref as R

needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built here")


def _model(c):
    return P.delay_model(c["kind"], P.ALGO_RING, c["alpha"], c["beta"], c["gamma"], c["fixed"], c["inject"])


# ---- schedule (dag.cpp:32-82, 232-393) --------------------------------------
def test_chunking_matches_reference_kats():
    g = golden("schedule.json")
    # test_dag.cpp:75-86
    assert [P.chunk_bytes(4, 1003, 1, c) for c in range(4)] == [250, 250, 250, 253]
    assert P.chunk_offset_bytes(4, 1003, 1, 3) == 750
    assert [P.chunk_bytes(3, 40, 4, c) for c in range(3)] == [12, 12, 16]
    for n, total, elem, c, nb, off in g["chunks"]:
        assert P.chunk_bytes(n, total, elem, c) == nb
        assert P.chunk_offset_bytes(n, total, elem, c) == off


def test_boundary_closed_form_equals_reference_projection():
    for case in golden("schedule.json")["boundary_dumps"]:
        got = P.dump_boundary(case["coll"], case["n"], case["bytes"], case["elem"], case["real"])
        assert got == case["text"], (case["coll"], case["n"], case["real"])


def test_boundary_matches_reference_golden_file():
    g = golden("schedule.json")
    n4 = [c for c in g["boundary_dumps"] if c["coll"] == 0 and c["n"] == 4 and c["real"] == 0][0]
    # proj/tests/data/boundary-allreduce-n4-real0.txt (checked at generation)
    text = P.dump_boundary(0, 4, 4096, 1, 0)
    assert text.splitlines()[0] == "# boundary allreduce n=4 side=emulated"
    assert text.splitlines()[-8:] == ["0 7", "1 2", "2 9", "3 4", "4 11", "5 6", "7 8", "9 10"]
    assert n4["text"].split("edges")[1] == text.split("edges")[1]


def test_send_chunk_schedule_formulas():
    # dag.hpp:64-74: RS step s sends (r-s) mod n, AG step t sends (r+1-t) mod n
    for n in range(2, 9):
        for r in range(n):
            for p in range(2 * (n - 1)):
                want = (r - p) % n if p <= n - 2 else (r + 1 - (p - (n - 1))) % n
                assert P.send_chunk_at(0, n, r, p) == want
            for t in range(n - 1):
                assert P.send_chunk_at(1, n, r, t) == (r - t) % n


# ---- delay model (delay.cpp:5-47, engine.cpp:36-42) -------------------------
def test_delay_kats():
    # test_delay.cpp:10-30
    assert P.lib().or_ring_allreduce_delay_us(4, 4096, 10.0, 0.01, 0.001) == pytest.approx(124.512, rel=1e-12)
    assert P.lib().or_ring_allgather_delay_us(4, 1024, 5.0, 0.02) == pytest.approx(76.44, rel=1e-12)
    assert P.lib().or_ring_allreduce_delay_us(2, 0, 10.0, 0.0, 0.0) == 20.0
    # config 1: 140 + 117,440.512 + 5,872.0256
    assert P.lib().or_ring_allreduce_delay_us(8, 64 << 20, 10, 0.001, 0.0001) == pytest.approx(123452.5376)
    m = P.delay_model(P.DELAY_NONE, inject=2500)
    assert list(P.release_offsets(m, 0, 2, 64, 2)) == [2500.0, 0.0]
    m = P.delay_model(P.DELAY_FIXED, fixed=10, inject=2500)
    assert list(P.release_offsets(m, 0, 2, 64, 2)) == [2510.0, 10.0]


def test_offsets_floors_latency_bit_exact_vs_reference_fixtures():
    for c in golden("delay.json")["cases"]:
        m = _model(c)
        k = P.to_real_count(c["coll"], c["n"], [0])
        assert k == len(c["offsets_bits"])
        total = P.lib().or_ring_allreduce_delay_us(c["n"], c["bytes"], c["alpha"], c["beta"], c["gamma"]) \
            if c["coll"] == 0 else P.lib().or_ring_allgather_delay_us(c["n"], c["bytes"], c["alpha"], c["beta"])
        assert np.float64(total).view(np.uint64) == c["total_bits"]
        offs = P.release_offsets(m, c["coll"], c["n"], c["bytes"], k)
        assert offs.view(np.uint64).tolist() == c["offsets_bits"]
        assert P.release_floors(m, c["coll"], c["n"], c["bytes"], k, 1000).tolist() == c["floors_now1000"]
        # A14: completion - registration of an instantaneous real node, from
        # the reference's OpState driven on a virtual clock
        assert P.call_latency_us(m, c["coll"], c["n"], c["bytes"], k) == c["latency_us"]
        assert max(c["release_us"]) == c["latency_us"]


def test_to_real_counts_vs_reference():
    for coll, n, real, k in golden("delay.json")["to_real_counts"]:
        assert P.to_real_count(coll, n, real) == k


def test_per_step_accumulation_1e9():
    # test_delay.cpp:54-86 / acceptance criterion 8: closed form vs per-step sum
    rng = np.random.default_rng(22)
    for _ in range(1000):
        n = 2 + int(rng.integers(15))
        m = int(rng.integers(1 << 30))
        a, b, g = rng.integers(10000) / 13.0, rng.integers(10000) / 777777.0, rng.integers(10000) / 3333333.0
        chunk = np.longdouble(m) / n
        acc = sum(np.longdouble(a) + chunk * b + chunk * g for _ in range(n - 1))
        acc += sum(np.longdouble(a) + chunk * b for _ in range(n - 1))
        got = P.lib().or_ring_allreduce_delay_us(n, m, a, b, g)
        assert abs(got - float(acc)) <= 1e-9 * max(1.0, abs(float(acc)))


# ---- collective results ------------------------------------------------------
def test_zero_mode_equals_reference_emulator_outputs():
    g = golden("emulated_zero.json")
    # KATs test_transport.cpp:129-167
    ar = [c for c in g["allreduce"] if c["n"] == 2 and c["elem"] == 4 and len(c["input"]) == 8][0]
    assert ar["output"][:4] == [0, 0, 0, 0] and ar["output"][4:] == ar["input"][4:]
    for c in g["allreduce"]:
        dt = 2 if c["elem"] == 4 else 1
        x = np.asarray(c["input"], dtype=P.DTYPES[dt])
        got = P.allreduce(dt, P.PAYLOAD_ZERO, c["n"], [0], 0, 1, [x], len(x))
        assert got.tolist() == c["output"], (c["n"], c["elem"], len(x))
    for c in g["allgather"]:
        dt = 2 if c["elem"] == 4 else 1
        full = np.asarray(c["input"], dtype=P.DTYPES[dt])
        block = len(full) // c["n"]
        got = P.allgather(dt, P.PAYLOAD_ZERO, c["n"], [0], 0, 1, [full[:block]], block)
        assert got.tolist() == c["output"]


def test_integer_hash_mode_equals_reference_real_ring():
    """Emulating ranks 1..n-1 with the hash payload gives exactly what the
    reference's all-real TCP ring computes when every rank r really holds
    payload(r): the integer hash path is pinned to the reference's ring."""
    g = golden("real_ring_hash.json")
    for c in g["allreduce"]:
        n, dt, count, seed = c["n"], c["dtype"], c["count"], c["seed"]
        mine = P.payload(dt, P.payload_key(seed, 0), 0, count)
        got = P.allreduce(dt, P.PAYLOAD_HASH, n, [0], 0, seed, [mine], count)
        assert got.tolist() == c["output"], (n, dt, count)
    for c in g["allgather"]:
        n, dt, block, seed = c["n"], c["dtype"], c["block"], c["seed"]
        mine = P.payload(dt, P.payload_key(seed, 0), 0, block)
        got = P.allgather(dt, P.PAYLOAD_HASH, n, [0], 0, seed, [mine], block)
        assert got.tolist() == c["output"], (n, dt, block)


def test_payload_regression_vectors():
    g = golden("payload.json")
    for seed, rank, key in g["keys"]:
        assert P.payload_key(seed, rank) == key
    for key, j, word in g["words"]:
        assert P.payload_word(key, j) == word


def test_ring_execute_integer_equals_direct_sum():
    # test_dag.cpp:94-118 restated on the oracle's ring executor
    rng = np.random.default_rng(101)
    for _ in range(60):
        n = 2 + int(rng.integers(7))
        elems = n + int(rng.integers(64))
        ins = [rng.integers(-2**31, 2**31, size=elems, dtype=np.int64).astype(np.int32) for _ in range(n)]
        want = np.zeros(elems, dtype=np.uint32)
        for x in ins:
            want += x.view(np.uint32)
        for r in range(n):
            assert np.array_equal(P.ring_execute_allreduce(2, ins, r).view(np.uint32), want)


def test_float_fold_definition():
    """fp32: local + S*2^-7 rounds once (S exact); the ring order of
    oracles.hpp:43-101 agrees within the north star's 1e-6 relative."""
    rng = np.random.default_rng(4)
    n, count, seed = 8, 4096, 1
    x = rng.standard_normal(count).astype(np.float32)
    got = P.allreduce(7, P.PAYLOAD_HASH, n, [0], 0, seed, [x], count)
    peers = [x] + [P.payload(7, P.payload_key(seed, r), 0, count) for r in range(1, n)]
    exact = np.sum(np.stack(peers).astype(np.float64), axis=0)
    assert np.array_equal(got, exact.astype(np.float32))  # single rounding of the exact sum
    ring = P.ring_execute_allreduce(7, peers, 0)
    denom = np.maximum(np.abs(exact), 1.0)
    assert np.max(np.abs(ring.astype(np.float64) - got) / denom) <= 1e-6


@needs_ref
def test_live_reference_boundary_and_delay_random():
    rng = random.Random(9)
    for _ in range(40):
        n = rng.randint(2, 24)
        coll = rng.randrange(2)
        real = rng.randrange(n)
        nbytes = rng.randint(n, 1 << 24) // 4 * 4
        assert P.dump_boundary(coll, n, nbytes, 4, real) == R.dump_boundary(coll, n, nbytes, 4, (real,))
        kind = rng.randrange(3)
        a, b, g = rng.random() * 30, rng.random() / 1e3, rng.random() / 1e4
        fx, inj = rng.random() * 500, rng.choice([0.0, rng.random() * 3000])
        m = P.delay_model(kind, 0, a, b, g, fx, inj)
        k = P.to_real_count(coll, n, [real])
        assert P.release_floors(m, coll, n, nbytes, k, 5).tolist() == \
            R.opstate_floors(coll, n, nbytes, 4, (real,), kind, a, b, g, fx, inj, now=5).tolist()


@needs_ref
def test_live_reference_reduce_kernel_wraps():
    # test_reduce.cpp:31-47: 200 + 100 wraps to 44 (u8), i32 wraps
    a = np.array([200], dtype=np.uint8)
    R.lib().ref_reduce_add_u8(a.ctypes.data, np.array([100], dtype=np.uint8).ctypes.data, 1)
    assert a[0] == 44
    x = np.array([2**31 - 1, -2**31, -1, 1], dtype=np.int32)
    y = np.array([1, -1, -1, 2**31 - 1], dtype=np.int32)
    want = (x.view(np.uint32) + y.view(np.uint32)).view(np.int32)
    R.lib().ref_reduce_add_i32(x.ctypes.data, y.ctypes.data, 4)
    assert np.array_equal(x, want)
