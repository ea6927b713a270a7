"""Known-answer cases from the reference's own unit tests (CPU only).

Each case restates one reference TEST_CASE / golden file and checks it on
BOTH the oracle (oracle/cemu_oracle.c) and the product's C-ABI schedule and
delay entry points (libcemu_b200.so via paper_2405_02969_b200.schedule),
which need no GPU.  The literals are copied from the reference test sources
cited per test, so nothing here reads /root/reference at run time.
"""
from __future__ import annotations

import pytest

from oracle import port as P
from paper_2405_02969_b200 import schedule as S

IMPLS = [pytest.param(P, id="oracle"), pytest.param(S, id="capi")]

# proj/tests/data/full-allreduce-n2.txt:1-16 (dump_dag format, dag.cpp:362-376)
FULL_ALLREDUCE_N2 = """\
# collective allreduce n=2 positions=2
0 send 0 0 1 0 32
0 recv 0 1 0 1 32
0 send 1 0 1 1 32
0 recv 1 1 0 0 32
0 send 0 1 0 1 32
0 recv 0 0 1 0 32
0 send 1 1 0 0 32
0 recv 1 0 1 1 32
edges
0 5
1 2
2 7
4 1
5 6
6 3
"""


def _full_dag_dump(M, n, nbytes, elem):
    """dump_dag of build_ring_dag (dag.cpp:73-166) from the closed-form ring
    schedule: vertices per rank, per position, send then recv; edges
    send(r,p) -> recv(succ r, p) and recv(r,p) -> send(r,p+1)."""
    P_ = M.positions(0, n)
    vid = lambda r, p, recv: (r * P_ + p) * 2 + recv
    lines = [f"# collective allreduce n={n} positions={P_}"]
    for r in range(n):
        pred, succ = (r + n - 1) % n, (r + 1) % n
        for p in range(P_):
            cs = M.send_chunk_at(0, n, r, p)
            cr = M.send_chunk_at(0, n, pred, p)
            lines.append(f"0 send {p} {r} {succ} {cs} {M.chunk_bytes(n, nbytes, elem, cs)}")
            lines.append(f"0 recv {p} {pred} {r} {cr} {M.chunk_bytes(n, nbytes, elem, cr)}")
    edges = []
    for r in range(n):
        for p in range(P_):
            edges.append((vid(r, p, 0), vid((r + 1) % n, p, 1)))
            if p + 1 < P_:
                edges.append((vid(r, p, 1), vid(r, p + 1, 0)))
    lines.append("edges")
    lines += [f"{u} {v}" for u, v in sorted(edges)]
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("M", IMPLS)
def test_full_allreduce_n2_golden_file(M):
    assert _full_dag_dump(M, 2, 64, 1) == FULL_ALLREDUCE_N2


@pytest.mark.parametrize("M", IMPLS)
def test_release_offsets_per_kind(M):
    # test_delay.cpp:88-114: n=4, 4096 B, real {0} -> 6 to-real messages
    k = M.to_real_count(0, 4, [0])
    assert k == 6
    none = M.delay_model()
    assert list(M.release_offsets(none, 0, 4, 4096, k)) == [0.0] * 6
    fixed = M.delay_model(kind=P.DELAY_FIXED, fixed=100.0)
    assert list(M.release_offsets(fixed, 0, 4, 4096, k)) == [100.0] * 6
    ab = M.delay_model(kind=P.DELAY_ALPHA_BETA, alpha=10.0, beta=0.01, gamma=0.001)
    total = M.model_total_us(ab, 0, 4, 4096)
    assert total == pytest.approx(124.512, rel=1e-12)
    offs = list(M.release_offsets(ab, 0, 4, 4096, k))
    for j in range(6):
        assert offs[j] == pytest.approx(total * (j + 1) / 6.0, rel=1e-12)
    assert all(offs[j] >= offs[j - 1] for j in range(1, 6))


@pytest.mark.parametrize("M", IMPLS)
def test_inject_lands_on_first_release(M):
    # test_delay.cpp:116-132: inject adds to offsets[0] only
    none = M.delay_model(inject=2500.0)
    assert list(M.release_offsets(none, 0, 2, 64, 2)) == [2500.0, 0.0]
    fixed = M.delay_model(kind=P.DELAY_FIXED, fixed=10.0, inject=2500.0)
    assert list(M.release_offsets(fixed, 0, 2, 64, 2)) == [2510.0, 10.0]


@pytest.mark.parametrize("M", IMPLS)
def test_release_respects_time_floor(M):
    # test_engine.cpp:108-116: offsets {500, 0} registered at t=1000 ->
    # nothing before 1499, the first release at exactly 1500
    m = M.delay_model(inject=500.0)
    assert list(M.release_offsets(m, 0, 2, 64, 2)) == [500.0, 0.0]
    floors = list(M.release_floors(m, 0, 2, 64, 2, 1000))
    assert floors == [1500, 1000]
    # head-of-line gating: the second release cannot precede the first, so
    # an instantaneous real node completes 500 us after registration (A14)
    assert M.call_latency_us(m, 0, 2, 64, 2) == 500


@pytest.mark.parametrize("M", IMPLS)
def test_n2_first_reply_is_emulated_ranks_own_chunk(M):
    # test_engine.cpp:81-106: at n=2 the step-0 to-real message carries
    # emulated rank 1's own chunk (src 1 -> dst 0, step 0); the step-1 one
    # forwards the real node's step-0 chunk back (chunk 0)
    assert M.positions(0, 2) == 2
    assert M.send_chunk_at(0, 2, 1, 0) == 1
    assert M.send_chunk_at(0, 2, 1, 1) == M.send_chunk_at(0, 2, 0, 0) == 0
    assert M.call_latency_us(M.delay_model(), 0, 2, 64, 2) == 0


@pytest.mark.parametrize("M", IMPLS)
def test_dummy_frame_is_tail_chunk(M):
    # test_transport.cpp:281-311: allreduce of 100 B (elem 1) at n=2 -> the
    # first DATA frame is emulated rank 1's chunk 1, the 50-byte tail
    c = M.send_chunk_at(0, 2, 1, 0)
    assert c == 1
    assert M.chunk_bytes(2, 100, 1, c) == 50
    assert M.chunk_offset_bytes(2, 100, 1, c) == 50
