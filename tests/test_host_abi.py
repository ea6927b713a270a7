"""Host side of the C-ABI (CPU only, no compute calls).

* libcemu_b200.so loads and exports every symbol include/cemu_b200.h declares;
* the C++ job-config parser renders and digests bit-identically to the
  reference (config.cpp:264-312) and rejects the same inputs, naming the
  offending field;
* the host schedule / delay-model functions equal the pinned oracle.
"""
from __future__ import annotations

import os
import random
import re
import subprocess

import numpy as np
import pytest

import paper_2405_02969_b200 as pb
from conftest import golden
from oracle import port as P
from paper_2405_02969_b200 import _capi
from paper_2405_02969_b200 import schedule as S


def _header_functions():
    text = open(_capi.HEADER_PATH).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cemu[A-Z]\w*)\s*\(", text)))


def test_library_exports_every_header_symbol():
    names = _header_functions()
    assert len(names) >= 35
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:  # and they resolve through the loader
        getattr(_capi.lib, n)


def test_nccl_interposer_exports_ncclapi():
    shim = os.path.join(os.path.dirname(_capi.LIB_PATH), "libnccl_cemu.so")
    out = subprocess.run(["nm", "-D", "--defined-only", shim], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines()}
    for name in ("ncclAllReduce", "ncclAllGather", "ncclReduceScatter", "ncclBroadcast", "ncclCommInitRank",
                 "ncclCommDestroy", "ncclCommCount", "ncclCommUserRank", "ncclGetUniqueId", "ncclGroupStart",
                 "ncclGroupEnd", "ncclGetErrorString", "ncclCommInitRankConfig", "ncclCommAbort",
                 "ncclCommRegister", "ncclCommDeregister", "ncclCommSplit", "ncclReduce", "ncclSend", "ncclRecv",
                 "ncclCommWindowRegister", "ncclCommWindowDeregister", "ncclMemAlloc", "ncclMemFree",
                 "ncclCommGetAsyncError", "ncclCommCuDevice"):
        assert name in exported, name


def test_round2_entry_points_reject_bad_arguments_without_a_device():
    """Registration, synthesis cache, queue chaining and delay footprint: a
    null communicator or an out-of-range argument is an invalid argument (4)
    before any device work."""
    import ctypes as C
    lib = _capi.lib
    h = C.c_void_p(1)
    assert lib.cemuCommRegister(None, None, 0, C.byref(h)) == 4
    assert lib.cemuCommDeregister(None, None) == 4
    assert lib.cemuCommSetSynthCache(None, 0, 16) == 4
    f, hits, b = C.c_uint64(), C.c_uint64(), C.c_size_t()
    assert lib.cemuCommSynthCacheStats(None, C.byref(f), C.byref(hits), C.byref(b)) == 4
    assert lib.cemuCommSetQueueChaining(None, 10) == 4
    assert lib.cemuCommSetDelayFootprint(None, 8, 0) == 4


def test_library_is_sm100a_and_links_no_torch():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in deps and "libcudart.so" not in deps  # cudart static, NCCL dlopen'ed


def test_version_and_errors():
    import ctypes as C
    v = C.c_int()
    assert _capi.lib.cemuGetVersion(C.byref(v)) == 0 and v.value >= 10000
    assert _capi.lib.cemuGetErrorString(4) == b"invalid argument"
    assert _capi.lib.cemuGetErrorString(5) == b"invalid usage"


def test_chain_entry_points_reject_null_arguments_without_a_device():
    import ctypes as C
    from paper_2405_02969_b200 import whatif  # noqa: F401  (declares the argtypes)
    lib = _capi.lib
    x = C.c_int64(0)
    assert lib.cemuChainJoin(None, None, C.byref(x)) == 4   # null chain
    assert lib.cemuChainJoin(None, C.byref(x), None) == 4   # null release end
    out = C.c_void_p(1)
    assert lib.cemuCommLastReleaseEnd(None, C.byref(out)) == 4  # null communicator


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="needs a host without a GPU")
def test_no_cpu_fallback_without_a_device():
    # the product path has no CPU route: a communicator cannot come up
    # without a CUDA device, through the Python mirror or the C-ABI
    import ctypes as C
    from gpu_util import config
    from paper_2405_02969_b200 import comm
    with pytest.raises(_capi.CemuError, match="cudaSetDevice"):
        comm.Communicator(config(8), 0, device=0)
    h = C.c_void_p()
    uid = comm.UniqueId()
    assert _capi.lib.cemuCommInitRankConfig(C.byref(h), config(8).encode(), uid, 0, 0) != 0
    assert h.value is None


# ---- job config (config.cpp) ------------------------------------------------
def test_shipped_configs_render_and_digest_like_reference():
    for name, c in golden("configs.json")["shipped"].items():
        cfg = pb.JobConfig.parse(c["text"])
        assert cfg.render() == c["render"], name
        assert cfg.digest == c["digest"], name


def test_random_configs_round_trip_like_reference():
    for c in golden("configs.json")["random"]:
        cfg = pb.JobConfig.parse(c["text"])
        assert cfg.render() == c["render"]
        assert cfg.digest == c["digest"]
        back = pb.JobConfig.parse(cfg.render())  # render/parse round trip (test_config.cpp:122-130)
        assert back.render() == c["render"] and back.digest == c["digest"]


def test_config_errors_name_the_field_like_reference():
    for c in golden("configs.json")["errors"]:
        with pytest.raises(pb.CemuError) as ei:
            pb.JobConfig.parse(c["text"])
        msg = str(ei.value).split("] ", 1)[1]
        if "collective_algo" in c["text"] and "mesh" in c["text"]:
            assert msg.startswith("collective_algo:")  # wording extended for tree/hierarchical
        else:
            assert msg == c["error"], c["text"]


def test_extension_keys_render_only_when_set():
    base = "world_size = 4\nreal_ranks = 0\nbucket_bytes = 8\n"
    plain = pb.JobConfig.parse(base)
    assert "payload" not in plain.render() and "topology" not in plain.render()
    ext = pb.JobConfig.parse(base + "payload.mode = zero\npayload.seed = 7\ncollective_algo = hierarchical\n"
                             "topology.gpus_per_node = 2\nlink.intra.alpha_us = 1.5\n")
    r = ext.render()
    assert "payload.mode = zero" in r and "payload.seed = 7" in r and "topology.gpus_per_node = 2" in r
    assert "collective_algo = hierarchical" in r and "link.intra.alpha_us = 1.5" in r
    assert pb.JobConfig.parse(r).render() == r
    with pytest.raises(pb.CemuError, match="topology.gpus_per_node"):
        pb.JobConfig.parse(base + "topology.gpus_per_node = 3\n")
    with pytest.raises(pb.CemuError, match="payload.mode"):
        pb.JobConfig.parse(base + "payload.mode = random\n")
    assert pb.JobConfig.parse(base).world_size == 4 and pb.JobConfig.parse(base).real_ranks == [0]


# ---- schedule / delay ---------------------------------------------------------
def test_host_schedule_equals_oracle_and_reference_fixtures():
    g = golden("schedule.json")
    for n, total, elem, c, nb, off in g["chunks"]:
        assert S.chunk_bytes(n, total, elem, c) == nb
        assert S.chunk_offset_bytes(n, total, elem, c) == off
    for case in g["boundary_dumps"]:
        assert S.boundary_dump(case["coll"], case["n"], case["bytes"], case["elem"], case["real"]) == case["text"]
    for n in range(2, 40):
        for r in range(n):
            for p in range(2 * (n - 1)):
                assert S.send_chunk_at(0, n, r, p) == P.send_chunk_at(0, n, r, p)


def test_host_delay_bit_exact_vs_reference_fixtures():
    for c in golden("delay.json")["cases"]:
        m = S.delay_model(c["kind"], S.RING, c["alpha"], c["beta"], c["gamma"], c["fixed"], c["inject"])
        k = S.to_real_count(c["coll"], c["n"], [0])
        assert S.release_offsets(m, c["coll"], c["n"], c["bytes"], k).view(np.uint64).tolist() == c["offsets_bits"]
        assert S.release_floors(m, c["coll"], c["n"], c["bytes"], k, 1000).tolist() == c["floors_now1000"]
        assert S.call_latency_us(m, c["coll"], c["n"], c["bytes"], k) == c["latency_us"]
    for coll, n, real, k in golden("delay.json")["to_real_counts"]:
        assert S.to_real_count(coll, n, real) == k


def test_host_delay_new_models_equal_oracle():
    """tree / hierarchical / reduce-scatter / broadcast are parity-unpinned by
    the reference: host and oracle must still agree bit for bit."""
    rng = random.Random(5)
    for _ in range(400):
        n = rng.choice([2, 3, 8, 16, 64, 128, 1024, rng.randint(2, 2000)])
        coll, algo, kind = rng.randrange(4), rng.randrange(3), rng.randrange(3)
        gpn = rng.choice([g for g in (1, 2, 4, 8, 16) if n % g == 0])
        args = (kind, algo, rng.random() * 20, rng.random() / 1e3, rng.random() / 1e4, rng.random() * 99,
                rng.choice([0.0, rng.random() * 1e4]), gpn, rng.random() * 3, rng.random() / 1e4)
        m1, m2 = S.delay_model(*args), P.delay_model(*args)
        nbytes = rng.randint(1, 1 << 34)
        real = sorted(rng.sample(range(n), min(n - 1, rng.randint(1, 8))))
        k = S.to_real_count(coll, n, real)
        assert k == P.to_real_count(coll, n, real)
        assert np.float64(S.model_total_us(m1, coll, n, nbytes)).view(np.uint64) == \
            np.float64(P.model_total_us(m2, coll, n, nbytes)).view(np.uint64)
        assert S.release_offsets(m1, coll, n, nbytes, k).view(np.uint64).tolist() == \
            P.release_offsets(m2, coll, n, nbytes, k).view(np.uint64).tolist()
        assert S.call_latency_us(m1, coll, n, nbytes, k) == P.call_latency_us(m2, coll, n, nbytes, k)


def test_c3_config_and_hierarchical_latency():
    """BASELINE config 3 as paper_2405_02969_b200.c3 builds it: 128 ranks =
    16 nodes x 8 GPUs, this node's k GPUs real; the host's hierarchical
    latency equals the oracle's and the model the B200 run recorded
    (profiles/r01_c3.json: 186 / 667 / 2135 us at 1 / 64 / 256 MiB)."""
    from paper_2405_02969_b200 import c3
    from paper_2405_02969_b200.fsdp import NET
    for k in (1, 2, 4):
        cfg = pb.JobConfig.parse(c3.config(k, True))
        assert cfg.world_size == 128 and cfg.real_ranks == list(range(k))
        assert "collective_algo = hierarchical" in cfg.render() and "topology.gpus_per_node = 8" in cfg.render()
        args = (S.ALPHA_BETA, S.HIERARCHICAL, NET["alpha_inter_us"], NET["beta_inter_us_per_byte"],
                NET["gamma_us_per_byte"], 0.0, 0.0, 8, NET["alpha_intra_us"], NET["beta_intra_us_per_byte"])
        m1, m2 = S.delay_model(*args), P.delay_model(*args)
        steps = S.to_real_count(S.ALLREDUCE, 128, list(range(k)))
        for mib, want in ((1, 186), (64, 667), (256, 2135)):
            got = S.call_latency_us(m1, S.ALLREDUCE, 128, mib << 20, steps)
            assert got == P.call_latency_us(m2, S.ALLREDUCE, 128, mib << 20, steps) == want, (k, mib, got)


def test_host_payload_equals_oracle():
    for key, j, word in golden("payload.json")["words"]:
        assert S.payload_word(key, j) == word
    for seed, rank, key in golden("payload.json")["keys"]:
        assert S.payload_key(seed, rank) == key


# ---- topology + ring order (config.cpp:314-376; test_config.cpp:120-165) -------
def _connected(n, edges):
    adj = {i: set() for i in range(n)}
    for s, d, *_ in edges:
        adj[s].add(d)
        adj[d].add(s)
    seen, stack = {0}, [0]
    while stack:
        for v in adj[stack.pop()] - seen:
            seen.add(v)
            stack.append(v)
    return len(seen) == n


def test_topology_covers_every_rank_and_stays_connected():
    cfg = pb.JobConfig.parse("world_size = 4\nreal_ranks = 0\nbucket_bytes = 8\nlink.alpha_us = 3\n")
    nodes, edges = cfg.topology()
    assert len(nodes) == 4 and [r for r, _ in nodes] == [True, False, False, False]
    assert all(nc == "default" for _, nc in nodes)
    assert _connected(4, edges) and all(e[2] == 3.0 for e in edges)


def test_topology_edge_structure_ignores_which_ranks_are_real():
    a = pb.JobConfig.parse("world_size = 8\nreal_ranks = 0\nbucket_bytes = 8\n").topology()[1]
    b = pb.JobConfig.parse("world_size = 8\nreal_ranks = 0,3,5\nbucket_bytes = 8\n").topology()[1]
    assert [(s, d) for s, d, *_ in a] == [(s, d) for s, d, *_ in b]
    assert _connected(8, a)


def test_ring_order_is_ascending_and_involutive():
    L = _capi.lib
    assert L.cemuRingSuccessor(4, 0) == 1 and L.cemuRingSuccessor(4, 3) == 0 and L.cemuRingPredecessor(4, 0) == 3
    for r in range(4):
        assert L.cemuRingSuccessor(4, L.cemuRingPredecessor(4, r)) == r
    assert L.cemuRingSuccessor(2, 0) == 1 and L.cemuRingSuccessor(2, 1) == 0


def test_exerciser_host_hash_equals_the_library_spec():
    """coll.py's vectorised payload words (its verify mode's expectation)
    equal cemuPayloadWord, including word indices past 2^32."""
    from paper_2405_02969_b200 import coll
    rng = random.Random(11)
    for _ in range(20):
        key = S.payload_key(rng.randrange(1 << 40), rng.randrange(4096))
        j0 = rng.choice([0, rng.randrange(1 << 31), (1 << 32) - 3, rng.randrange(1 << 40)])
        w = coll.payload_words(key, j0, 8)
        assert [int(v) for v in w] == [S.payload_word(key, j0 + i) for i in range(8)]
