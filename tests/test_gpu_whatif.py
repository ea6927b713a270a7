"""GPU: the DDP what-if loop (BASELINE config 4).

The device loop must reproduce the ideal timeline of the same schedule --
compute exactly as profiled, every bucket's collective exactly its modelled
latency -- to within the north star's 1% end-to-end step-time error, and the
sweep must have the reference's what-if shape (cemu_bench.cpp:457-480: tail
slope within [0.9, 1.1] x buckets, marginal slope below the bucket count,
monotone)."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2405_02969_b200 as pb
from paper_2405_02969_b200.whatif import ModelSpec, run_loop, sweep

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bert_like_whatif_sweep(cuda, tmp_path):
    # acceptance criterion 7's sweep (acceptance_main.cpp:323-334)
    res = sweep("bert-like", [0, 500, 1000, 4000, 6000, 8000, 10000], world=2, bucket_bytes=65536,
                iterations=30, trace_csv=str(tmp_path / "trace.csv"))
    from paper_2405_02969_b200.whatif import read_iteration_csv
    tr = read_iteration_csv(str(tmp_path / "trace_inject4000.csv"))  # reference columns, 30 x 4 rows
    assert len(tr) == 30 and all(len(t["buckets"]) == 4 for t in tr.values())
    assert res["buckets"] == 4 and res["knee_us"] == 2000
    assert res["checks_pass"], res
    assert res["max_rel_err"] < 0.01, res
    assert 0.9 * 4 <= res["tail_slope"] <= 1.1 * 4


def test_resnet50_25MiB_buckets_whatif(cuda):
    model = os.path.join(ROOT, "profiles", "resnet50.model")
    res = sweep(model, [0, 500, 1000, 2000, 4000, 6000, 8000, 10000], world=8, bucket_bytes=25 << 20,
                iterations=20, extra_config="delay.kind = alpha_beta\nlink.alpha_us = 10\n"
                                            "link.beta_us_per_byte = 0.00004\n")
    assert res["buckets"] == 5
    assert res["max_rel_err"] < 0.01, [(p["inject_us"], p["mean_us"], p["ideal_us"]) for p in res["points"]]
    assert res["checks_pass"], res


def test_loop_trace_respects_modelled_latency(cuda):
    comm = pb.Communicator("world_size = 4\nreal_ranks = 0\nbucket_bytes = 65536\ndelay.inject_us = 700\n", 0, 0)
    spec = ModelSpec.load("bert-like")
    r = run_loop(comm, spec, 65536)
    issue, done = r["issue_us"], r["complete_us"]
    assert issue.shape == (60, 4)
    # each bucket completes >= 700 us after it could start (in-order comm stream)
    start = np.maximum(issue, np.concatenate([np.zeros((60, 1)), done[:, :-1]], axis=1))
    assert np.all(done - start >= 700 - 1)
    assert np.all(done - start <= 700 + 30)
    comm.close()
