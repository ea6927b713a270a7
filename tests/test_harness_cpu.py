"""The DDP what-if harness's host side (CPU): model-spec format and bucketing
equal the reference's (proj/src/harness.cpp:27-189), and the ideal-timeline
predictor agrees with a hand-computed schedule."""
from __future__ import annotations

import os
import random

import pytest

from oracle import ref as R
from paper_2405_02969_b200 import CemuError
from paper_2405_02969_b200.whatif import ModelSpec

needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built here")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _random_model(rng):
    n = rng.randint(1, 40)
    lines = [f"name = m{rng.randrange(1000)}", f"iterations = {rng.randint(2, 90)}", "warmup = 1",
             f"update_us = {rng.randrange(500)}"]
    lines += [f"layer = {rng.randrange(3000)} {rng.randrange(3000)} {rng.randrange(1 << 22)}" for _ in range(n)]
    return "# random\n" + "\n".join(lines) + "\n"


@needs_ref
def test_model_spec_render_and_buckets_equal_reference():
    rng = random.Random(12)
    texts = [open(os.path.join(ROOT, "profiles", "resnet50.model")).read()]
    for name in ("bert-like", "small", "wide"):
        texts.append(ModelSpec.load(name).render())
    texts += [_random_model(rng) for _ in range(50)]
    for t in texts:
        spec = ModelSpec.parse(t)
        assert spec.render() == R.model_render(t)
        for bb in (1, 4096, 65536, 1 << 20, 25 << 20, 1 << 40):
            assert spec.buckets(bb) == R.bucketize(t, bb), bb


def test_builtin_profiles_match_shipped_files():
    # proj/profiles/*.model are the built-ins written out (harness.cpp:116-134)
    shipped = {"bert-like": (4, 1000, 2000, 65536), "small": (2, 1000, 2000, 32768), "wide": (16, 1000, 1000, 65536)}
    for name, (n, f, b, g) in shipped.items():
        info = ModelSpec.load(name).layers()
        assert len(info["forward_us"]) == n and set(info["forward_us"]) == {f}
        assert set(info["backward_us"]) == {b} and set(info["grad_bytes"]) == {g}
        assert info["iterations"] == 60 and info["warmup"] == 10


def test_model_spec_errors():
    with pytest.raises(CemuError, match="layer"):
        ModelSpec.parse("iterations = 2\nlayer = 1 2\n")
    with pytest.raises(CemuError, match="warmup"):
        ModelSpec.parse("iterations = 2\nwarmup = 2\nlayer = 1 2 3\n")
    with pytest.raises(CemuError, match="bogus"):
        ModelSpec.parse("iterations = 2\nbogus = 1\nlayer = 1 2 3\n")


def test_predicted_timeline_hand_computed():
    import ctypes as C

    import numpy as np

    from paper_2405_02969_b200._capi import lib
    spec = ModelSpec.load("bert-like")  # 4 x (F=1000, B=2000, 64 KiB), one bucket per layer
    for d in (0.0, 500.0, 1000.0, 2000.0, 5000.0):
        lat = np.full(4, d)
        got = lib.cemuPredictIterationUs(spec._h, 65536, lat.ctypes.data, 4)
        # forward 4000; bucket b issues at 4000 + 2000 (b+1); comm in order
        t, free = 4000.0, 0.0
        for _ in range(4):
            t += 2000
            free = max(t, free) + d
        assert got == max(t, free)
    assert lib.cemuPredictIterationUs(spec._h, 65536, np.zeros(4).ctypes.data, 4) == 12000.0
    _ = C


def test_iteration_csv_round_trip_and_stats(tmp_path):
    """write_iteration_csv / read_iteration_csv / iteration_stats with the
    reference's columns and semantics (harness.cpp:256-319)."""
    import numpy as np
    from paper_2405_02969_b200 import whatif as W
    trace = {"start_us": np.array([0.0, 1000.4, 2100.0]), "end_us": np.array([990.0, 2080.0, 3300.6]),
             "issue_us": np.array([[10.0, 500.0], [1010.0, 1600.0], [2110.0, 2700.0]]),
             "complete_us": np.array([[400.0, 980.0], [1500.0, 2070.0], [2600.0, 3290.0]])}
    trace["iter_us"] = trace["end_us"] - trace["start_us"]
    p = tmp_path / "t.csv"
    W.write_iteration_csv(str(p), trace)
    lines = p.read_text().splitlines()
    assert lines[0] == "iter,start_us,end_us,bucket_id,issue_us,complete_us" and len(lines) == 7
    back = W.read_iteration_csv(str(p))
    assert sorted(back) == [0, 1, 2] and back[1]["buckets"] == [(0, 1010, 1500), (1, 1600, 2070)]
    st = W.iteration_stats(trace, warmup=1)
    assert st["count"] == 2 and abs(st["mean_us"] - np.mean(trace["iter_us"][1:])) < 1e-9


@needs_ref
def test_reference_loop_in_a_bounded_process():
    """bench.py's what-if comparison arm runs the reference's own
    run_training_loop in a separate, killable process (oracle/ref_loop.py):
    per-iteration times come back as JSON; a bad model is a nonzero exit
    with the reference's error, not an exception in the bench."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = ModelSpec.load("bert-like").render()
    lines = [ln for ln in text.splitlines() if not ln.startswith(("iterations", "warmup"))]
    short = "\n".join(lines + ["iterations = 4", "warmup = 1"]) + "\n"
    r = subprocess.run([sys.executable, "-m", "oracle.ref_loop"], cwd=root, text=True, capture_output=True, timeout=120,
                       input=json.dumps({"text": short, "world": 2, "bucket_bytes": 65536, "inject": 100.0}))
    assert r.returncode == 0, r.stderr
    it = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(it) == 4 and all(t > 0 for t in it)
    bad = subprocess.run([sys.executable, "-m", "oracle.ref_loop"], cwd=root, text=True, capture_output=True,
                         timeout=60, input=json.dumps({"text": "nonsense = 1\n", "world": 2, "bucket_bytes": 65536,
                                                       "inject": 0}))
    assert bad.returncode == 1 and bad.stderr.strip()
