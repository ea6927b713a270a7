"""Diagnose the ResNet-50 what-if overhead: per-bucket issue/complete vs the
ideal timeline, repeated Communicators at the same inject."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch  # noqa: F401,E402

from paper_2405_02969_b200.comm import Communicator  # noqa: E402
from paper_2405_02969_b200.whatif import ModelSpec, run_loop, predicted_us  # noqa: E402
import ctypes as C  # noqa: E402
from paper_2405_02969_b200._capi import lib  # noqa: E402

ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo")
spec = ModelSpec.load(os.path.join(ROOT, "profiles", "resnet50.model"))
info = spec.layers()
bb = 25 << 20
extra = "delay.kind = alpha_beta\nlink.alpha_us = 10\nlink.beta_us_per_byte = 0.00004\n"
bks = spec.buckets(bb)
out = {"buckets": bks, "fwd_sum": int(info["forward_us"].sum()), "bwd_sum": int(info["backward_us"].sum()),
       "runs": []}
for d in [0, 500, 0, 500, 2000, 2000, 2000]:
    cfg = f"world_size = 8\nreal_ranks = 0\nbucket_bytes = {bb}\ndelay.inject_us = {float(d)!r}\n" + extra
    comm = Communicator(cfg, 0, 0)
    lats = []
    for _, _, nbytes in bks:
        v = C.c_int64()
        lib.cemuCommModelLatencyUs(comm._h, 0, nbytes, C.byref(v))
        lats.append(int(v.value))
    r = run_loop(comm, spec, bb)
    ideal = predicted_us(comm, spec, bb)
    comm.close()
    wu = info["warmup"]
    it = r["iter_us"][wu:]
    # per-iteration relative bucket times (issue/complete from iteration start), averaged
    iss = (r["issue_us"][wu:] - r["start_us"][wu:, None]).mean(0)
    com = (r["complete_us"][wu:] - r["start_us"][wu:, None]).mean(0)
    gap = (r["start_us"][wu + 1:] - r["end_us"][wu:-1]).mean()
    out["runs"].append({"inject": d, "lat": lats, "ideal": ideal, "mean": float(it.mean()),
                        "std": float(it.std(ddof=1)), "min": float(it.min()), "max": float(it.max()),
                        "issue_rel": [round(x, 1) for x in iss], "complete_rel": [round(x, 1) for x in com],
                        "dur": [round(c - i, 1) for c, i in zip(com, iss)], "inter_iter_gap": float(gap)})
    print(json.dumps(out["runs"][-1]), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/whatif_diag.json", "w"), indent=1)
