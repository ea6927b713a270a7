"""DDP what-if with real compute (paper_2405_02969_b200.ddp): a bf16 MLP's
gradients, bucketed by autograd hooks and all-reduced by the emulated
collective on a comm stream, equal the oracle's allreduce of the local
gradients; the injected-delay sweep exposes one stall per bucket (tail slope
~ bucket count, the cemu-bench what-if criterion, cemu_bench.cpp:457-480)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2405_02969_b200 as pb
from gpu_util import to_np
from oracle import port as P
from paper_2405_02969_b200 import ddp as D

pytestmark = pytest.mark.gpu


def test_bucketed_gradients_equal_the_oracle_allreduce(cuda):
    torch.manual_seed(0)
    model = D.build_model(3, 512, "cuda")
    x = torch.randn(256, 512, device="cuda", dtype=torch.bfloat16)
    model(x).float().pow(2).mean().backward()
    local = {p: p.grad.detach().clone() for p in model.parameters()}
    model.zero_grad(set_to_none=False)
    W = 8
    comm = pb.Communicator(f"world_size = {W}\nreal_ranks = 0\nbucket_bytes = 1\n", 0, 0)
    ddp = D.EmulatedDDP(model, comm, bucket_bytes=600 * 1024)  # 512x512 bf16 = 512 KiB: one param per bucket
    model(x).float().pow(2).mean().backward()
    ddp.finish()
    torch.cuda.synchronize()
    assert len(ddp.buckets) == 3
    for b in ddp.buckets:
        flat = torch.cat([local[p].view(-1) for p in b])
        want = P.allreduce(9, P.PAYLOAD_HASH, W, [0], 0, 1, [to_np(flat)], flat.numel())
        got = torch.cat([p.grad.view(-1) for p in b])
        assert np.array_equal(to_np(got), want)
    ddp.close()
    comm.close()


def test_real_compute_whatif_tail_slope_is_the_bucket_count(cuda):
    r = D.run(layers=4, width=2048, tokens=4096, bucket_mib=8, world=8, delays_us=(0, 4000, 8000, 12000),
              iterations=6, warmup=2)
    B = r["buckets"]
    assert B == 4
    assert 0.95 * B <= r["tail_slope"] <= 1.05 * B, r
    means = [p["mean_us"] for p in r["points"]]
    assert means == sorted(means)
