"""FSDP all-gather / reduce-scatter trace at 1024 emulated ranks (BASELINE
config 5).  Parity unpinned: the reference has neither
reduce-scatter nor tree/hierarchical costs, and its O(n^3) boundary
projection cannot run at n = 1024; the closed forms here can.

One B200 is real rank 0 of a 1024-rank job training a Llama-3-8B-shaped
model with FSDP (full sharding, bf16 parameters and gradients):

  forward   all-gather unit i (prefetched while unit i-1 computes), compute
  backward  re-gather unit i (prefetched), compute (2x forward), then
            reduce-scatter its gradients; wait for every reduce-scatter

Compute is a chained %globaltimer spin on a compute stream (cemuSpinChainUs);
every collective is the real emulated collective through the C-ABI (device
synthesis of the 1023 emulated ranks' shards, device-evaluated delay model)
on an in-order comm stream.  The measured iteration time (device events) is
compared with the ideal timeline of the same schedule: compute exactly as
specified, each collective exactly its modelled latency (A14), in issue
order.  The what-if axes are the cost model (ring | tree | hierarchical 128
nodes x 8 GPUs) and the inter-node bandwidth (1x, 2x).

    python -m paper_2405_02969_b200.fsdp [--world 1024] [--iterations 2]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math

import numpy as np

from ._capi import lib

C_VOID = C.c_void_p
from . import whatif as _whatif  # noqa: F401  (declares cemuSpinChainUs / cemuCommModelLatencyUs)

LLAMA3_8B = {"hidden": 4096, "intermediate": 14336, "layers": 32, "heads": 32, "kv_heads": 8,
             "head_dim": 128, "vocab": 128256}

# Assumed cluster (documented in DESIGN.md): 128 nodes x 8 B200, NVLink 5
# inside a node (measured 770 GB/s peer), one 400 Gb/s NIC per GPU between
# nodes (50 GB/s), bf16 reduction at ~3 TB/s.
NET = {"alpha_inter_us": 5.0, "beta_inter_us_per_byte": 1 / 50e3, "alpha_intra_us": 2.0,
       "beta_intra_us_per_byte": 1 / 770e3, "gamma_us_per_byte": 1 / 3000e3, "gpus_per_node": 8}
TOKENS_PER_GPU = 8192
EFFECTIVE_TFLOPS = 800.0  # bf16, ~50% of the measured dense peak


def llama3_8b_units():
    """FSDP units in forward order: (name, parameter count)."""
    c = LLAMA3_8B
    h, kv = c["hidden"], c["kv_heads"] * c["head_dim"]
    attn = h * h + 2 * h * kv + h * h
    mlp = 3 * h * c["intermediate"]
    block = attn + mlp + 2 * h  # + two RMSNorm weights
    units = [("embed", c["vocab"] * h)]
    units += [(f"block{i}", block) for i in range(c["layers"])]
    units.append(("norm+head", h + c["vocab"] * h))
    return units


def unit_plan(units, world: int, tokens: int = TOKENS_PER_GPU, tflops: float = EFFECTIVE_TFLOPS):
    """Per unit: shard elements (bf16, padded to the world), forward/backward us."""
    plan = []
    for name, params in units:
        shard = math.ceil(params / world)
        fwd = 2.0 * params * tokens / (tflops * 1e12) * 1e6
        if name == "embed":  # a gather, not a GEMM
            fwd = max(1.0, tokens * LLAMA3_8B["hidden"] * 2 / 3e12 * 1e6)
        plan.append({"name": name, "params": params, "shard": shard, "fwd_us": round(fwd), "bwd_us": round(2 * fwd)})
    return plan


def cost_config(world: int, algo: str, bw_scale: float = 1.0) -> str:
    """Job config text for one what-if point."""
    lines = [f"world_size = {world}", "real_ranks = 0", "bucket_bytes = 1", "delay.kind = alpha_beta",
             f"collective_algo = {algo}",
             f"link.alpha_us = {NET['alpha_inter_us']!r}",
             f"link.beta_us_per_byte = {NET['beta_inter_us_per_byte'] / bw_scale!r}",
             f"link.gamma_us_per_byte = {NET['gamma_us_per_byte']!r}"]
    if algo == "hierarchical":
        lines += [f"topology.gpus_per_node = {NET['gpus_per_node']}",
                  f"link.intra.alpha_us = {NET['alpha_intra_us']!r}",
                  f"link.intra.beta_us_per_byte = {NET['beta_intra_us_per_byte']!r}"]
    return "\n".join(lines) + "\n"


def _latency(comm, coll: int, nbytes: int) -> float:
    v = C.c_int64()
    lib.cemuCommModelLatencyUs(comm._h, coll, nbytes, C.byref(v))
    return float(v.value)


def ideal_iteration_us(plan, lat_ag, lat_rs) -> float:
    """The schedule's critical path with modelled collective latencies."""
    U = len(plan)
    t = 0.0          # compute stream
    net = 0.0        # comm stream (in order)

    def coll(issue, lat):
        nonlocal net
        net = max(net, issue) + lat
        return net

    ag = [0.0] * U
    ag[0] = coll(0.0, lat_ag[0])
    for i in range(U):
        t = max(t, ag[i])
        if i + 1 < U:
            ag[i + 1] = coll(t, lat_ag[i + 1])
        t += plan[i]["fwd_us"]
    agb = [0.0] * U
    agb[U - 1] = coll(t, lat_ag[U - 1])
    last = 0.0
    for i in reversed(range(U)):
        t = max(t, agb[i])
        if i > 0:
            agb[i - 1] = coll(t, lat_ag[i - 1])
        t += plan[i]["bwd_us"]
        last = coll(t, lat_rs[i])
    return max(t, last)


def run_trace(comm, plan, iterations: int = 2, device: int = 0):
    """Enqueue the FSDP schedule on the device; per-iteration times (us)."""
    import torch
    W = comm.world_size
    compute, net = torch.cuda.Stream(device), torch.cuda.Stream(device)
    chain = torch.zeros(1, dtype=torch.int64, device=device)
    max_shard = max(u["shard"] for u in plan)
    full = torch.zeros(max_shard * W, dtype=torch.bfloat16, device=device)
    shard = torch.zeros(max_shard, dtype=torch.bfloat16, device=device)
    rs_out = torch.zeros(max_shard, dtype=torch.bfloat16, device=device)
    U = len(plan)
    state = {"resync": True}

    def spin(us):
        lib.cemuSpinChainUs(compute.cuda_stream, int(us), C.c_void_p(chain.data_ptr()), int(state["resync"]))
        state["resync"] = False

    def issue_from_compute(fn):
        e = torch.cuda.Event()
        e.record(compute)
        net.wait_event(e)
        fn()
        d = torch.cuda.Event()
        d.record(net)
        end = C_VOID()
        lib.cemuCommLastReleaseEnd(comm._h, C.byref(end))
        return d, end

    def ag(i):
        s = plan[i]["shard"]
        return lambda: comm.all_gather(shard[:s], full[:s * W], stream=net)

    def rs(i):
        s = plan[i]["shard"]
        return lambda: comm.reduce_scatter(full[:s * W], rs_out[:s], stream=net)

    def wait(d):
        ev, end = d
        compute.wait_event(ev)
        if end.value and not state["resync"]:
            # continue the compute chain from max(its deadline, the
            # collective's release end), not after the event-to-kernel gap
            lib.cemuChainJoin(compute.cuda_stream, C.c_void_p(chain.data_ptr()), end)
        else:
            state["resync"] = True

    starts, ends = [], []
    for _ in range(iterations):
        st = torch.cuda.Event(enable_timing=True)
        st.record(compute)
        starts.append(st)
        d_ag = [None] * U
        d_ag[0] = issue_from_compute(ag(0))
        for i in range(U):
            wait(d_ag[i])
            if i + 1 < U:
                d_ag[i + 1] = issue_from_compute(ag(i + 1))
            spin(plan[i]["fwd_us"])
        d_agb = [None] * U
        d_agb[U - 1] = issue_from_compute(ag(U - 1))
        last = None
        for i in reversed(range(U)):
            wait(d_agb[i])
            if i > 0:
                d_agb[i - 1] = issue_from_compute(ag(i - 1))
            spin(plan[i]["bwd_us"])
            last = issue_from_compute(rs(i))
        wait(last)
        en = torch.cuda.Event(enable_timing=True)
        en.record(compute)
        ends.append(en)
    torch.cuda.synchronize(device)
    return [s.elapsed_time(e) * 1e3 for s, e in zip(starts, ends)]


def whatif_table(world: int = 1024, iterations: int = 2, device: int = 0, units=None):
    """Iteration time per (cost model, inter-node bandwidth), measured on the
    device and ideal; plus per-collective modelled latencies of one block."""
    from .comm import Communicator
    units = units or llama3_8b_units()
    plan = unit_plan(units, world)
    rows = []
    for algo in ("ring", "tree", "hierarchical"):
        for scale in (1.0, 2.0):
            comm = Communicator(cost_config(world, algo, scale), 0, device)
            # the trace issues every collective on one in-order comm stream:
            # model that channel (a queued collective starts on the wire when
            # the previous one leaves it; cemuCommSetQueueChaining)
            comm.set_queue_chaining(10)
            lat_ag = [_latency(comm, 1, u["shard"] * 2) for u in plan]
            lat_rs = [_latency(comm, 2, u["shard"] * 2 * world) for u in plan]
            ideal = ideal_iteration_us(plan, lat_ag, lat_rs)
            meas = run_trace(comm, plan, iterations, device)
            comm.close()
            m = float(np.mean(meas[1:] if len(meas) > 1 else meas))
            blk = next(i for i, u in enumerate(plan) if u["name"].startswith("block"))
            rows.append({"algo": algo, "inter_bw_x": scale, "iteration_ms": round(m / 1e3, 3),
                         "ideal_ms": round(ideal / 1e3, 3), "rel_err": abs(m - ideal) / ideal,
                         "block_allgather_ms": round(lat_ag[blk] / 1e3, 3),
                         "block_reducescatter_ms": round(lat_rs[blk] / 1e3, 3)})
    return {"world": world, "units": len(plan), "params": int(sum(p for _, p in units)),
            "tokens_per_gpu": TOKENS_PER_GPU, "effective_tflops": EFFECTIVE_TFLOPS,
            "compute_ms_per_iteration": round(sum(u["fwd_us"] + u["bwd_us"] for u in plan) / 1e3, 3),
            "network": NET, "rows": rows, "max_rel_err": max(r["rel_err"] for r in rows)}


def main():
    ap = argparse.ArgumentParser(description="FSDP Llama-3-8B trace at 1024 emulated ranks")
    ap.add_argument("--world", type=int, default=1024)
    ap.add_argument("--iterations", type=int, default=2)
    a = ap.parse_args()
    res = whatif_table(a.world, a.iterations)
    for r in res["rows"]:
        print(f"{r['algo']:12s} inter bw x{r['inter_bw_x']:.0f}: iteration {r['iteration_ms']:9.3f} ms "
              f"(ideal {r['ideal_ms']:9.3f}, err {100 * r['rel_err']:.3f}%)  block AG {r['block_allgather_ms']} ms, "
              f"RS {r['block_reducescatter_ms']} ms")
    print(json.dumps({k: v for k, v in res.items() if k != "rows"}))


if __name__ == "__main__":
    main()
