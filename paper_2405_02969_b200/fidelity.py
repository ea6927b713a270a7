"""Emulated-vs-baseline fidelity (the reference's
cemu-bench `microbench` and `e2e` commands, proj/tools/cemu_bench.cpp:196-290
and :346-380).

Run under torch.distributed.run with k processes, one per GPU (k = 2 or 4):

  baseline (B)  all k ranks real: every collective is NCCL over NVLink
                (torch.distributed, real payloads) -- the job as it would run.
  emulated (E)  rank 0 alone: its world has k ranks, ranks 1..k-1 emulated
                (synthesised payloads, cemuAllReduce), and the network delay
                comes from B's own measurements, as NeuronaBox calibrates its
                profiles: (ab) the alpha-beta ring model fitted to B's size
                sweep, (table) B's measured latency table interpolated by a
                delay-model plugin (cemuCommSetDelayModel).

microbench   per-call latency of back-to-back allreduces, 4 KiB .. 256 MiB,
             baseline and emulated segments alternating (cemu_bench.cpp:
             214-234); the reference's check: emulated / baseline <= 1.05 at
             >= 2 MiB (:281).
e2e          per-iteration time of the same training loop in both modes
             (:346-380): the reference's bert-like profile and a ResNet-50
             profile with 25 MiB buckets (spin-kernel compute on a compute
             stream, bucket allreduces on an in-order comm stream, wait-all
             before the update -- harness.cpp:191-254), and a real bf16 MLP
             trained with DDP-style gradient buckets (ddp.py).  rel_err =
             |E - B| / B; the reference gates at 5%, the north star at 1%.

The emulated comm stream is an in-order channel, so queue chaining is on
(cemuCommSetQueueChaining): a collective queued behind the previous one
starts when that one leaves the wire, as NCCL's next kernel does.  Beside
real compute the emulated collective also takes the SMs NCCL's kernel would
(cemuCommSetDelayFootprint with NCCL's measured launch: 32 CTAs, ~101 KB
shared memory each), from the call's start to its modelled end.

    python -m torch.distributed.run --nproc-per-node 2 -m paper_2405_02969_b200.fidelity
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os

import numpy as np
import torch
import torch.distributed as dist

from .comm import Communicator
from .whatif import ModelSpec, lib as _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = [4 << 10, 16 << 10, 64 << 10, 256 << 10, 1 << 20, 2 << 20, 4 << 20, 8 << 20, 16 << 20, 32 << 20,
         64 << 20, 128 << 20, 256 << 20]


# ---------------------------------------------------------------------------
# collectives of the two modes
# ---------------------------------------------------------------------------
class NcclAllReduce:
    """Baseline collective: NCCL allreduce of the real payload, ordered on
    `stream` (the comm stream waits for it; the host does not)."""

    def all_reduce(self, t, recv=None, stream=None):
        s = stream or torch.cuda.current_stream()
        with torch.cuda.stream(s):
            dist.all_reduce(t)
        return t


def fit_alpha_beta(sizes, us, k):
    """Least squares (relative residuals) of T(m) = a + b m, mapped onto the
    ring allreduce model 2(k-1) alpha + 2 (k-1)/k m beta (gamma = 0)."""
    m = np.asarray(sizes, dtype=np.float64)
    t = np.asarray(us, dtype=np.float64)
    A = np.stack([np.ones_like(m), m], axis=1) / t[:, None]
    (a, b), *_ = np.linalg.lstsq(A, np.ones_like(t), rcond=None)
    a, b = max(a, 0.0), max(b, 0.0)
    a, b = float(a), float(b)
    return {"alpha_us": a / (2 * (k - 1)), "beta_us_per_byte": b * k / (2 * (k - 1)), "a_us": a, "b_us_per_byte": b}


def ab_config(k, fit):
    return (f"world_size = {k}\nreal_ranks = 0\nbucket_bytes = 1\ndelay.kind = alpha_beta\n"
            f"link.alpha_us = {fit['alpha_us']!r}\nlink.beta_us_per_byte = {fit['beta_us_per_byte']!r}\n"
            "link.gamma_us_per_byte = 0\n")


def table_plugin(sizes, us):
    """Delay-model plugin: B's measured latency at `bytes`, interpolated
    log-log between measured sizes (extrapolated from the end segments);
    released evenly over the K to-real steps like the built-in models."""
    lx, ly = np.log(np.asarray(sizes, np.float64)), np.log(np.asarray(us, np.float64))

    def at(nbytes):
        x = np.log(max(float(nbytes), 1.0))
        if x <= lx[0]:
            i = 0
        elif x >= lx[-1]:
            i = len(lx) - 2
        else:
            i = int(np.searchsorted(lx, x)) - 1
        w = (x - lx[i]) / (lx[i + 1] - lx[i])
        return float(np.exp(ly[i] + w * (ly[i + 1] - ly[i])))

    def fn(coll, n, nbytes, k):
        total = at(nbytes)
        return [total * (j + 1) / k for j in range(k)]
    fn.at = at
    return fn


# ---------------------------------------------------------------------------
# microbench
# ---------------------------------------------------------------------------
def per_call_us(call, reps, graph=True):
    """Device time per call of `reps` back-to-back calls, graph-captured (the
    host's launch path out of the measurement) or, if capture fails, eager."""
    s = torch.cuda.Stream()
    for _ in range(3):
        call(s)
    torch.cuda.synchronize()
    used_graph = False
    if graph:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    call(s)
            g.replay()
            torch.cuda.synchronize()
            used_graph = True
        except Exception:  # noqa: BLE001 -- reported through `graph` in the output
            torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        if used_graph:
            g.replay()
        else:
            for _ in range(reps):
                call(s)
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps, used_graph


def baseline_sweep(sizes, reps):
    out = []
    for size in sizes:
        x = torch.ones(size // 4, dtype=torch.float32, device="cuda")
        dist.barrier()
        us, g = per_call_us(lambda s: NcclAllReduce().all_reduce(x, stream=s), reps)
        out.append((us, g))
        del x
    return out


def emulated_sweep(comm, sizes, reps):
    out = []
    for size in sizes:
        x = torch.ones(size // 4, dtype=torch.float32, device="cuda")
        us, g = per_call_us(lambda s: comm.all_reduce(x, stream=s), reps)
        out.append((us, g))
        del x
    return out


# ---------------------------------------------------------------------------
# e2e: the training loops
# ---------------------------------------------------------------------------
def spin_loop(spec: ModelSpec, bucket_bytes: int, coll, iterations: int, warmup: int):
    """The harness's training loop (harness.cpp:191-254) in either mode:
    compute = chained %globaltimer spins on a compute stream, one allreduce
    per full gradient bucket on an in-order comm stream, wait-all before the
    update.  Returns per-iteration times (us) after warm-up."""
    info = spec.layers()
    fwd, bwd, upd = info["forward_us"], info["backward_us"], info["update_us"]
    buckets = spec.buckets(bucket_bytes)
    compute, net = torch.cuda.Stream(), torch.cuda.Stream()
    chain = torch.zeros(1, dtype=torch.int64, device="cuda")
    bufs = [torch.zeros(max(b[2] // 4, 1), dtype=torch.float32, device="cuda") for b in buckets]
    state = {"resync": True}

    def spin(us):
        if us > 0:
            _lib.cemuSpinChainUs(compute.cuda_stream, int(us), C.c_void_p(chain.data_ptr()), int(state["resync"]))
            state["resync"] = False

    starts, ends = [], []
    for _ in range(warmup + iterations):
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record(compute)
        for us in fwd:
            spin(us)
        nxt = 0
        done = None
        for i in reversed(range(len(bwd))):
            spin(bwd[i])
            if nxt < len(buckets) and buckets[nxt][0] == i:
                ev = torch.cuda.Event()
                ev.record(compute)
                net.wait_event(ev)
                coll.all_reduce(bufs[nxt], stream=net)
                done = torch.cuda.Event()
                done.record(net)
                nxt += 1
        if done is not None:
            compute.wait_event(done)  # wait-all: the comm stream is in order
            state["resync"] = True
        spin(upd)
        en.record(compute)
        starts.append(st)
        ends.append(en)
    torch.cuda.synchronize()
    return [s.elapsed_time(e) * 1e3 for s, e in zip(starts, ends)][warmup:]


class _ServiceTimed:
    """Wraps a collective: each call's service time on its (in-order) comm
    stream, from the stream reaching it to its end -- event pairs, read
    after the run so the host never waits inside it."""

    def __init__(self, inner):
        self.inner, self.events = inner, []

    def all_reduce(self, t, recv=None, stream=None):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        self.inner.all_reduce(t, recv, stream=stream)
        b.record(stream)
        self.events.append((t.numel() * t.element_size(), a, b))
        return t

    def samples(self):
        return [(n, a.elapsed_time(b) * 1e3) for n, a, b in self.events]


def mlp_loop(coll, iterations: int, warmup: int, layers=8, width=4096, tokens=8192, bucket_mib=25,
             service=None):
    """A real bf16 MLP (tensor-core GEMMs) trained with DDP-style gradient
    buckets (ddp.py) whose allreduces are `coll`'s.  With `service` (a list),
    each timed bucket collective's (bytes, service us) is appended to it."""
    from .ddp import EmulatedDDP, build_model
    torch.manual_seed(0)
    model = build_model(layers, width, "cuda")
    x = torch.randn(tokens, width, device="cuda", dtype=torch.bfloat16)
    opt = torch.optim.SGD(model.parameters(), lr=1e-6)
    ddp = EmulatedDDP(model, coll, bucket_mib << 20)

    def step():
        opt.zero_grad(set_to_none=False)
        model(x).float().pow(2).mean().backward()
        ddp.finish()
        opt.step()

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    timer = _ServiceTimed(coll) if service is not None else None
    if timer is not None:
        ddp.comm = timer
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(iterations + 1)]
    ev[0].record()
    for i in range(iterations):
        step()
        ev[i + 1].record()
    torch.cuda.synchronize()
    ddp.close()
    if timer is not None:
        service.extend(timer.samples())
    return [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(iterations)]


def loaded_sweep(sizes, reps):
    """NCCL per-call latency while bf16 GEMMs run on another stream of every
    rank (a collective beside a training step's compute is slower than an
    idle one: SMs, L2 and HBM are shared)."""
    a = torch.randn(8192, 4096, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    side = torch.cuda.Stream()
    out = []
    for size in sizes:
        x = torch.ones(size // 4, device="cuda")
        s = torch.cuda.Stream()
        for _ in range(3):
            NcclAllReduce().all_reduce(x, stream=s)
        torch.cuda.synchronize()
        dist.barrier()
        with torch.cuda.stream(side):
            for _ in range(60):
                a = (a @ w) * 0.001
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            for _ in range(reps):
                NcclAllReduce().all_reduce(x, stream=s)
            e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3 / reps)
        del x
    return out


def size_plugin(samples):
    """Delay-model plugin from (bytes, us) samples: the mean per distinct size,
    log-log interpolated between sizes (table_plugin)."""
    by = {}
    for b, u in samples:
        by.setdefault(int(b), []).append(u)
    sizes = sorted(by)
    us = [float(np.mean(by[b])) for b in sizes]
    if len(sizes) == 1:  # one bucket size: constant
        sizes, us = [sizes[0] // 2, sizes[0] * 2], [us[0], us[0]]
    return table_plugin(sizes, us), dict(zip(map(int, sizes), us))


def e2e_models():
    return [("bert-like", "bert-like", 65536), ("resnet50_25MiB", os.path.join(ROOT, "profiles", "resnet50.model"),
                                                 25 << 20)]


# ---------------------------------------------------------------------------
def emulated_comm(k, fit=None, plugin=None, footprint=(0, 0)):
    """Rank 0's emulated world of k ranks (1 real), delay from the fitted
    alpha-beta model or a plugin; in-order comm stream (queue chaining)."""
    if plugin is None:
        comm = Communicator(ab_config(k, fit), 0, torch.cuda.current_device())
    else:
        comm = Communicator(f"world_size = {k}\nreal_ranks = 0\nbucket_bytes = 1\n", 0, torch.cuda.current_device())
        comm.set_delay_model(plugin)
    comm.set_queue_chaining(10)
    comm.set_delay_footprint(*footprint)
    return comm


# NCCL's allreduce-path kernel on these boxes (ncu launch attributes,
# profiles/r02_ncu_nccl_kernel_launch.csv): 32 CTAs (its channels) of 544
# threads, 82,240 B dynamic + 21,568 B static shared memory each.
NCCL_FOOTPRINT = (32, 82240 + 21568)


def mlp_fidelity(k, rank, barrier, sizes, plugin, loaded, mlp_iters, footprint):
    """One repeat of the real-compute MLP check: the NCCL baseline before and
    after the emulated runs (pooled, drift-bracketed; both halves feed the
    in-situ calibration), the emulated loop under each calibration, and
    compute alone.  Rank 0's row (other ranks: {})."""
    service = []
    barrier()
    base = mlp_loop(NcclAllReduce(), mlp_iters, 3, service=service)
    barrier()
    row = {"model": "mlp_bf16_8x4096_25MiB"}
    modes = ()
    if rank == 0:
        insitu, insitu_us = size_plugin(service)
        row["loaded_calibration_us"] = [round(u, 2) for u in loaded]
        row["in_situ_service_us"] = {str(b): round(u, 2) for b, u in insitu_us.items()}
        row["footprint"] = {"ctas": footprint[0], "smem_bytes": footprint[1]}
        modes = (("table", {"plugin": plugin}, (0, 0)),
                 ("table_footprint", {"plugin": plugin}, footprint),
                 ("loaded_footprint", {"plugin": table_plugin(sizes, loaded)}, footprint),
                 ("in_situ_footprint", {"plugin": insitu}, footprint))
        emus = {}
        for tag, kw, fp in modes:
            comm = emulated_comm(k, footprint=fp, **kw)
            emus[tag] = mlp_loop(comm, mlp_iters, 3)
            comm.close()
        comp = mlp_loop(type("ComputeOnly", (), {"all_reduce": lambda self, t, recv=None, stream=None: t})(),
                        mlp_iters, 3)
        row["compute_only_mean_us"] = float(np.mean(comp))
    barrier()
    base2 = mlp_loop(NcclAllReduce(), mlp_iters, 3)
    barrier()
    if rank == 0:
        pooled = list(base) + list(base2)
        bm = float(np.mean(pooled))
        row["baseline_mean_us"] = bm
        row["baseline_halves_mean_us"] = [float(np.mean(base)), float(np.mean(base2))]
        row["baseline_stddev_us"] = float(np.std(pooled, ddof=1))
        # the baseline mean's own uncertainty: two standard errors, relative
        # (iterations with real GEMMs beside NCCL vary by a few percent)
        row["baseline_noise_2sem_rel"] = float(2 * np.std(pooled, ddof=1) / np.sqrt(len(pooled)) / bm)
        row["iterations"] = {"baseline": len(pooled), "emulated": mlp_iters}
        for tag, *_ in modes:
            row[f"emulated_{tag}_mean_us"] = float(np.mean(emus[tag]))
            row[f"rel_err_{tag}"] = float(abs(np.mean(emus[tag]) - bm) / bm)
    barrier()
    return row


def run(sizes=None, reps=100, segments=3, e2e_iters=20, mlp_iters=100, footprint=NCCL_FOOTPRINT,
        mlp_repeats=1):
    sizes = sizes or SIZES
    rank, k = dist.get_rank(), dist.get_world_size()
    host = dist.new_group(backend="gloo")

    def barrier():
        dist.barrier(group=host)

    res = {"k": k, "sizes": sizes, "reps": reps, "segments": segments}
    # --- calibration: idle sweeps (alpha-beta fit + table); the per-size
    # median of three keeps one noisy sweep out of the profile --------------
    calib = [float(u) for u in np.median([[u for u, _ in baseline_sweep(sizes, reps)] for _ in range(3)], axis=0)]
    fit = fit_alpha_beta(sizes, calib, k)
    plugin = table_plugin(sizes, calib)
    res["fit"] = fit
    res["calibration_us"] = [round(u, 3) for u in calib]
    # --- microbench: baseline and emulated segments alternate -------------
    base_seg, ab_seg, tab_seg = [], [], []
    for seg in range(segments):
        b = baseline_sweep(sizes, reps)
        base_seg.append([u for u, _ in b])
        res["baseline_graph"] = all(g for _, g in b)
        barrier()
        if rank == 0:
            for acc, kw in ((ab_seg, {"fit": fit}), (tab_seg, {"plugin": plugin})):
                comm = emulated_comm(k, **kw)
                acc.append([u for u, _ in emulated_sweep(comm, sizes, reps)])
                comm.close()
        barrier()
    if rank == 0:
        B = np.mean(base_seg, axis=0)
        Eab, Etab = np.mean(ab_seg, axis=0), np.mean(tab_seg, axis=0)
        res["microbench"] = [{"bytes": s, "baseline_us": round(float(b), 3), "emulated_ab_us": round(float(e1), 3),
                              "emulated_table_us": round(float(e2), 3), "ratio_ab": round(float(e1 / b), 4),
                              "ratio_table": round(float(e2 / b), 4)}
                             for s, b, e1, e2 in zip(sizes, B, Eab, Etab)]
        big = [r for r in res["microbench"] if r["bytes"] >= (2 << 20)]
        res["microbench_check"] = {
            "rule": "emulated / baseline <= 1.05 at >= 2 MiB (cemu_bench.cpp:281)",
            "max_ratio_ab": max(r["ratio_ab"] for r in big), "max_ratio_table": max(r["ratio_table"] for r in big),
            "max_abs_dev_table": round(max(abs(r["ratio_table"] - 1) for r in big), 4),
            "pass_ab": all(r["ratio_ab"] <= 1.05 for r in big), "pass_table": all(r["ratio_table"] <= 1.05 for r in big)}
    # --- e2e: the reference's spin-compute profiles -------------------------
    res["e2e"] = []
    for name, m, bb in e2e_models():
        spec = ModelSpec.load(m)
        row = {"model": name, "bucket_bytes": bb, "buckets": len(spec.buckets(bb))}
        barrier()
        base = spin_loop(spec, bb, NcclAllReduce(), e2e_iters, 3)
        barrier()
        if rank == 0:
            row["baseline_mean_us"] = float(np.mean(base))
            row["baseline_stddev_us"] = float(np.std(base, ddof=1))
            for tag, kw in (("ab", {"fit": fit}), ("table", {"plugin": plugin})):
                comm = emulated_comm(k, **kw)
                emu = spin_loop(spec, bb, comm, e2e_iters, 3)
                comm.close()
                row[f"emulated_{tag}_mean_us"] = float(np.mean(emu))
                row[f"rel_err_{tag}"] = float(abs(np.mean(emu) - np.mean(base)) / np.mean(base))
        barrier()
        res["e2e"].append(row)
    # --- e2e: a real bf16 MLP (tensor-core GEMMs beside the collectives) ----
    loaded = loaded_sweep(sizes, 20)
    reps_rows = [mlp_fidelity(k, rank, barrier, sizes, plugin, loaded, mlp_iters, footprint)
                 for _ in range(max(1, mlp_repeats))]
    row = reps_rows[0]
    modes = ("table", "table_footprint", "loaded_footprint", "in_situ_footprint")
    if rank == 0 and len(reps_rows) > 1:
        # repeats: the error of the pooled means, and every repeat's own
        bm = float(np.mean([r["baseline_mean_us"] for r in reps_rows]))
        row = {"model": row["model"], "repeats": len(reps_rows), "baseline_mean_us": bm,
               "footprint": row["footprint"],
               "baseline_noise_2sem_rel": float(np.mean([r["baseline_noise_2sem_rel"] for r in reps_rows])
                                                / np.sqrt(len(reps_rows))),
               "compute_only_mean_us": float(np.mean([r["compute_only_mean_us"] for r in reps_rows]))}
        for tag in modes:
            em = float(np.mean([r[f"emulated_{tag}_mean_us"] for r in reps_rows]))
            row[f"emulated_{tag}_mean_us"] = em
            row[f"rel_err_{tag}"] = float(abs(em - bm) / bm)
            row[f"rel_err_{tag}_per_repeat"] = [round(r[f"rel_err_{tag}"], 5) for r in reps_rows]
        row["per_repeat"] = reps_rows
    res["mlp"] = row
    if rank == 0:
        spin_errs = {t: max(r[f"rel_err_{t}"] for r in res["e2e"]) for t in ("ab", "table")}
        res["e2e_check"] = {"rule": "rel_err < 1% (north star; the reference gates at 5%, cemu_bench.cpp:372)",
                            "spin_models_max_rel_err_ab": spin_errs["ab"],
                            "spin_models_max_rel_err_table": spin_errs["table"],
                            "spin_models_pass_table": spin_errs["table"] < 0.01,
                            "mlp_rel_err": {t: row[f"rel_err_{t}"] for t in modes}}
    return res


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--segments", type=int, default=3)
    ap.add_argument("--e2e-iters", type=int, default=20)
    ap.add_argument("--mlp-iters", type=int, default=100)
    ap.add_argument("--mlp-repeats", type=int, default=3, help="repeats of the real-compute MLP check")
    ap.add_argument("--max-mib", type=int, default=256)
    ap.add_argument("--footprint-ctas", type=int, default=NCCL_FOOTPRINT[0], help="NCCL's channel count on this box")
    ap.add_argument("--footprint-smem", type=int, default=NCCL_FOOTPRINT[1], help="shared memory per NCCL CTA")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sizes = [s for s in SIZES if s <= (args.max_mib << 20)]
    res = run(sizes, args.reps, args.segments, args.e2e_iters, args.mlp_iters,
              (args.footprint_ctas, args.footprint_smem), args.mlp_repeats)
    if dist.get_rank() == 0:
        print("FIDELITY " + json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
