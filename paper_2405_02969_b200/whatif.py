"""DDP what-if sweep on the B200 (BASELINE config 4).

The reference's `cemu-bench whatif` (proj/tools/cemu_bench.cpp:384-481)
re-expressed over the C-ABI: for each injected per-call delay d, run the
synthetic training loop (cemuRunTrainingLoop: spin-kernel compute, one
emulated allreduce per gradient bucket on an in-order comm stream), then fit
the latency-vs-iteration-time curve:

  knee      the largest per-bucket backward compute: below it an injected
            stall hides behind the backward pass (cemu_bench.cpp:391-403)
  tail      OLS slope above the knee -- every bucket's stall is exposed, so
            the slope approaches the bucket count (cemu_bench.cpp:424-435)
  marginal  OLS slope below the knee (< bucket count)

Each point also carries the ideal (predicted) iteration time of the same
loop -- compute exactly as specified, each collective taking exactly its
modelled latency -- and the what-if step-time error |measured - ideal| /
ideal, the north star's "< 1%" quantity.

    python -m paper_2405_02969_b200.whatif --model bert-like \
        --delays-us 0 500 1000 4000 6000 8000 10000
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os

import numpy as np

from ._capi import CemuError, lib

C_VOID = C.c_void_p
lib.cemuModelSpecParse.restype = C.c_int
lib.cemuModelSpecParse.argtypes = [C.c_char_p, C.POINTER(C_VOID), C.c_char_p, C.c_size_t]
lib.cemuModelSpecBuiltin.restype = C.c_int
lib.cemuModelSpecBuiltin.argtypes = [C.c_char_p, C.POINTER(C_VOID)]
lib.cemuModelSpecFree.restype = None
lib.cemuModelSpecFree.argtypes = [C_VOID]
lib.cemuModelSpecRender.restype = C.c_int
lib.cemuModelSpecRender.argtypes = [C_VOID, C.c_char_p, C.c_size_t]
lib.cemuModelSpecLayers.restype = C.c_uint32
lib.cemuModelSpecLayers.argtypes = [C_VOID, C_VOID, C_VOID, C_VOID, C.c_size_t, C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_uint32), C.POINTER(C.c_int64)]
lib.cemuBucketize.restype = C.c_uint32
lib.cemuBucketize.argtypes = [C_VOID, C.c_uint64, C_VOID, C_VOID, C_VOID, C.c_size_t]
lib.cemuRunTrainingLoop.restype = C.c_int
lib.cemuRunTrainingLoop.argtypes = [C_VOID, C_VOID, C.c_uint64, C_VOID, C_VOID, C_VOID, C_VOID, C.c_size_t]
lib.cemuPredictIterationUs.restype = C.c_double
lib.cemuPredictIterationUs.argtypes = [C_VOID, C.c_uint64, C_VOID, C.c_size_t]
lib.cemuCommModelLatencyUs.restype = C.c_int
lib.cemuCommModelLatencyUs.argtypes = [C_VOID, C.c_int, C.c_uint64, C.POINTER(C.c_int64)]
lib.cemuSpinUs.restype = C.c_int
lib.cemuSpinUs.argtypes = [C_VOID, C.c_uint64]
lib.cemuSpinChainUs.restype = C.c_int
lib.cemuSpinChainUs.argtypes = [C_VOID, C.c_uint64, C_VOID, C.c_int]
lib.cemuChainJoin.restype = C.c_int
lib.cemuChainJoin.argtypes = [C_VOID, C_VOID, C_VOID]
lib.cemuCommLastReleaseEnd.restype = C.c_int
lib.cemuCommLastReleaseEnd.argtypes = [C_VOID, C.POINTER(C_VOID)]


class ModelSpec:
    """A model profile in the reference's format (harness.cpp:27-114)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def parse(cls, text: str) -> "ModelSpec":
        h = C_VOID()
        err = C.create_string_buffer(1024)
        rc = lib.cemuModelSpecParse(text.encode(), C.byref(h), err, 1024)
        if rc:
            raise CemuError(rc, err.value.decode())
        return cls(h)

    @classmethod
    def load(cls, name_or_path: str) -> "ModelSpec":
        """Built-in profile name (bert-like, small, wide) or a file path
        (load_model_spec, harness.cpp:136-150)."""
        h = C_VOID()
        if lib.cemuModelSpecBuiltin(name_or_path.encode(), C.byref(h)) == 0:
            return cls(h)
        if not os.path.exists(name_or_path):
            raise CemuError(4, f"model '{name_or_path}' is neither a built-in profile nor a readable file")
        with open(name_or_path) as f:
            return cls.parse(f.read())

    def render(self) -> str:
        n = lib.cemuModelSpecRender(self._h, None, 0)
        buf = C.create_string_buffer(-n)
        lib.cemuModelSpecRender(self._h, buf, -n)
        return buf.value.decode()

    def layers(self):
        it, wu, up = C.c_uint32(), C.c_uint32(), C.c_int64()
        n = lib.cemuModelSpecLayers(self._h, None, None, None, 0, C.byref(it), C.byref(wu), C.byref(up))
        f, b, g = (np.zeros(n, np.int64), np.zeros(n, np.int64), np.zeros(n, np.uint64))
        lib.cemuModelSpecLayers(self._h, f.ctypes.data, b.ctypes.data, g.ctypes.data, n, None, None, None)
        return {"forward_us": f, "backward_us": b, "grad_bytes": g, "iterations": it.value,
                "warmup": wu.value, "update_us": up.value}

    def buckets(self, bucket_bytes: int):
        n = lib.cemuBucketize(self._h, bucket_bytes, None, None, None, 0)
        first, last, nb = np.zeros(n, np.uint32), np.zeros(n, np.uint32), np.zeros(n, np.uint64)
        lib.cemuBucketize(self._h, bucket_bytes, first.ctypes.data, last.ctypes.data, nb.ctypes.data, n)
        return [(int(a), int(b), int(c)) for a, b, c in zip(first, last, nb)]

    def __del__(self):
        if getattr(self, "_h", None):
            lib.cemuModelSpecFree(self._h)
            self._h = None


def run_loop(comm, spec: ModelSpec, bucket_bytes: int):
    """One cemuRunTrainingLoop: per-iteration device times (us) and traces."""
    info = spec.layers()
    iters = info["iterations"]
    nb = len(spec.buckets(bucket_bytes))
    start, end = np.zeros(iters), np.zeros(iters)
    issue, done = np.zeros(iters * max(nb, 1)), np.zeros(iters * max(nb, 1))
    rc = lib.cemuRunTrainingLoop(comm._h, spec._h, bucket_bytes, start.ctypes.data, end.ctypes.data,
                                 issue.ctypes.data, done.ctypes.data, iters)
    if rc:
        raise CemuError(rc, "cemuRunTrainingLoop failed")
    return {"iter_us": end - start, "start_us": start, "end_us": end,
            "issue_us": issue.reshape(iters, -1)[:, :nb], "complete_us": done.reshape(iters, -1)[:, :nb]}


TRACE_COLUMNS = ["iter", "start_us", "end_us", "bucket_id", "issue_us", "complete_us"]


def write_iteration_csv(path: str, trace: dict) -> None:
    """One row per (iteration, bucket) with the reference's columns
    (harness.cpp:256-271); times are device-event microseconds from the
    loop's first event, rounded to whole microseconds as the reference's
    integer clock is."""
    import csv
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(TRACE_COLUMNS)
        for it in range(len(trace["start_us"])):
            for b in range(trace["issue_us"].shape[1]):
                w.writerow([it, round(float(trace["start_us"][it])), round(float(trace["end_us"][it])), b,
                            round(float(trace["issue_us"][it, b])), round(float(trace["complete_us"][it, b]))])


def read_iteration_csv(path: str) -> dict:
    """read_iteration_csv (harness.cpp:273-303): the rows back, by iteration."""
    import csv
    rows = {}
    with open(path) as f:
        lines = [l for l in f if l.strip() and not l.startswith("#")]
    r = csv.reader(lines[1:])
    for cols in r:
        if len(cols) != 6:
            raise ValueError(f"bad trace csv row: {','.join(cols)}")
        it, s, e, b, iu, cu = (int(c) for c in cols)
        t = rows.setdefault(it, {"start_us": s, "end_us": e, "buckets": []})
        t["buckets"].append((b, iu, cu))
    return rows


def iteration_stats(trace: dict, warmup: int) -> dict:
    """iteration_stats (harness.cpp:305-319): count, mean and sample stddev
    of the iteration times after `warmup` iterations."""
    xs = np.asarray(trace["iter_us"])[warmup:]
    return {"count": int(len(xs)), "mean_us": float(np.mean(xs)) if len(xs) else 0.0,
            "stddev_us": float(np.std(xs, ddof=1)) if len(xs) > 1 else 0.0}


def predicted_us(comm, spec: ModelSpec, bucket_bytes: int) -> float:
    lats = []
    for _, _, nbytes in spec.buckets(bucket_bytes):
        v = C.c_int64()
        lib.cemuCommModelLatencyUs(comm._h, 0, nbytes, C.byref(v))
        lats.append(float(v.value))
    arr = np.asarray(lats, dtype=np.float64)
    return lib.cemuPredictIterationUs(spec._h, bucket_bytes, arr.ctypes.data, len(arr))


def knee_us(spec: ModelSpec, bucket_bytes: int) -> float:
    info = spec.layers()
    return float(max(sum(int(info["backward_us"][l]) for l in range(a, b + 1))
                     for a, b, _ in spec.buckets(bucket_bytes)))


def ols_slope(x, y):
    x, y = np.asarray(x, float), np.asarray(y, float)
    if len(x) < 2:
        return None
    return float(np.polyfit(x, y, 1)[0])


def sweep(model: str, delays_us, world: int = 2, bucket_bytes: int = 65536, device: int = 0,
          extra_config: str = "", iterations: int | None = None, reference_fn=None,
          trace_csv: str | None = None):
    """`reference_fn(model_text, world, bucket_bytes, inject_us) -> per-iteration
    times (us)` optionally times a comparison emulator on the same loop (the
    callers pass the reference CPU emulator; this package never imports it)."""
    import torch  # noqa: F401  (device memory/context only)

    from .comm import Communicator
    spec = ModelSpec.load(model)
    if iterations is not None:
        txt = spec.render().replace(f"iterations = {spec.layers()['iterations']}", f"iterations = {iterations}")
        wu = min(spec.layers()["warmup"], iterations // 4)
        txt = txt.replace(f"warmup = {spec.layers()['warmup']}", f"warmup = {wu}")
        spec = ModelSpec.parse(txt)
    info = spec.layers()
    nb = len(spec.buckets(bucket_bytes))
    knee = knee_us(spec, bucket_bytes)
    points = []
    for d in sorted(delays_us):
        cfg = (f"world_size = {world}\nreal_ranks = 0\nbucket_bytes = {bucket_bytes}\n"
               f"delay.inject_us = {float(d)!r}\n" + extra_config)
        comm = Communicator(cfg, 0, device)
        r = run_loop(comm, spec, bucket_bytes)
        if trace_csv:  # one file per injected delay: <stem>_inject<us>.csv
            stem, ext = os.path.splitext(trace_csv)
            write_iteration_csv(f"{stem}_inject{int(d)}{ext or '.csv'}", r)
        ideal = predicted_us(comm, spec, bucket_bytes)
        comm.close()
        xs = r["iter_us"][info["warmup"]:]
        pt = {"inject_us": float(d), "mean_us": float(np.mean(xs)), "stddev_us": float(np.std(xs, ddof=1)),
              "samples": int(len(xs)), "ideal_us": ideal,
              "rel_err": float(abs(np.mean(xs) - ideal) / ideal)}
        if reference_fn is not None:
            ref_iters = reference_fn(spec.render(), world, bucket_bytes, float(d))
            if ref_iters is not None:  # None: the comparison emulator gave no result for this point
                ri = np.asarray(ref_iters)[info["warmup"]:]
                pt["reference_mean_us"] = float(np.mean(ri))
                pt["reference_rel_err"] = float(abs(np.mean(ri) - ideal) / ideal)
        points.append(pt)
    tail = [(p["inject_us"], p["mean_us"]) for p in points if p["inject_us"] > knee]
    marg = [(p["inject_us"], p["mean_us"]) for p in points if p["inject_us"] < knee]
    res = {"model": model, "world": world, "bucket_bytes": bucket_bytes, "buckets": nb, "knee_us": knee,
           "tail_slope": ols_slope(*zip(*tail)) if len(tail) >= 2 else None,
           "marginal_slope": ols_slope(*zip(*marg)) if len(marg) >= 2 else None,
           "max_rel_err": max(p["rel_err"] for p in points), "points": points}
    if any("reference_rel_err" in p for p in points):
        res["reference_max_rel_err"] = max(p["reference_rel_err"] for p in points if "reference_rel_err" in p)
    ok = True
    if res["tail_slope"] is not None:
        ok &= 0.9 * nb <= res["tail_slope"] <= 1.1 * nb
    if res["marginal_slope"] is not None:
        ok &= res["marginal_slope"] < nb
    for a, b in zip(points, points[1:]):  # monotone within two stddevs
        ok &= b["mean_us"] + 2 * max(a["stddev_us"], b["stddev_us"]) >= a["mean_us"]
    res["checks_pass"] = bool(ok)
    return res


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--model", default="bert-like")
    ap.add_argument("--delays-us", type=float, nargs="+", default=[0, 500, 1000, 4000, 6000, 8000, 10000])
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--bucket-bytes", type=int, default=65536)
    ap.add_argument("--iterations", type=int, default=None)
    ap.add_argument("--trace-csv", default=None, help="per-(iteration, bucket) trace, reference columns")
    a = ap.parse_args()
    res = sweep(a.model, a.delays_us, a.world, a.bucket_bytes, iterations=a.iterations, trace_csv=a.trace_csv)
    for p in res["points"]:
        ref_txt = (f"   reference {p['reference_mean_us']:9.1f} us (err {100 * p['reference_rel_err']:.2f}%)"
                   if "reference_mean_us" in p else "")
        print(f"inject {p['inject_us']:8.0f} us -> iteration {p['mean_us']:9.1f} +- {p['stddev_us']:6.1f} us "
              f"(ideal {p['ideal_us']:9.1f}, err {100 * p['rel_err']:.3f}%){ref_txt}")
    print(f"buckets={res['buckets']} knee_us={res['knee_us']:.0f} tail_slope={res['tail_slope']} "
          f"marginal_slope={res['marginal_slope']} checks={'pass' if res['checks_pass'] else 'FAIL'}")
    print(json.dumps({k: v for k, v in res.items() if k != "points"}))


if __name__ == "__main__":
    main()
