"""One rank of the multi-GPU parity check (launched by test_gpu_multigpu.py
under torch.distributed.run).  Real ranks 0..N-1 of a world of 8N (or a
non-contiguous real set), NCCL inside libcemu_b200 for the real part."""
from __future__ import annotations

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2405_02969_b200 as pb  # noqa: E402
from gpu_util import TORCH, assert_bit_equal, to_np  # noqa: E402
from oracle import port as P  # noqa: E402


def trace(msg):
    if os.environ.get("MGPU_TRACE"):
        print(f"[{os.environ['LOCAL_RANK']}] {msg}", file=sys.stderr, flush=True)


def main():
    import threading
    # a rank that fails leaves its peers inside collectives: bound the run
    limit = float(os.environ.get("MGPU_WATCHDOG_S", "240"))
    threading.Timer(limit, lambda: (print(f"watchdog: {limit}s", file=sys.stderr, flush=True), os._exit(3))).start()
    try:
        run()
    except BaseException as e:  # noqa: BLE001
        print(f"[{os.environ.get('LOCAL_RANK')}] FAILED: {e!r}", file=sys.stderr, flush=True)
        os._exit(1)
    sys.stdout.flush()
    os._exit(0)


CANARY = 0xA5


def check_guards(base, off, count, what):
    """Every byte of `base` outside elements [off, off + count) still holds the canary."""
    torch.cuda.synchronize()
    es = base.element_size()
    raw = base.view(torch.uint8).cpu()
    bad = int((raw[:off * es] != CANARY).sum()) + int((raw[(off + count) * es:] != CANARY).sum())
    assert bad == 0, f"{what}: {bad} guard bytes overwritten"


def run():
    os.environ["CEMU_HOST_CHUNK_MIB"] = "1"  # host-buffer pipeline: many chunks per call
    local = int(os.environ["LOCAL_RANK"])
    n = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    layouts = [list(range(n)), [2 * i + 1 for i in range(n)]]  # contiguous, strided
    for real in layouts:
        W = 8 * n
        me = real[local]
        obj = [pb.get_unique_id() if local == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        cfg = f"world_size = {W}\nreal_ranks = {','.join(map(str, real))}\nbucket_bytes = 1\n"
        comm = pb.Communicator(cfg, me, local, obj[0])
        for dt in (7, 9, 2, 4, 8):
            for count in (1, n * 1000 + 3, (1 << 20) + 7):
                trace(f"real={real} dt={dt} count={count}")
                sends = []
                for i in range(n):
                    g = np.random.default_rng(1000 * i + count)
                    if dt in (7, 9, 8):  # dyadic, <= 5 significant bits: the real sum of <= 8
                        # values is exact even in bf16, so NCCL's fold order cannot matter
                        v = torch.from_numpy((g.integers(-16, 16, size=count) / 8).astype(np.float32)).to(TORCH[dt])
                    elif dt == 4:
                        v = torch.from_numpy(g.integers(-2**62, 2**62, size=count).astype(np.int64))
                    else:
                        v = torch.from_numpy(g.integers(-2**31, 2**31, size=count).astype(np.int32))
                    sends.append(v)
                x = sends[local].cuda()
                y = torch.empty_like(x)
                comm.all_reduce(x, y)
                torch.cuda.synchronize()
                want = P.allreduce(dt, P.PAYLOAD_HASH, W, real, me, 1, [to_np(s) for s in sends], count)
                assert_bit_equal(to_np(y), want, f"allreduce real={real} dt={dt} n={count}")
                trace('allgather')
                # allgather
                blk = max(count // 8, 1)
                recv = torch.empty(blk * W, dtype=x.dtype, device="cuda")
                comm.all_gather(x[:blk].contiguous(), recv)
                torch.cuda.synchronize()
                want = P.allgather(dt, P.PAYLOAD_HASH, W, real, me, 1, [to_np(s[:blk]) for s in sends], blk)
                assert_bit_equal(to_np(recv), want, f"allgather real={real} dt={dt}")
                trace('reduce-scatter over a buffer of W chunks')
                # reduce-scatter over a buffer of W chunks
                rc = max(count // 16, 1)
                full = [torch.cat([s] * -(-rc * W // count))[: rc * W] for s in sends]
                out = torch.empty(rc, dtype=x.dtype, device="cuda")
                comm.reduce_scatter(full[local].cuda(), out)
                torch.cuda.synchronize()
                want = P.reducescatter(dt, P.PAYLOAD_HASH, W, real, me, 1, [to_np(f) for f in full], rc)
                assert_bit_equal(to_np(out), want, f"reducescatter real={real} dt={dt}")
                trace('broadcast from a real and from an emulated root')
                # broadcast from a real and from an emulated root
                for root in (real[-1], (real[-1] + 1) % W):
                    b = torch.empty_like(x)
                    src = x if me == root else None
                    comm.broadcast(src if src is not None else torch.empty_like(x), b, root)
                    torch.cuda.synchronize()
                    rs = to_np(sends[real.index(root)]) if root in real else None
                    want = P.broadcast(dt, P.PAYLOAD_HASH, W, real, me, root, 1, rs, count)
                    assert_bit_equal(to_np(b), want, f"broadcast root={root} dt={dt}")
        # NCCL path (plain buffers) with arbitrary floats: the real part is
        # summed in NCCL's order, so the result is held to the north star's
        # tolerances (fp32 1e-6, bf16 1e-2), relative to the inputs' magnitude
        for dt, rtol in ((7, 1e-6), (9, 1e-2)):
            count = 3 * 4096 + 7
            sends = [torch.from_numpy(np.random.default_rng(900 + i).standard_normal(count).astype(np.float32) * 3)
                     .to(TORCH[dt]) for i in range(n)]
            y = torch.empty(count, dtype=TORCH[dt], device="cuda")
            comm.all_reduce(sends[local].cuda(), y)
            torch.cuda.synchronize()
            want = P.allreduce(dt, P.PAYLOAD_HASH, W, real, me, 1, [to_np(s) for s in sends], count)
            w = torch.from_numpy(want.view(np.int16) if dt == 9 else want).view(TORCH[dt]).double().numpy()
            g = y.double().cpu().numpy()
            scale = sum(np.abs(s.double().numpy()) for s in sends) + np.abs(w) + 1.0
            assert np.max(np.abs(g - w) / scale) <= rtol, (dt, float(np.max(np.abs(g - w) / scale)))
        # host-buffer allreduce: chunks pipelined through symmetric pipe buffers,
        # one fused kernel per chunk (1 MiB chunks: the buffers rotate)
        for dt in (7, 9, 2):
            for count in (5, (5 << 20) // 2 + 7):
                sends = []
                for i in range(n):
                    gi = np.random.default_rng(300 * i + count + dt)
                    if dt in (7, 9):
                        v = torch.from_numpy(gi.standard_normal(count).astype(np.float32)).to(TORCH[dt])
                    else:
                        v = torch.from_numpy(gi.integers(-2**31, 2**31, size=count).astype(np.int64)).to(TORCH[dt])
                    sends.append(v)
                trace(f"host pipeline real={real} dt={dt} count={count}")
                hin = sends[local].pin_memory()
                hout = torch.empty_like(hin).pin_memory()
                comm.all_reduce_host(hin, hout)
                torch.cuda.synchronize()
                assert comm.async_error() is None
                want = P.allreduce(dt, P.PAYLOAD_HASH, W, real, me, 1, [to_np(s) for s in sends], count)
                assert_bit_equal(to_np(hout), want, f"host allreduce real={real} dt={dt} n={count}")
        # fused path: symmetric buffers -> one kernel over NVLink peer memory,
        # arbitrary (non-dyadic) floats: the real fold order is the oracle's
        for dt in (7, 9, 6, 2, 1):
            for count in (1, 5, 4096 * n + 13, (1 << 22) + 3):
                g = np.random.default_rng(7 + count)
                sends = []
                for i in range(n):
                    gi = np.random.default_rng(100 * i + count)
                    if dt in (7, 9, 6):
                        v = torch.from_numpy(gi.standard_normal(count).astype(np.float32)).to(TORCH[dt])
                    else:
                        v = torch.from_numpy(gi.integers(-2**31, 2**31, size=count).astype(np.int64)).to(TORCH[dt])
                    sends.append(v)
                off = int(g.integers(0, 64)) * 16 // torch.empty(0, dtype=TORCH[dt]).element_size()
                trace(f"fused real={real} dt={dt} count={count}")
                # guard band of canary bytes after each buffer (and the
                # offset's bytes before it): the fused kernel's peer pushes
                # must land inside every GPU's [off, off + count)
                guard = 4096 // torch.empty(0, dtype=TORCH[dt]).element_size()
                xb = comm.alloc(count + off + guard, TORCH[dt])
                yb = comm.alloc(count + off + guard, TORCH[dt])
                for b in (xb, yb):
                    b.view(torch.uint8).fill_(CANARY)
                x, y = xb[off:off + count], yb[off:off + count]
                x.copy_(sends[local].cuda())
                torch.cuda.synchronize()
                before, fills = comm.kernel_launches, comm.synth_cache_stats()["fills"]
                comm.all_reduce(x, y)
                torch.cuda.synchronize()
                trace("fused call done")
                # one fused kernel (plus the synthesis-cache fill when this
                # call wrote the cache's entries for its slice)
                filled = comm.synth_cache_stats()["fills"] - fills
                assert comm.kernel_launches - before == 1 + filled, "fused path not taken"
                assert comm.async_error() is None
                want = P.allreduce(dt, P.PAYLOAD_HASH, W, real, me, 1, [to_np(s) for s in sends], count)
                assert_bit_equal(to_np(y), want, f"fused allreduce real={real} dt={dt} n={count}")
                assert_bit_equal(to_np(x), to_np(sends[local]), f"fused input modified real={real} dt={dt}")
                check_guards(xb, off, count, f"fused send real={real} dt={dt} n={count}")
                check_guards(yb, off, count, f"fused recv real={real} dt={dt} n={count}")
                comm.all_reduce(x, x)  # in place
                torch.cuda.synchronize()
                assert_bit_equal(to_np(x), want, f"fused in-place real={real} dt={dt} n={count}")
                check_guards(xb, off, count, f"fused in-place real={real} dt={dt} n={count}")
                comm.free(xb)
                comm.free(yb)
                # fused reduce-scatter (symmetric send) and allgather (symmetric recv)
                rc = max(count // 3, 8) // 8 * 8  # 16-byte chunks: the fused path (checked below)
                full = [torch.cat([v] * -(-rc * W // count))[: rc * W] for v in sends]
                xs = comm.alloc(rc * W, TORCH[dt])
                xs.copy_(full[local].cuda())
                # rank-local misalignment of the output must not change the path
                out = torch.empty(rc + 1, dtype=TORCH[dt], device="cuda")[local % 2:][:rc]
                torch.cuda.synchronize()
                before, fills = comm.kernel_launches, comm.synth_cache_stats()["fills"]
                comm.reduce_scatter(xs, out)
                torch.cuda.synchronize()
                filled = comm.synth_cache_stats()["fills"] - fills
                assert comm.kernel_launches - before == 1 + filled and comm.async_error() is None
                want = P.reducescatter(dt, P.PAYLOAD_HASH, W, real, me, 1, [to_np(f) for f in full], rc)
                assert_bit_equal(to_np(out), want, f"fused reducescatter real={real} dt={dt} rc={rc}")
                blk = rc
                ag = comm.alloc(blk * W, TORCH[dt])
                mine = torch.cat([full[local][:1], full[local][:blk]]).cuda()[1:] if local % 2 else \
                    full[local][:blk].cuda()
                torch.cuda.synchronize()
                before = comm.kernel_launches
                comm.all_gather(mine, ag)
                torch.cuda.synchronize()
                assert comm.kernel_launches - before == 1 and comm.async_error() is None
                want = P.allgather(dt, P.PAYLOAD_HASH, W, real, me, 1, [to_np(f[:blk]) for f in full], blk)
                assert_bit_equal(to_np(ag), want, f"fused allgather real={real} dt={dt} blk={blk}")
                comm.free(xs)
                comm.free(ag)
        # fused calls captured in a CUDA graph and replayed: the barrier epoch
        # lives in device memory, so every replay synchronises afresh
        xg, yg = comm.alloc(1 << 16, torch.float32), comm.alloc(1 << 16, torch.float32)
        src = torch.from_numpy(np.random.default_rng(local).standard_normal(1 << 16).astype(np.float32)).cuda()
        xg.copy_(src)
        comm.all_reduce(xg, yg)
        torch.cuda.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph):
            for _ in range(3):
                comm.all_reduce(xg, yg)
        allsrc = [torch.from_numpy(np.random.default_rng(i).standard_normal(1 << 16).astype(np.float32)) for i in range(n)]
        want = P.allreduce(7, P.PAYLOAD_HASH, W, real, me, 1, [to_np(v) for v in allsrc], 1 << 16)
        for _ in range(4):
            yg.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            gph.replay()
            torch.cuda.synchronize()
            assert comm.async_error() is None
            assert_bit_equal(to_np(yg), want, f"fused graph replay real={real}")
        comm.free(xg)
        comm.free(yg)
        if real == layouts[-1]:
            # ranks that disagree on a fused call fail loudly (error 3), not silently
            x, y = comm.alloc(4096, torch.float32), comm.alloc(4096, torch.float32)
            cnt = 1024 + 16 * local
            comm.all_reduce(x[:cnt], y[:cnt])
            torch.cuda.synchronize()
            err = comm.async_error()
            assert err is not None and "disagree" in err, err
        comm.close()
        dist.barrier()
    run_c3(n, local)
    if local == 0:
        print("MGPU OK", n)
    dist.destroy_process_group()


def run_c3(n, local):
    """BASELINE config 3: bf16 in a 128-rank world of 16 nodes x 8 GPUs whose
    real ranks are this node's GPUs 0..n-1; hierarchical alpha-beta delay on.
    The fused path (symmetric buffers, arbitrary floats) and the NCCL path
    (plain buffers, dyadic values) equal the oracle bit for bit, and every
    rank's injected delay is within max(1%, 2 us) of the model."""
    from paper_2405_02969_b200 import c3
    W, real = c3.WORLD, list(range(n))
    obj = [pb.get_unique_id() if local == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = pb.Communicator(c3.config(n, True), local, local, obj[0])
    for count in (4097, (1 << 21) + 3):
        trace(f"C3 count={count}")
        rngs = [np.random.default_rng(5000 + 17 * i + count) for i in range(n)]
        sends = [torch.from_numpy(g.standard_normal(count).astype(np.float32)).to(torch.bfloat16) for g in rngs]
        want = P.allreduce(9, P.PAYLOAD_HASH, W, real, local, 1, [to_np(s) for s in sends], count)
        x, y = comm.alloc(count, torch.bfloat16), comm.alloc(count, torch.bfloat16)
        x.copy_(sends[local].cuda())
        torch.cuda.synchronize()
        dist.barrier()
        before = comm.kernel_launches
        comm.all_reduce(x, y)
        torch.cuda.synchronize()
        assert comm.async_error() is None
        rec = comm.call_record()
        assert comm.kernel_launches > before
        assert_bit_equal(to_np(y), want, f"C3 fused bf16 n={count}")
        # delay: a real collective also waits for its slowest real peer, so a
        # call that starts skewed against the others (barrier release, first
        # use of fresh buffers) measures skew + delay; the best of three warm
        # calls isolates the injection (asserted per call on one GPU in
        # test_gpu_delay.py)
        errs = []
        for _ in range(3):
            dist.barrier()
            comm.all_reduce(x, y)
            torch.cuda.synchronize()
            rec = comm.call_record()
            model = rec["model_latency_us"]
            errs.append(abs((rec["t_end_ns"] - rec["t_start_ns"]) / 1e3 - model))
        assert model > 0 and min(errs) <= max(0.01 * model, 2.0), (count, errs, model)
        comm.free(x)
        comm.free(y)
        dy = [torch.from_numpy((g.integers(-16, 16, size=count) / 8).astype(np.float32)).to(torch.bfloat16)
              for g in rngs]
        want = P.allreduce(9, P.PAYLOAD_HASH, W, real, local, 1, [to_np(s) for s in dy], count)
        yp = torch.empty(count, dtype=torch.bfloat16, device="cuda")
        dist.barrier()
        comm.all_reduce(dy[local].cuda(), yp)
        torch.cuda.synchronize()
        assert_bit_equal(to_np(yp), want, f"C3 NCCL-path bf16 n={count}")
    comm.close()
    dist.barrier()


if __name__ == "__main__":
    main()
