"""torchrun worker (2 GPUs): the copy-engine allreduce (CEMU_CE, the default
for two real GPUs and >= 512 MiB) equals the fused kernel (CEMU_CE=0) bit
for bit on arbitrary floats, out of place and in place, for every dtype
the fused path folds; prints the per-call time of both.  Run by
tests/test_gpu_multigpu.py; `python -m torch.distributed.run
--nproc-per-node 2 tests/ce_check.py` by hand."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_02969_b200 as pb  # noqa: E402
import ctypes as C  # noqa: E402
from paper_2405_02969_b200._capi import lib  # noqa: E402

lib.cemuCommKernelLaunches.restype = C.c_uint64
lib.cemuCommKernelLaunches.argtypes = [C.c_void_p]


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(rank)
    cfg = (f"world_size = {8 * world}\nreal_ranks = {','.join(str(r) for r in range(world))}\n"
           "bucket_bytes = 1\n")
    out = {"k": world, "cases": []}
    for dtype, nbytes in ((torch.float32, 1 << 30), (torch.bfloat16, 768 << 20), (torch.int32, 512 << 20)):
        count = nbytes // torch.tensor([], dtype=dtype).element_size()
        g = torch.Generator(device="cuda").manual_seed(1234 + rank)
        if dtype.is_floating_point:
            src = torch.randn(count, device="cuda", generator=g).to(dtype)
        else:
            src = torch.randint(-2**31, 2**31 - 1, (count,), device="cuda", dtype=dtype, generator=g)
        res = {}
        for ce in ("1", "0"):
            os.environ["CEMU_CE"] = ce
            obj = [pb.get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            comm = pb.Communicator(cfg, rank, rank, obj[0])
            x, y = comm.alloc(count, dtype), comm.alloc(count, dtype)
            x.copy_(src)
            comm.all_reduce(x, y)  # out of place
            z = comm.alloc(count, dtype)
            z.copy_(src)
            comm.all_reduce(z, z)  # in place
            torch.cuda.synchronize()
            err = comm.async_error() if hasattr(comm, "async_error") else None
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            dist.barrier()
            l0 = lib.cemuCommKernelLaunches(comm._h)
            e0.record()
            for _ in range(10):
                comm.all_reduce(x, y)
            e1.record()
            torch.cuda.synchronize()
            res[ce] = {"out": y.view(torch.uint8).clone(), "inplace": z.view(torch.uint8).clone(),
                       "ms": e0.elapsed_time(e1) / 10, "err": err,
                       "launches": (lib.cemuCommKernelLaunches(comm._h) - l0) / 10}
            comm.close()
        same = bool(torch.equal(res["1"]["out"], res["0"]["out"]))
        same_ip = bool(torch.equal(res["1"]["inplace"], res["0"]["inplace"])) and \
            bool(torch.equal(res["1"]["inplace"], res["1"]["out"]))
        out["cases"].append({"rank": rank, "dtype": str(dtype), "bytes": nbytes, "equal": same,
                             "equal_in_place": same_ip, "ce_ms": round(res["1"]["ms"], 4),
                             "fused_ms": round(res["0"]["ms"], 4), "ce_launches": res["1"]["launches"],
                             "fused_launches": res["0"]["launches"], "errors": [res["1"]["err"], res["0"]["err"]]})
        del res
        torch.cuda.empty_cache()
    out["safety"] = safety(cfg, rank)
    print(json.dumps(out), flush=True)
    dist.destroy_process_group()
    ok = all(c["equal"] and c["equal_in_place"] for c in out["cases"]) and all(out["safety"].values())
    sys.exit(0 if ok else 1)


CANARY = 0xA5


def safety(cfg, rank):
    """Offsets, ragged counts, guard bands and disagreeing ranks on the
    copy-engine path (CEMU_CE=1) -- it only reads peer memory."""
    res = {}
    count, off = 128 << 20, 4  # 512 MiB fp32 at a 16-byte offset inside the region
    guard = 1024
    src = torch.randn(count + 3, device="cuda", generator=torch.Generator(device="cuda").manual_seed(99 + rank))
    outs = {}
    for ce in ("1", "0"):
        os.environ["CEMU_CE"] = ce
        obj = [pb.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = pb.Communicator(cfg, rank, rank, obj[0])
        for n in (count, count + 3):  # the ragged count takes the fused kernel on every rank alike
            xb, yb = comm.alloc(n + off + guard, torch.float32), comm.alloc(n + off + guard, torch.float32)
            for b in (xb, yb):
                b.view(torch.uint8).fill_(CANARY)
            x, y = xb[off:off + n], yb[off:off + n]
            x.copy_(src[:n])
            torch.cuda.synchronize()
            dist.barrier()
            l0 = lib.cemuCommKernelLaunches(comm._h)
            comm.all_reduce(x, y)
            torch.cuda.synchronize()
            launches = lib.cemuCommKernelLaunches(comm._h) - l0
            raw = yb.view(torch.uint8)
            guards_ok = bool((raw[:off * 4] == CANARY).all()) and bool((raw[(off + n) * 4:] == CANARY).all())
            outs[(ce, n)] = (y.view(torch.int32).clone(), launches, guards_ok, comm.async_error())
            comm.free(xb)
            comm.free(yb)
        comm.close()
    res["offset_ce_equals_fused"] = bool(torch.equal(outs[("1", count)][0], outs[("0", count)][0]))
    res["offset_ce_took_pipeline"] = outs[("1", count)][1] > 2
    res["ragged_took_fused_kernel"] = outs[("1", count + 3)][1] <= 2  # (+ a synthesis-cache fill)
    res["ragged_equals_fused"] = bool(torch.equal(outs[("1", count + 3)][0], outs[("0", count + 3)][0]))
    res["guards_intact"] = all(v[2] for v in outs.values())
    res["no_async_errors"] = all(v[3] is None for v in outs.values())
    # disagreeing ranks: rank 1 passes a different recv buffer than rank 0.
    # Both must report it, and neither may write the other's memory: rank
    # 1's buffer that rank 0 thinks is the recv stays untouched.
    for ce, n in (("1", count), ("0", 1 << 20)):
        os.environ["CEMU_CE"] = ce
        os.environ["CEMU_FUSED_TIMEOUT_S"] = "5"
        obj = [pb.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = pb.Communicator(cfg, rank, rank, obj[0])
        x, y, y2 = (comm.alloc(n, torch.float32) for _ in range(3))
        x.copy_(src[:n])
        y.view(torch.uint8).fill_(CANARY)
        y2.view(torch.uint8).fill_(CANARY)
        torch.cuda.synchronize()
        dist.barrier()
        comm.all_reduce(x, y if rank == 0 else y2)
        torch.cuda.synchronize()
        untouched = y2 if rank == 0 else y  # the buffer this rank did not pass
        res[f"disagree_ce{ce}_reported"] = comm.async_error() is not None
        res[f"disagree_ce{ce}_peer_memory_untouched"] = bool((untouched.view(torch.uint8) == CANARY).all())
        dist.barrier()
        comm.close()
    os.environ.pop("CEMU_FUSED_TIMEOUT_S", None)
    return res


if __name__ == "__main__":
    main()
