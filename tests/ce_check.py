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
    print(json.dumps(out), flush=True)
    dist.destroy_process_group()
    ok = all(c["equal"] and c["equal_in_place"] for c in out["cases"])
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
