"""Centred 16-bit synthesis-cache entries (kernels.hpp kCacheCentered16) at
257..8192 emulated ranks, and their escapes, against the oracle.

Run directly (one GPU) or under torch.distributed.run (k real GPUs, the fused
kernels' cached modes over symmetric buffers).  Arguments: world sizes.  With
CEMU_SYNTH_CACHE_C16_MAX raised to the world, a world of ~20,000 ranks makes
~1.5% of the entries escapes (t - offset outside [1, 65535]): the fold then
recomputes those sums from the keys.  Prints one JSON line per rank."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2405_02969_b200 as pb  # noqa: E402
from gpu_util import TORCH, assert_bit_equal, host_input, to_np  # noqa: E402
from oracle import port as P  # noqa: E402


def escapes(W: int, nreal: int, e0: int, count: int) -> int:
    """Entries of elements [e0, e0 + count) that are escapes: from the oracle's
    fp32 fold of a zero buffer, t = 128 * out + 128 n exactly."""
    n = W - nreal
    z = [np.zeros(e0 + count, np.float32) for _ in range(nreal)]
    out = P.allreduce(7, P.PAYLOAD_HASH, W, list(range(nreal)), 0, 1, z, e0 + count)[e0:]
    t = np.rint(out.astype(np.float64) * 128).astype(np.int64) + 128 * n
    u = t - (n * 255 // 2 - 32768)
    return int(((u < 1) | (u > 65535)).sum())


def main():
    worlds = [int(a) for a in sys.argv[1:]] or [300, 1024]
    k = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    uid = None
    if k > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    real = list(range(k))
    res = {"rank": local, "k": k, "cases": []}
    for W in worlds:
        if k > 1:
            obj = [pb.get_unique_id() if local == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        cfg = f"world_size = {W}\nreal_ranks = {','.join(map(str, real))}\nbucket_bytes = 1\n"
        comm = pb.Communicator(cfg, local, local, uid) if k > 1 else pb.Communicator(cfg, 0, 0)
        # >= 1 MiB per slice for every kind, or a "heavy" range (>= 2^27
        # peer-elements, >= 64 KiB) at very large worlds; ragged tail
        count = ((1 << 20) if W <= 8192 else (1 << 16)) * k + 7
        for dt in (7, 9, 6, 1, 0):
            for i in range(2):  # the first call of the comm fills, the rest hit
                sends = [host_input(dt, count, seed=1000 * W + 10 * dt + 100 * g + i) for g in range(k)]
                if k > 1:  # symmetric buffers: the fused kernel reads its slice's entries
                    x = comm.alloc(count, TORCH[dt])
                    y = comm.alloc(count, TORCH[dt])
                    x.copy_(sends[local].cuda())
                else:
                    x = sends[0].cuda()
                    y = torch.empty_like(x)
                comm.all_reduce(x, y)
                torch.cuda.synchronize()
                want = P.allreduce(dt, P.PAYLOAD_HASH, W, real, local, 1, [to_np(s) for s in sends], count)
                assert_bit_equal(to_np(y), want, f"W={W} dt={dt} call {i} rank {local}")
                if k > 1:
                    comm.free(x)
                    comm.free(y)
        st = comm.synth_cache_stats()
        assert st["hits"] >= 9 and st["fills"] >= 1, st
        if k == 1:  # one segment, 2 bytes per element (whole payload words)
            assert st["bytes"] == (count + 3) // 4 * 4 * 2, st
        err = comm.async_error()
        assert err is None, err
        comm.close()
        res["cases"].append({"world": W, "count": count, "stats": st,
                             "escapes": escapes(W, k, 0, count) if local == 0 else None})
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
