import sys, os, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, os.environ.get("PKGROOT", "/root/repo"))
import torch, paper_2405_02969_b200 as pb
out = {}
for W in (8, 64, 1024):
    comm = pb.Communicator(f"world_size = {W}\nreal_ranks = 0\nbucket_bytes = 1\n", 0, 0)
    for dn, dt in (("fp32", torch.float32), ("bf16", torch.bfloat16), ("u8", torch.uint8), ("i32", torch.int32)):
        tot = (1 << 30) // torch.empty(0, dtype=dt).element_size()
        sc = tot // W
        recv = torch.empty(sc * W, dtype=dt, device="cuda")
        own = recv[:sc]
        for _ in range(3): comm.all_gather(own, recv)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        best = 1e9
        for r in range(5):
            e0.record()
            for _ in range(4): comm.all_gather(own, recv)
            e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 4)
        out[f"W{W}_{dn}_ag1GiB_ms"] = round(best, 4)
    comm.close()
print(os.environ.get("CEMU_FILL_GRID", "default"), json.dumps(out))
