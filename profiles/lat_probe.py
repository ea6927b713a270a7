import sys, os, json
sys.path.insert(0, "/root/repo")
import torch, paper_2405_02969_b200 as pb
W = 64
comm = pb.Communicator(f"world_size = {W}\nreal_ranks = 0\nbucket_bytes = 1\n", 0, 0)
out = {}
for dn, dt in (("fp32", torch.float32), ("bf16", torch.bfloat16)):
    es = torch.empty(0, dtype=dt).element_size()
    for kb in (4, 16, 64, 128, 256, 512, 1024):
        n = kb * 1024 // es
        x = torch.randn(n, device="cuda").to(dt); y = torch.empty_like(x)
        s = torch.cuda.Stream()
        reps = 50
        with torch.cuda.stream(s):
            comm.all_reduce(x, y, stream=s); torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps): comm.all_reduce(x, y, stream=s)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        best = 1e9
        for r in range(5):
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1000 / reps)
        out[f"{dn}_{kb}KiB_us"] = round(best, 2)
print(os.environ.get("CEMU_SYNTH_SPLIT", "default"), json.dumps(out))
