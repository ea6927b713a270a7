import os, sys, json, subprocess
sys.path.insert(0, "/root/repo")
import torch
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2405_02969_b200 as pb
    comm = pb.Communicator("world_size = 8\nreal_ranks = 0\nbucket_bytes = 1\n", 0, 0)
    n = 1 << 28
    hi = torch.randn(n).pin_memory(); ho = torch.empty(n).pin_memory()
    for _ in range(2): comm.all_reduce_host(hi, ho)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5): comm.all_reduce_host(hi, ho)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"chunk": os.environ.get("CEMU_HOST_CHUNK_MIB"), "ms": e0.elapsed_time(e1) / 5}))
    sys.exit(0)
n = 1 << 28
hi = torch.randn(n).pin_memory(); ho = torch.empty(n).pin_memory()
d1 = torch.empty(n, device="cuda"); d2 = torch.randn(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): f()
    torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
h2d = t(lambda: d1.copy_(hi, non_blocking=True))
d2h = t(lambda: ho.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
bi = t(both)
print(json.dumps({"h2d_GBps": round(1.073741824 / h2d * 1e3, 1), "d2h_GBps": round(1.073741824 / d2h * 1e3, 1),
                  "bidir_ms": round(bi, 3), "bidir_each_GBps": round(1.073741824 / bi * 1e3, 1)}))
for c in (4, 8, 16, 32, 64):
    r = subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, CEMU_HOST_CHUNK_MIB=str(c)),
                       capture_output=True, text=True)
    print(r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-400:])
