import sys, time, json
sys.path.insert(0, "/root/repo")
import torch, paper_2405_02969_b200 as pb
torch.cuda.set_device(0)
comm = pb.Communicator("world_size = 8\nreal_ranks = 0\nbucket_bytes = 1\n", 0, 0)
x = torch.zeros(1 << 20, device="cuda"); r = torch.empty(8 << 20, device="cuda"); s_ = torch.zeros(8 << 20, device="cuda")
o = torch.empty(1 << 20, device="cuda")
def free():
    torch.cuda.synchronize(); torch.cuda.empty_cache(); return torch.cuda.mem_get_info()[0]
pts = []
f0 = free()
for rnd in range(6):
    for i in range(20000):
        k = i % 3
        if k == 0: comm.all_reduce(x, x)
        elif k == 1: comm.all_gather(r[:1 << 20], r)
        else: comm.reduce_scatter(s_, o)
    pts.append(round((f0 - free()) / 2**20, 2))
print(json.dumps({"calls_per_point": 20000, "used_MiB_after_each_20k_calls": pts}))
