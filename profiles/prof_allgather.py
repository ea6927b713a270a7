"""ncu target: emulated allgather, world 64 (63 emulated blocks), 1 GiB recv,
fp32, in place -- the config-2 shape's synth_fill_vec launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2405_02969_b200 as pb  # noqa: E402
W = 64
comm = pb.Communicator(f"world_size = {W}\nreal_ranks = 0\nbucket_bytes = 1\n", 0, 0)
sc = (1 << 30) // 4 // W
recv = torch.zeros(sc * W, device="cuda")
for _ in range(3):
    comm.all_gather(recv[:sc], recv)
torch.cuda.synchronize()
print("ok")
