import sys, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import torch
torch.cuda.set_device(0)
import test_gpu_fuzz as F
t0 = time.time(); n = 0
lo, hi = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (16, 216)
for block in range(lo, hi):
    F.test_random_collectives_equal_the_oracle(None, block)
    n += 40
print(f"fuzz ok: {n} random collectives (blocks {lo}..{hi - 1}) in {time.time() - t0:.0f} s")
