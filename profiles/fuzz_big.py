import sys, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import torch
torch.cuda.set_device(0)
import test_gpu_fuzz as F
t0 = time.time(); n = 0
for block in range(16, 216):
    F.test_random_collectives_equal_the_oracle(None, block)
    n += 40
print(f"fuzz ok: {n} random collectives in {time.time() - t0:.0f} s")
