"""Long run of tests/test_gpu_fuzz.py's mid-size synthesis-cache fuzz:
random 64 KiB - 1 MiB allreduces / reduce-scatters at worlds 33-1025 (the
cache's lower bound, split-shape fills, every entry form), every result
against the oracle.
    python profiles/fuzz_mid_big.py [first_block] [end_block]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

torch.cuda.set_device(0)
import test_gpu_fuzz as F  # noqa: E402

t0 = time.time()
lo, hi = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (3, 53)
for block in range(lo, hi):
    F.test_random_mid_size_calls_through_the_synthesis_cache(None, block)
print(f"mid-size cache fuzz ok: {16 * (hi - lo)} random cached collectives (blocks {lo}..{hi - 1}) "
      f"in {time.time() - t0:.0f} s")
