"""Helpers shared by the GPU tests: tensor <-> oracle numpy views."""
from __future__ import annotations

import numpy as np
import torch

from oracle import port as P

TORCH = {0: torch.int8, 1: torch.uint8, 2: torch.int32, 4: torch.int64, 6: torch.float16,
         7: torch.float32, 8: torch.float64, 9: torch.bfloat16}
FLOATS = (6, 7, 8, 9)


def host_input(dt: int, count: int, seed: int, scale: float = 3.0) -> torch.Tensor:
    g = torch.Generator().manual_seed(seed)
    if dt in FLOATS:
        return (torch.randn(count, generator=g, dtype=torch.float64) * scale).to(TORCH[dt])
    if dt == 4:
        return torch.randint(-2**62, 2**62, (count,), generator=g, dtype=torch.int64)
    lo, hi = {0: (-128, 128), 1: (0, 256), 2: (-2**31, 2**31)}[dt]
    return torch.randint(lo, hi, (count,), generator=g, dtype=torch.int64).to(TORCH[dt])


def to_np(t: torch.Tensor) -> np.ndarray:
    t = t.detach().cpu().contiguous()
    if t.dtype in (torch.bfloat16, torch.float16):
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a).view(np.uint8)


def assert_bit_equal(got: np.ndarray, want: np.ndarray, what: str = ""):
    g, w = bits(got), bits(want)
    if not np.array_equal(g, w):
        es = got.dtype.itemsize
        if g.size != w.size:
            raise AssertionError(f"{what}: size {got.size} != {want.size}")
        diff = np.nonzero((g.reshape(-1, es) != w.reshape(-1, es)).any(axis=1))[0]
        raise AssertionError(f"{what}: {len(diff)} of {len(got)} elements differ; first at {diff[:5]}: "
                             f"got {got[diff[:3]]} want {want[diff[:3]]}")


def config(W: int, real=(0,), mode: str = "hash", seed: int = 1, extra: str = "") -> str:
    return (f"world_size = {W}\nreal_ranks = {','.join(map(str, real))}\nbucket_bytes = 65536\n"
            f"payload.mode = {mode}\npayload.seed = {seed}\n" + extra)


def oracle_mode(mode: str) -> int:
    return P.PAYLOAD_ZERO if mode == "zero" else P.PAYLOAD_HASH
