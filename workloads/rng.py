"""Counter-based splitmix64 hashing shared by the host generators and the device
generator kernel (workloads/csrc/gen_sstar.cu implements the same function bit
for bit).  Input generation only -- none of the method's arithmetic.

    fmix(z)            = splitmix64 output function of (z + golden)
    mix64(seed, stream, a, b) = fmix(fmix(fmix(seed ^ (stream << 48)) ^ a) ^ b)
    u24(x)             = top 24 bits of x   (uniform integer in [0, 2^24))
"""
from __future__ import annotations

import numpy as np

MASK = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB


def fmix(z: int) -> int:
    z = (z + GOLDEN) & MASK
    z = ((z ^ (z >> 30)) * C1) & MASK
    z = ((z ^ (z >> 27)) * C2) & MASK
    return z ^ (z >> 31)


def mix64(seed: int, stream: int, a: int, b: int) -> int:
    return fmix(fmix(fmix((seed ^ (stream << 48)) & MASK) ^ (a & MASK)) ^ (b & MASK))


def u24(x: int) -> int:
    return x >> 40


# ---- vectorised numpy versions (uint64 arithmetic wraps mod 2^64) ----
_G = np.uint64(GOLDEN)
_C1 = np.uint64(C1)
_C2 = np.uint64(C2)


def fmix_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z.astype(np.uint64) + _G
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def mix64_np(seed: int, stream: int, a, b) -> np.ndarray:
    h0 = np.uint64(fmix((seed ^ (stream << 48)) & MASK))
    a = np.asarray(a).astype(np.uint64)
    b = np.asarray(b).astype(np.uint64)
    return fmix_np(fmix_np(h0 ^ a) ^ b)


def u24_np(x: np.ndarray) -> np.ndarray:
    return (x >> np.uint64(40)).astype(np.int64)
