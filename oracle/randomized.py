"""CPU ORACLE: randomized two-phase rounding.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the CUDA path.

The paper's randomized rounding of S* draws Pr[S_int = 1] = S*  (§5.1:
"randomized rounding (Pr[x_int_i = 1] = x*_i)"; "a single relaxed solution can be used to
sample many integral solutions"; App. D).  The paper fixes no
random number generator, so DESIGN.md reading R1 fixes one, exactly reproducible on both sides:

  u(s, j, t, i) = Philox4x32-10(ctr, key)[(i - 1) mod 4] * 2^-32            (32-bit, in [0, 1))
      ctr = ((i - 1) div 4, t - 1, s mod 2^32, j),  key = (seed mod 2^32, seed div 2^32)
  S_{t,i} = 1[u(s, j, t, i) < S*_{t,i}]  for i < t        (exact compare of the real values)

for S* number s (global index) and sample j: one Philox block gives four consecutive nodes of
one row of one sample (round 2's reading; round 1 took the four samples of one element from a
block, which wasted three of its words below four samples).  The uniform is the whole 32-bit
word (round 2's second reading; the first used its top 24 bits, (w >> 8) 2^-24): u and the
fp32 S* are both exact in float64, so the compare below is the exact one.  S* = 0 never sets a bit, S* = 1 always does;
NaN compares false.  Phase 2 (R, FREE, U, cost) is unchanged (checkmate_oracle).

Philox4x32-10 is Salmon et al., "Parallel random numbers: as easy as 1, 2, 3" (SC'11):
ten rounds of  (c0, c1, c2, c3) -> (hi(M1 c2) ^ c1 ^ k0, lo(M1 c2), hi(M0 c0) ^ c3 ^ k1, lo(M0 c0))
with M0 = 0xD2511F53, M1 = 0xCD9E8D57 and the key bumped by (0x9E3779B9, 0xBB67AE85)
between rounds.  Pinned by the published known-answer vectors (tests/test_oracle_randomized.py).
"""
from __future__ import annotations

import numpy as np

from .checkmate_oracle import Instance, evaluate_S

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """One block: ctr = 4 x uint32, key = 2 x uint32 -> 4 x uint32 (plain Python ints)."""
    c0, c1, c2, c3 = (int(x) & MASK for x in ctr)
    k0, k1 = (int(x) & MASK for x in key)
    for r in range(10):
        if r:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & MASK, p1 & MASK, ((p0 >> 32) ^ c3 ^ k1) & MASK, p0 & MASK
    return c0, c1, c2, c3


def philox4x32_10_np(c0, c1, c2, c3, k0, k1):
    """The same block over numpy uint32 arrays (products in uint64), for whole matrices."""
    c0, c1, c2, c3 = (np.asarray(c, np.uint64) for c in (c0, c1, c2, c3))
    k0, k1 = np.uint64(k0), np.uint64(k1)
    m32 = np.uint64(MASK)
    for r in range(10):
        if r:
            k0 = (k0 + np.uint64(W0)) & m32
            k1 = (k1 + np.uint64(W1)) & m32
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        c0, c1, c2, c3 = ((p1 >> np.uint64(32)) ^ c1 ^ k0) & m32, p1 & m32, ((p0 >> np.uint64(32)) ^ c3 ^ k1) & m32, p0 & m32
    return [c.astype(np.uint32) for c in (c0, c1, c2, c3)]


def uniform32(word):
    """word * 2^-32 as float64: exact (a 32-bit integer times a power of two)."""
    return np.asarray(word, np.uint32).astype(np.float64) * 2.0 ** -32


def uniforms(n: int, s: int, j: int, seed: int) -> np.ndarray:
    """u(s, j, t, i) for t, i = 1..n as U[t-1][i-1] (float64); the whole matrix, i < t used."""
    t = np.repeat(np.arange(n, dtype=np.uint64), n)           # t - 1
    i = np.tile(np.arange(n, dtype=np.uint64), n)             # i - 1
    out = philox4x32_10_np(i // np.uint64(4), t, np.full(n * n, s & MASK, np.uint64),
                           np.full(n * n, j & MASK, np.uint64), seed & MASK, (seed >> 32) & MASK)
    word = np.choose((i % np.uint64(4)).astype(np.int64), out)  # output word (i - 1) mod 4
    return uniform32(word).reshape(n, n)


def round_S_randomized(inst: Instance, sstar, s: int, j: int, seed: int) -> np.ndarray:
    """A1 (randomized): S[t][i] = 1[u < S*_{t,i}] for i < t; same [n+2][n+1] layout as round_S."""
    n = inst.n
    U = uniforms(n, s, j, seed)
    S = np.zeros((n + 2, n + 1), dtype=bool)
    for t in range(1, n + 1):
        row = np.asarray(sstar[t - 1][: t - 1], dtype=np.float32).astype(np.float64)   # exact
        S[t, 1:t] = U[t - 1, : t - 1] < row      # NaN compares false
    return S


def evaluate_randomized(inst: Instance, sstar, s: int, j: int, seed: int, keep=False) -> dict:
    """One randomized candidate (S* number s, sample j): A1 randomized, then A2-A6."""
    return evaluate_S(inst, round_S_randomized(inst, sstar, s, j, seed), keep=keep)
