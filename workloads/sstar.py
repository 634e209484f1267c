"""Seeded fractional checkpoint matrices S* (the hot path's input).

Input generation only -- none of the method's arithmetic.  S* is the LP's
fractional storage matrix; the LP solve itself is out of
scope, so S* is synthesised with the structure an LP solution has.

Row r (0-based stage t = r+1) holds S*_{t, i} for nodes i < r (0-based), the
strict lower triangle (Eq. 12b).  Entries with i >= r are never
read by the method; generators fill them with ``upper`` (default 0.0; tests use
NaN / 1.0 to prove they are never read).

Families (fp32):
  G0  binary:   an exact 0/1 pattern given by the caller.
  G1  LP-like:  a Chen-segmented anchor S0 generalised to DAGs, then jittered:
                S* = 1 - g where S0 = 1, g where S0 = 0, with g = |d| * SIGMA_SCALE,
                d = (sum of four 16-bit uniforms) - 2*65535 (Irwin-Hall(4), an exactly
                reproducible stand-in for |N(0, 0.15)|); a fraction PHI of strict-lower
                entries is redrawn U(0,1) and a fraction PSI set to exactly 0.5.
  G2  uniform:  i.i.d. U(0,1) (24-bit), adversarial for R.
  mix           per-S* choice between G1 and G2.

All values are exact in fp32 and computed with one IEEE-rounded fp32 multiply and
one fp32 subtract, so the device generator reproduces them bit for bit.

Layouts:
  dense   [n][ld] row-major, ld >= n, ld % 4 == 0
  tri4    packed lower triangle: row r starts at float offset tri4_offset(r) =
          sum_{r' < r} roundup4(r'); rows are 16-byte aligned.
"""
from __future__ import annotations

import numpy as np

from .rng import fmix, mix64, mix64_np, u24_np

SIGMA = 0.15
# Irwin-Hall(4) of 16-bit uniforms: std = sqrt(4/12) * 65536
SIGMA_SCALE = np.float32(SIGMA / (np.sqrt(4.0 / 12.0) * 65536.0))
PHI24 = 16777          # round(1e-3 * 2^24): redraw U(0,1)
PSI24 = 16777          # round(1e-3 * 2^24): set to exactly 0.5
RHO24 = (1677722, 5033165, 10066330)   # round(rho * 2^24), rho in {0.1, 0.3, 0.6}
INV24 = np.float32(1.0 / (1 << 24))

STREAM_G2 = 1
STREAM_RHO = 2
STREAM_K = 3
STREAM_JIT = 4
STREAM_REDRAW = 5
STREAM_REDRAW_U = 6
STREAM_FAMILY = 7

FAMILY_IDS = {"g1": 1, "g2": 2, "mix": 3}


def roundup4(x):
    return (x + 3) // 4 * 4


def tri4_offset(r: int) -> int:
    """Float offset of row r in the tri4 layout: sum_{r'<r} roundup4(r').

    Rows 4a..4a+3 have padded lengths 4a, 4a+4, 4a+4, 4a+4 (sum 16a+12)."""
    q, m = divmod(r, 4)
    full = 8 * q * (q - 1) + 12 * q
    rest = (4 * q if m > 0 else 0) + max(m - 1, 0) * (4 * q + 4)
    return full + rest


def tri4_size(n: int) -> int:
    return tri4_offset(n)


def _keys(r, i):
    return (np.asarray(r, np.uint64) << np.uint64(32)) | np.asarray(i, np.uint64)


def g2_row(seed: int, s: int, r: int) -> np.ndarray:
    """Strict-lower part (length r) of row r of S* #s, family G2."""
    i = np.arange(r)
    x = mix64_np(seed, STREAM_G2, np.uint64(s), _keys(r, i))
    return (u24_np(x).astype(np.float32) * INV24).astype(np.float32)


def segment_tops(L: int, K: np.ndarray) -> np.ndarray:
    """tau(i): top (largest index) of the maximal run of non-K forward nodes containing i."""
    tau = np.full(L, -1, np.int64)
    top = -1
    for v in range(L - 1, -1, -1):
        if K[v]:
            top = -1
        else:
            if top < 0:
                top = v
            tau[v] = top
    return tau


def g1_params(seed: int, s: int, L: int):
    rho24 = RHO24[fmix(mix64(seed, STREAM_RHO, s, 0)) % 3]
    x = mix64_np(seed, STREAM_K, np.uint64(s), np.arange(L, dtype=np.uint64))
    K = u24_np(x) < rho24
    return K, segment_tops(L, K)


def g1_anchor_row(r: int, L: int, K, tau, last, lastF) -> np.ndarray:
    """Binary anchor S0 for row r (0-based), nodes i < r."""
    i = np.arange(r)
    a = np.zeros(r, bool)
    if r == 0:
        return a
    lst = last[:r]
    bwd = i >= L                         # loss and backward nodes: liveness
    a |= bwd & (r <= lst)
    fw = ~bwd
    Kf = np.zeros(r, bool)
    Kf[fw] = K[i[fw]]
    a |= fw & Kf & (r <= lst)
    nk = fw & ~Kf
    tau_i = np.zeros(r, np.int64)
    tau_i[fw] = tau[i[fw]]
    a |= nk & ((r <= lastF[:r]) | ((2 * L - tau_i < r) & (r <= lst)))
    return a


def g1_row(seed: int, s: int, r: int, L: int, K, tau, last, lastF) -> np.ndarray:
    a = g1_anchor_row(r, L, K, tau, last, lastF)
    i = np.arange(r)
    keys = _keys(r, i)
    x = mix64_np(seed, STREAM_JIT, np.uint64(s), keys)
    d = np.zeros(r, np.int64)
    for f in range(4):
        d += ((x >> np.uint64(16 * f)) & np.uint64(0xFFFF)).astype(np.int64)
    d = np.abs(d - 2 * 65535)
    g = (d.astype(np.float32) * SIGMA_SCALE).astype(np.float32)
    v = np.where(a, np.float32(1.0) - g, g).astype(np.float32)
    q = u24_np(mix64_np(seed, STREAM_REDRAW, np.uint64(s), keys))
    u = (u24_np(mix64_np(seed, STREAM_REDRAW_U, np.uint64(s), keys)).astype(np.float32) * INV24)
    v = np.where(q < PHI24, u.astype(np.float32), v)
    v = np.where((q >= PHI24) & (q < PHI24 + PSI24), np.float32(0.5), v)
    return v.astype(np.float32)


def family_of(family: str, seed: int, s: int) -> str:
    if family == "mix":
        return "g2" if (fmix(mix64(seed, STREAM_FAMILY, s, 0)) & 1) else "g1"
    return family


def blk_rows(n: int, g: int) -> int:
    return min(32, n - 1 - 32 * g)


def blk_diag_chunks(h: int) -> int:
    return sum(max(0, h - 4 * k) for k in range(8))


def blk_block_off(g: int, w: int, h: int) -> int:
    """Float offset of block (g, w) in a CM_LAYOUT_BLK S* (every group before g is full)."""
    return 4 * (128 * g * (g - 1) + 144 * g) + 32 * h * w


def blk_size(n: int) -> int:
    """Floats per S* in CM_LAYOUT_BLK (include/cm.h)."""
    if n < 2:
        return 0
    gr = (n - 2) // 32 + 1
    h = blk_rows(n, gr - 1)
    return blk_block_off(gr - 1, gr - 1, h) + 4 * blk_diag_chunks(h)


def blk_positions(n: int):
    """(rows, cols, positions): the float position of every strict-lower entry (r, i) in the
    blocked layout: row group g = (r-1) div 32, row l = (r-1) mod 32 of it, block w = i div 32;
    every block chunk-major (16-byte chunk c = nodes 32w+4c .. +3): off-diagonal chunk c of
    row l at chunk h c + l, diagonal chunk c of rows l = 4c .. h-1 at chunk B_c + l - 4c."""
    r, i = np.tril_indices(n, -1)
    g, l = (r - 1) // 32, (r - 1) % 32
    w, q = i // 32, i % 32
    c, e = q // 4, q % 4
    h = np.minimum(32, n - 1 - 32 * g)
    base = 4 * (128 * g * (g - 1) + 144 * g) + 32 * h * w
    off = base + 4 * (h * c + l) + e
    bc = np.zeros_like(c)
    for k in range(8):
        bc += np.where(k < c, np.maximum(0, h - 4 * k), 0)
    diag = base + 4 * (bc + l - 4 * c) + e
    return r, i, np.where(w < g, off, diag)


def dense_to_blk(dense: np.ndarray, upper: float = 0.0) -> np.ndarray:
    """Repack [count][n][ld] dense S* into CM_LAYOUT_BLK (strict lower part only)."""
    count, n, _ = dense.shape
    out = np.full((count, blk_size(n)), np.float32(upper), np.float32)
    r, i, pos = blk_positions(n)
    out[:, pos] = dense[:, r, i]
    return out


def gen_sstar(graph, family: str, seed: int, s_begin: int, count: int,
              layout: str = "dense", ld: int | None = None, upper: float = 0.0) -> np.ndarray:
    """Generate S* #s_begin .. s_begin+count-1 for ``graph``.

    Returns float32 array [count][n][ld] (dense), [count][tri4_size(n)] (tri4) or
    [count][blk_size(n)] (blk).
    """
    n = graph.n
    if layout == "blk":
        return dense_to_blk(gen_sstar(graph, family, seed, s_begin, count, upper=upper), upper=upper)
    if layout == "dense":
        ld = roundup4(n) if ld is None else ld
        assert ld >= n and ld % 4 == 0
        out = np.full((count, n, ld), np.float32(upper), np.float32)
    elif layout == "tri4":
        out = np.full((count, tri4_size(n)), np.float32(upper), np.float32)
        offs = [tri4_offset(r) for r in range(n)]
    else:
        raise ValueError(layout)
    last = graph.last_use()
    lastF = graph.last_forward_use()
    for c in range(count):
        s = s_begin + c
        fam = family_of(family, seed, s)
        if fam == "g1":
            K, tau = g1_params(seed, s, graph.L)
        for r in range(n):
            if fam == "g2":
                row = g2_row(seed, s, r)
            elif fam == "g1":
                row = g1_row(seed, s, r, graph.L, K, tau, last, lastF)
            else:
                raise ValueError(fam)
            if layout == "dense":
                out[c, r, :r] = row
            else:
                out[c, offs[r]:offs[r] + r] = row
    return out


def from_binary(S: np.ndarray, ld: int | None = None, upper: float = 0.0) -> np.ndarray:
    """G0: an exact 0/1 pattern S[r][i] (r = 0-based stage row, only i < r used) -> dense fp32."""
    n = S.shape[0]
    ld = roundup4(n) if ld is None else ld
    out = np.full((n, ld), np.float32(upper), np.float32)
    for r in range(n):
        out[r, :r] = S[r, :r].astype(np.float32)
    return out


def dense_to_tri4(dense: np.ndarray) -> np.ndarray:
    """Repack [count][n][ld] dense S* into the tri4 layout (strict lower part only)."""
    count, n, _ = dense.shape
    out = np.zeros((count, tri4_size(n)), np.float32)
    for r in range(n):
        o = tri4_offset(r)
        out[:, o:o + r] = dense[:, r, :r]
    return out
