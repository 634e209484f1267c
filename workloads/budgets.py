"""Budget grids and threshold lists (SURVEY §8(d) "Budget rules").

Input placement only: these graph-level quantities decide WHERE budgets sit on
the memory axis; they are not the hot path's per-candidate accounting.

  P_live  = ovh + max_t (M_t + sum_{i < t <= last(i)} M_i)   (checkpoint-all liveness)
  P_floor = ovh + max_k (M_k + sum_{i in DEPS(k)} M_i)
  grid    = 16 geometric points from max(P_floor, 0.2 P_live) to P_live, floored
"""
from __future__ import annotations

import numpy as np


def p_live(g) -> int:
    last = g.last_use()
    best = 0
    for t in range(g.n):
        live = int(g.mem[t]) + sum(int(g.mem[i]) for i in range(t) if last[i] >= t)
        best = max(best, live)
    return g.ovh + best


def p_floor(g) -> int:
    deps = [[] for _ in range(g.n)]
    for (i, j) in g.edges:
        deps[j].append(i)
    return g.ovh + max(int(g.mem[k]) + sum(int(g.mem[i]) for i in deps[k]) for k in range(g.n))


def geometric_grid(g, points: int = 16) -> np.ndarray:
    hi = p_live(g)
    lo = max(p_floor(g), int(0.2 * hi))
    if points == 1:
        return np.array([hi], np.int64)
    r = (hi / lo) ** (1.0 / (points - 1))
    out = [int(lo * r ** j) for j in range(points)]
    out[-1] = hi
    return np.array(out, np.int64)


def unet_grid(g_base) -> np.ndarray:
    """Config 4: P_live(base M) x {1, 1.25, 1.5, 2}; candidates run with 5x-scaled M."""
    pl = p_live(g_base)
    return np.array([int(pl * f) for f in (1.0, 1.25, 1.5, 2.0)], np.int64)


def eq13_cost_limit(g) -> int:
    """Eq. 13's right side: 2 sum_{fwd} C_i + sum_{bwd} C_i, with the
    training graph's forward nodes 0..L-1 and the loss node L counted as forward (R2).
    Caller-side input of the max-batch epilogue, like the budgets."""
    c = np.asarray(g.cost, np.int64)
    return int(2 * c[: g.L + 1].sum() + c[g.L + 1:].sum())
