"""CPU ORACLE for Checkmate two-phase rounding + memory accounting.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product path
(paper_1910_02653_b200) never imports it and shares no code with it.

Plain, slow, obviously correct: it follows the paper step by step, 1-based
indices as in the paper, numpy vectors over the independent stage axis t only
(each stage's constraints are independent, so evaluating them for all t at
once is the same per-stage computation written in lockstep).

  A1  round      S_{t,i} = 1[S*_{t,i} > theta], i < t           Alg. 2 line 1, PAPER.md:395;
                 strict '>', fp32 compare, NaN -> 0 (Q6);
                 strict lower triangle (12b); S_{n+1} := 0 (Q3)
  A2  R <- I_n                                                   Alg. 2 line 2; (12a) PAPER.md:296
  A3a while (3) violated: R_{t-1,i} <- 1                         Alg. 2 lines 3-5; (3) PAPER.md:189
  A3b while (2) violated: R_{t,i} <- 1, each stage scanned right to left
                                                                 Alg. 2 lines 6-8; (2) PAPER.md:188
  A4  FREE_{t,i,k} = R_{t,k} (1 - S_{t+1,i}) prod_{j in USERS(i), j>k} (1 - R_{t,j})
                 for i in DEPS(k) u {k}                          Eq. 9; Eq. 8 set PAPER.md:220 (Q4)
  A5  U_{t,0} = ovh + sum_i M_i S_{t,i}                          Eq. 6
      U_{t,k} = U_{t,k-1} - GC(v_{k-1}, t) + R_{t,k} M_k, GC(v_0,t) = 0
      GC(v_k, t) = sum_{i in DEPS(k) u {k}} M_i FREE_{t,i,k}     Eqs. 7-8
      peak = max_{t, k>=1} U_{t,k}                               Fig. 4 caption PAPER.md:168 (Q8, Q9)
  A6  cost = sum_t sum_i C_i R_{t,i}                             objective (1)
  A7  best_b = argmin_{c : peak_c <= b} (cost_c, c), -1 if none  budget row PAPER.md:311 (Q7, Q11, Q12)
  A8  counters: sum R, sum S, closure visits, free events        (SURVEY §8(d) algorithmic ops)

Integers are int64 (bit-exact units); evaluate() asserts the
int64 bounds it relies on.
"""
from __future__ import annotations

import numpy as np

INT64_MAX = (1 << 63) - 1


class Instance:
    """A DAG G=(V,E) with per-node C, M and the Eq. 6 constant.

    ``edges`` are 0-based pairs (i, j), i < j; internally stored 1-based."""

    def __init__(self, n, edges, cost, mem, ovh):
        self.n = int(n)
        E = sorted({(int(i) + 1, int(j) + 1) for (i, j) in edges})
        assert len(E) == len(edges), "E is a set (PAPER.md:158): duplicate edge"
        for (i, j) in E:
            assert 1 <= i < j <= self.n, "nodes numbered in topological order (PAPER.md:159-160)"
        self.E = E
        self.C = np.zeros(self.n + 1, np.int64)
        self.M = np.zeros(self.n + 1, np.int64)
        self.C[1:] = np.asarray(cost, np.int64)
        self.M[1:] = np.asarray(mem, np.int64)
        self.ovh = int(ovh)
        assert (self.C >= 0).all() and (self.M >= 0).all() and self.ovh >= 0
        # DEPS(k) = {i : (v_i, v_k) in E}, USERS(i) = {j : (v_i, v_j) in E}
        self.DEPS = [[] for _ in range(self.n + 1)]
        self.USERS = [[] for _ in range(self.n + 1)]
        for (i, j) in E:
            self.DEPS[j].append(i)
            self.USERS[i].append(j)
        assert self.ovh + int(self.M.sum()) < (1 << 62)
        assert sum((self.n - i + 1) * int(self.C[i]) for i in range(1, self.n + 1)) < (1 << 62)

    @classmethod
    def from_graph(cls, g):
        return cls(g.n, g.edges, g.cost, g.mem, g.ovh)


def round_S(inst: Instance, sstar, theta) -> np.ndarray:
    """A1.  Returns bool S[t][i], t = 0..n+1, i = 0..n (row 0, row n+1 and column 0 are 0).

    ``sstar`` is indexable as sstar[t-1][i-1] (any row-major [n][>=n] array); only
    i < t is read (Eq. 12b)."""
    n = inst.n
    th = np.float32(theta)
    S = np.zeros((n + 2, n + 1), dtype=bool)
    for t in range(1, n + 1):
        row = np.asarray(sstar[t - 1][: t - 1], dtype=np.float32)
        S[t, 1:t] = row > th           # NaN > th is False
    return S


def two_phase_R(inst: Instance, S: np.ndarray, counters: dict | None = None) -> np.ndarray:
    """A2-A3: the minimal R given S (Alg. 2 phase 2).  R[t][i], t = 0..n+1, i = 0..n."""
    n = inst.n
    R = np.zeros((n + 2, n + 1), dtype=bool)
    for t in range(1, n + 1):                         # R <- I_n
        R[t, t] = True
    # while exists t >= 2, i: S_{t,i} > R_{t-1,i} + S_{t-1,i}: R_{t-1,i} <- 1.
    # Setting R_{t-1,i} only touches constraint (3) at (t, i), so fixing every violation
    # found in one scan is the same as fixing them one at a time.
    while True:
        viol = S[2:n + 1, :] & ~R[1:n, :] & ~S[1:n, :]
        if not viol.any():
            break
        R[1:n, :] |= viol
    # while exists t, (i,j) in E: R_{t,j} > R_{t,i} + S_{t,i}: R_{t,i} <- 1, scanning each
    # stage in reverse topological order, right to left.  The outer loop
    # re-scans until a full scan finds no violation (the literal "while").
    T = slice(1, n + 1)
    while True:
        changed = False
        for j in range(n, 0, -1):
            for i in sorted(inst.DEPS[j], reverse=True):
                viol = R[T, j] & ~R[T, i] & ~S[T, i]
                if viol.any():
                    R[T, i] |= viol
                    changed = True
        if not changed:
            break
    if counters is not None:
        counters["closure_visits"] = int(sum(R[T, k].sum() * len(inst.DEPS[k]) for k in range(1, n + 1)))
    return R


def free_matrix(inst: Instance, R: np.ndarray, S: np.ndarray) -> dict:
    """A4, Eq. 9: FREE[(i, k)] = bool vector over t = 1..n (index t-1)."""
    n = inst.n
    T = slice(1, n + 1)
    Tn = slice(2, n + 2)                              # S_{t+1}, with S_{n+1} = 0
    FREE = {}
    for k in range(1, n + 1):
        for i in inst.DEPS[k] + [k]:
            f = R[T, k] & ~S[Tn, i]
            for j in inst.USERS[i]:
                if j > k:
                    f = f & ~R[T, j]
            FREE[(i, k)] = f
    return FREE


def memory_U(inst: Instance, R: np.ndarray, S: np.ndarray, FREE: dict) -> np.ndarray:
    """A5, Eqs. 6-8: U[t-1][k] for t = 1..n, k = 0..n (int64)."""
    n = inst.n
    T = slice(1, n + 1)
    U = np.zeros((n, n + 1), np.int64)
    U[:, 0] = inst.ovh + (S[T, 1:].astype(np.int64) * inst.M[1:]).sum(axis=1)
    for k in range(1, n + 1):
        gc = np.zeros(n, np.int64)                    # GC(v_{k-1}, t); GC(v_0, t) = 0
        if k - 1 >= 1:
            for i in inst.DEPS[k - 1] + [k - 1]:
                gc += inst.M[i] * FREE[(i, k - 1)].astype(np.int64)
        U[:, k] = U[:, k - 1] - gc + R[T, k].astype(np.int64) * inst.M[k]
    return U


def evaluate(inst: Instance, sstar, theta, keep=False) -> dict:
    """One candidate (S*, theta): A1-A6 (+ A8 counters)."""
    return evaluate_S(inst, round_S(inst, sstar, theta), keep=keep)


def evaluate_S(inst: Instance, S: np.ndarray, keep=False) -> dict:
    """A2-A6 (+ A8 counters) for a rounded S[t][i] (the layout round_S returns)."""
    n = inst.n
    counters = {}
    R = two_phase_R(inst, S, counters)
    FREE = free_matrix(inst, R, S)
    U = memory_U(inst, R, S, FREE)
    T = slice(1, n + 1)
    peak = int(U[:, 1:].max())
    cost = int((R[T, 1:].astype(np.int64) * inst.C[1:]).sum())
    counters["sum_R"] = int(R[T, 1:].sum())
    counters["sum_S"] = int(S[T, 1:].sum())
    counters["free_events"] = int(sum(int(v.sum()) for v in FREE.values()))
    out = {"peak": peak, "cost": cost, "counters": counters}
    if keep:
        out.update(S=S, R=R, FREE=FREE, U=U)
    return out


def best_per_budget(peaks, costs, budgets, index_base: int = 0):
    """A7: for each budget b, the candidate c minimising (cost_c, c) among peak_c <= b.

    Returns a list of (idx, cost); idx = -1 (cost = None) if no candidate fits."""
    out = []
    for b in budgets:
        best = None
        for c, (p, q) in enumerate(zip(peaks, costs)):
            if p <= b:
                key = (int(q), index_base + c)
                if best is None or key < best:
                    best = key
        out.append((-1, None) if best is None else (best[1], best[0]))
    return out


def masks_u64(inst: Instance, X: np.ndarray) -> np.ndarray:
    """Pack rows t = 1..n of a bool matrix X[t][i] into u64 words: bit (i-1)%64 of
    word (i-1)//64 in row t-1 (the C-ABI's mask layout)."""
    n = inst.n
    W = (n + 63) // 64
    out = np.zeros((n, W), np.uint64)
    for t in range(1, n + 1):
        for i in np.nonzero(X[t, 1:])[0]:
            out[t - 1, i // 64] |= np.uint64(1) << np.uint64(i % 64)
    return out
