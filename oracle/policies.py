"""CPU ORACLE: baseline checkpoint policies (Table 1 PAPER.md:103-125,
PAPER.md:447-455; App. B).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the CUDA path.

A policy picks a checkpoint set K among the forward nodes 1..L of a training graph (forward
f_1..f_L, loss L+1, b_v = 2L+2-v); S follows from K (R3), then the optimal R and the
accounting are Alg. 2's phase 2 as for a rounded S ("implement baselines as a static policy for
the decision variable S and then solve for the lowest-cost recomputation schedule").

  candidates   Chen / linearized: every forward node in topological order;
               AP: the articulation points of the undirected forward graph plus its first and
               last node ("or the input if there is no such AP"; R5),
               found here by brute force (remove v, count components).
  sqrt         s = ceil(sqrt(|cands|)); every s-th candidate, the last forward node excluded
               (SPEC.md chen_sqrt: L = 16 -> {4, 8, 12}).
  greedy(b)    walk f_1..f_L accumulating M; at a candidate with accumulated >= b (not f_L):
               checkpoint it and reset (R4).
  all          K = every forward node (checkpoint all: S is then pure liveness).
  S from K     for i < t:  i > L (loss, gradients): t <= last(i);  i in K: t <= last(i);
               i forward not in K: t <= lastF(i)  or  2L+2 - tau(i) < t <= last(i)
               (last = latest user, lastF = latest forward user incl. the loss, tau(i) = top of
               i's maximal run of non-K forward nodes: recomputed at tau's backward stage).
"""
from __future__ import annotations

import math

import numpy as np

from .checkmate_oracle import Instance, evaluate_S


def forward_edges(inst: Instance, L: int):
    return [(i, j) for (i, j) in inst.E if j <= L]


def components(nodes, edges) -> int:
    nodes = set(nodes)
    adj = {v: [] for v in nodes}
    for (i, j) in edges:
        if i in nodes and j in nodes:
            adj[i].append(j)
            adj[j].append(i)
    seen, comps = set(), 0
    for v in sorted(nodes):
        if v in seen:
            continue
        comps += 1
        stack = [v]
        seen.add(v)
        while stack:
            u = stack.pop()
            for w in adj[u]:
                if w not in seen:
                    seen.add(w)
                    stack.append(w)
    return comps


def articulation_points(inst: Instance, L: int):
    """Brute force: v is an AP iff removing it increases the number of components."""
    fe = forward_edges(inst, L)
    base = components(range(1, L + 1), fe)
    return [v for v in range(1, L + 1)
            if components([u for u in range(1, L + 1) if u != v], fe) > base]


def candidates(inst: Instance, L: int, family: str):
    if family == "ap":
        return sorted(set(articulation_points(inst, L)) | {1, L})
    return list(range(1, L + 1))


def sqrt_K(cands, L: int):
    s = math.ceil(math.sqrt(len(cands)))
    return {c for j, c in enumerate(cands) if (j + 1) % s == 0 and c != L}


def greedy_K(inst: Instance, cands, L: int, b: int):
    cs = set(cands)
    K, acc = set(), 0
    for v in range(1, L + 1):
        acc += int(inst.M[v])
        if v in cs and acc >= b and v != L:
            K.add(v)
            acc = 0
    return K


def policy_K(inst: Instance, L: int, policy: str, b: int = 0):
    """policy in {'all', 'chen_sqrt', 'chen_greedy', 'ap_sqrt', 'ap_greedy', 'lin_sqrt',
    'lin_greedy'}; chen_* and lin_* coincide on topologically numbered graphs."""
    if policy == "all":
        return set(range(1, L + 1))
    family, kind = policy.split("_")
    cands = candidates(inst, L, "ap" if family == "ap" else "lin")
    return sqrt_K(cands, L) if kind == "sqrt" else greedy_K(inst, cands, L, b)


def S_from_K(inst: Instance, L: int, K) -> np.ndarray:
    """Binary S[t][i] in round_S's layout ([n+2][n+1], 1-based) from a checkpoint set."""
    n = inst.n
    last = [i for i in range(n + 1)]
    lastF = [i for i in range(n + 1)]
    for (i, j) in inst.E:
        last[i] = max(last[i], j)
        if j <= L + 1:
            lastF[i] = max(lastF[i], j)
    tau = [0] * (n + 1)
    top = 0
    for v in range(L, 0, -1):
        if v in K:
            top = 0
        else:
            top = top or v
            tau[v] = top
    S = np.zeros((n + 2, n + 1), dtype=bool)
    for t in range(1, n + 1):
        for i in range(1, t):
            if i > L:
                S[t, i] = t <= last[i]
            elif i in K:
                S[t, i] = t <= last[i]
            else:
                S[t, i] = t <= lastF[i] or (2 * L + 2 - tau[i] < t <= last[i])
    return S


def evaluate_policy(inst: Instance, L: int, policy: str, b: int = 0, keep=False) -> dict:
    K = policy_K(inst, L, policy, b)
    out = evaluate_S(inst, S_from_K(inst, L, K), keep=keep)
    out["K"] = K
    return out
