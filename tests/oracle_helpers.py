"""Test-side helpers: binary S patterns written from their definitions."""
from __future__ import annotations

import numpy as np

from workloads import graphs as G
from workloads.sstar import from_binary


def S_zero(n):
    return np.zeros((n, n), bool)


def S_all(n):
    """keep everything: S_{t,i} = 1 for all i < t (0-based rows r = t-1)."""
    return np.tril(np.ones((n, n), bool), -1)


def S_liveness(g):
    """S_{t,i} = [i < t <= last(i)] (1-based); 0-based: [i < r <= last0(i)]."""
    n = g.n
    last = g.last_use()
    S = np.zeros((n, n), bool)
    for r in range(n):
        for i in range(r):
            S[r, i] = r <= last[i]
    return S


def S_chen(L, K):
    """Chen-segmented S on the training chain; 1-based K."""
    n = 2 * L + 1
    S1 = np.zeros((n + 2, n + 2), bool)
    for t in range(2, n + 1):
        S1[t, t - 1] = True
    for c in K:
        for t in range(c + 1, 2 * L + 2 - c + 1):
            S1[t, c] = True
    seg = []
    segs = []
    for v in range(1, L + 1):
        if v in K:
            if seg:
                segs.append(seg)
            seg = []
        else:
            seg.append(v)
    if seg:
        segs.append(seg)
    for sg in segs:
        tau = max(sg)
        for i in sg:
            if i == tau:
                continue
            for t in range(2 * L + 2 - tau + 1, 2 * L + 2 - i + 1):
                S1[t, i] = True
    return S1[1:n + 1, 1:n + 1]


def sstar_of(S):
    return from_binary(S)


def chain_weighted(L, cost, mem, ovh):
    g = G.training_chain(L)
    g.cost = np.asarray(cost, np.int64)
    g.mem = np.asarray(mem, np.int64)
    g.ovh = ovh
    return g
