"""Pins for the CPU oracle against values fixed by the paper and by mathematics
(closed forms, the Fig. 4 example, brute-force Pareto fronts).  CPU only."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import Instance, best_per_budget, evaluate
from tests.oracle_helpers import S_all, S_chen, S_liveness, S_zero, chain_weighted, sstar_of
from workloads import graphs as G

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def run(g, S, theta=0.5, keep=False):
    return evaluate(Instance.from_graph(g), sstar_of(S), theta, keep=keep)


@pytest.mark.parametrize("key", ["path8_unit", "path8_weighted"])
def test_path_golden(key):
    d = GOLD[key]
    g = G.path(d["n"], d["cost"], d["mem"], d["ovh"])
    pats = {"zero": S_zero(g.n), "all": S_all(g.n), "liveness": S_liveness(g)}
    for case, want in d["cases"].items():
        out = run(g, pats[case])
        assert (out["cost"], out["peak"]) == (want["cost"], want["peak"]), case


def test_chain17_golden():
    d = GOLD["chain17"]
    g = G.training_chain(d["L"])
    assert g.n == 17 and len(g.edges) == 3 * d["L"]
    pats = {"zero": S_zero(g.n), "all": S_all(g.n), "liveness": S_liveness(g)}
    for case, want in d["cases"].items():
        out = run(g, pats[case])
        assert (out["cost"], out["peak"]) == (want["cost"], want["peak"]), case


@pytest.mark.parametrize("case", GOLD["chen_segmented"]["cases"])
def test_chen_segmented_golden(case):
    L, K = case["L"], case["K"]
    g = G.training_chain(L)
    out = run(g, S_chen(L, K))
    assert (out["cost"], out["peak"]) == (case["cost"], case["peak"])
    # the closed form itself: cost = n + (L - |K|)
    assert out["cost"] == g.n + L - len(K)


def test_fig4_golden():
    d = GOLD["fig4"]
    g = G.fig4_fixture()
    out = run(g, S_zero(5), keep=True)
    R, U, FREE = out["R"], out["U"], out["FREE"]
    for t, row in enumerate(d["R_rows"], start=1):
        assert sorted(np.nonzero(R[t, 1:])[0] + 1) == row
    assert U[4, 4] == d["U_5_4"] and U[4, 5] == d["U_5_5"]
    assert (out["peak"], out["cost"]) == (d["peak"], d["cost"])
    a, b, c, k, j = 1, 2, 3, 4, 5
    f5 = d["FREE_5"]
    assert FREE[(b, k)][4] == f5["b_at_k"] and FREE[(c, k)][4] == f5["c_at_k"]
    assert FREE[(a, k)][4] == f5["a_at_k"] and FREE[(a, j)][4] == f5["a_at_j"]
    sf = d["self_free"]
    assert FREE[(k, k)][3] == sf["t4_k"] and FREE[(j, j)][4] == sf["t5_j"]
    assert FREE[(k, k)][4] == sf["t5_k"]


# ---------------------------------------------------------------- closed forms on random DAGs

def ancestors(g):
    n = g.n
    anc = [set() for _ in range(n)]
    for j in range(n):
        for (i, jj) in g.edges:
            if jj == j:
                anc[j] |= anc[i] | {i}
    return anc


@pytest.mark.parametrize("seed", range(12))
def test_closed_forms_random_dag(seed):
    g = G.random_dag(7 + seed % 5, 0.35, seed)
    n = g.n
    last = g.last_use()
    # keep-all: R = I, cost = sum C, peak = ovh + sum M
    out = run(g, S_all(n))
    assert out["cost"] == int(g.cost.sum())
    assert out["peak"] == g.ovh + int(g.mem.sum())
    # liveness: R = I, cost = sum C, peak = ovh + max_t(M_t + sum_{i<t<=last(i)} M_i)
    out = run(g, S_liveness(g), keep=True)
    assert out["cost"] == int(g.cost.sum())
    want = g.ovh + max(int(g.mem[t]) + sum(int(g.mem[i]) for i in range(t) if last[i] >= t)
                       for t in range(n))
    assert out["peak"] == want
    # S = 0: R_t = {t} u ancestors(t)
    anc = ancestors(g)
    out = run(g, S_zero(n), keep=True)
    for t in range(n):
        assert set(np.nonzero(out["R"][t + 1, 1:])[0]) == anc[t] | {t}
    assert out["cost"] == sum(int(g.cost[i]) for t in range(n) for i in anc[t] | {t})


@pytest.mark.parametrize("n", [1, 2, 3, 6, 11])
def test_path_zero_closed_form(n):
    rng = np.random.default_rng(n)
    C = rng.integers(0, 50, n)
    M = rng.integers(0, 50, n)
    g = G.path(n, C, M, ovh=7)
    out = run(g, S_zero(n))
    assert out["cost"] == sum((n - i) * int(C[i]) for i in range(n))
    want = 7 + max([int(M[0])] + [int(M[k - 1] + M[k]) for k in range(1, n)])
    assert out["peak"] == want


@pytest.mark.parametrize("L", [1, 2, 5, 9])
def test_training_chain_closed_forms(L):
    g = G.training_chain(L)
    n = g.n
    assert (n, len(g.edges)) == (2 * L + 1, 3 * L)
    assert (run(g, S_liveness(g))["cost"], run(g, S_liveness(g))["peak"]) == (2 * L + 1, L + 2)
    out = run(g, S_zero(n))
    assert (out["cost"], out["peak"]) == (n * (n + 1) // 2, L + 2)
    out = run(g, S_all(n))
    assert (out["cost"], out["peak"]) == (n, n)


# ---------------------------------------------------------------- brute-force Pareto fronts

def pareto_front(g):
    n = g.n
    pos = [(r, i) for r in range(n) for i in range(r)]
    pts = {}
    inst = Instance.from_graph(g)
    for bits in itertools.product((0, 1), repeat=len(pos)):
        S = np.zeros((n, n), bool)
        for (r, i), b in zip(pos, bits):
            S[r, i] = b
        out = evaluate(inst, sstar_of(S), 0.5)
        p, c = out["peak"], out["cost"]
        pts[p] = min(pts.get(p, c), c)
    front = []
    for p in sorted(pts):
        if not front or pts[p] < front[-1][1]:
            front.append([p, pts[p]])
    return front


@pytest.mark.parametrize("case", [c for c in GOLD["pareto_fronts"]["cases"] if not c.get("slow")])
def test_pareto_front_golden(case):
    if case["graph"] == "path":
        g = G.path(case["n"])
    elif case["graph"] == "chain":
        g = G.training_chain(case["L"])
    else:
        g = chain_weighted(case["L"], case["cost"], case["mem"], case["ovh"])
    assert pareto_front(g) == case["front"]


def test_best_per_budget_matches_front():
    """A7 on all 2^10 binary S of the L=2 chain: best cost per budget is the front's step
    function; budgets below the front are infeasible (idx -1)."""
    g = G.training_chain(2)
    n = g.n
    pos = [(r, i) for r in range(n) for i in range(r)]
    inst = Instance.from_graph(g)
    peaks, costs = [], []
    for bits in itertools.product((0, 1), repeat=len(pos)):
        S = np.zeros((n, n), bool)
        for (r, i), b in zip(pos, bits):
            S[r, i] = b
        out = evaluate(inst, sstar_of(S), 0.5)
        peaks.append(out["peak"])
        costs.append(out["cost"])
    best = best_per_budget(peaks, costs, [2, 3, 4, 5])
    assert best[0] == (-1, None)
    assert best[1][1] == 6 and best[2][1] == 5 and best[3][1] == 5
    # lowest index among ties (Q11)
    for (idx, cost), b in zip(best[1:], [3, 4, 5]):
        ties = [c for c in range(len(peaks)) if peaks[c] <= b and costs[c] == cost]
        assert idx == min(ties)
