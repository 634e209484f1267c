"""Oracle invariants (SURVEY §8(c) 'Invariants'), brute force on tiny inputs and the
independent plan / greedy simulators.  CPU only."""
import random

import numpy as np
import pytest

from oracle import Instance, evaluate
from oracle.checkmate_oracle import round_S, two_phase_R
from oracle.plan_sim import (brute_force_min_R, constraints_hold, generate_plan, simulate_greedy,
                             simulate_plan)
from workloads import graphs as G
from workloads.sstar import gen_sstar


def cases(count, nmax=8):
    out = []
    for s in range(count):
        if s % 3 == 2:
            g = G.random_training(1 + s % 4, 0.3, s)
        else:
            g = G.random_dag(2 + s % (nmax - 1), 0.3 + 0.1 * (s % 4), s)
        fam = "g2" if s % 2 else "g1"
        sstar = gen_sstar(g, fam, seed=100 + s, s_begin=s, count=1)[0]
        theta = [0.5, 0.3, 0.7, 0.9][s % 4]
        out.append((g, sstar, theta))
    return out


CASES = cases(160)


@pytest.mark.parametrize("g,sstar,theta", CASES[:160])
def test_invariants(g, sstar, theta):
    inst = Instance.from_graph(g)
    out = evaluate(inst, sstar, theta, keep=True)
    R, S, FREE, U = out["R"], out["S"], out["FREE"], out["U"]
    n = g.n
    # 1. R_t[t] = 1, R lower triangular, R and S disjoint
    for t in range(1, n + 1):
        assert R[t, t]
        assert not R[t, t + 1:].any()
        assert not (R[t] & S[t]).any()
    # 2. constraints (2), (3), (12a-c)
    assert constraints_hold(inst, R, S)
    # 3. minimality: clearing any off-diagonal R bit breaks (2) or (3)
    for t in range(1, n + 1):
        for i in range(1, t):
            if R[t, i]:
                R2 = R.copy()
                R2[t, i] = False
                assert not constraints_hold(inst, R2, S), (t, i)
    # 4. Theorem 1: sum_{k in USERS(i)} FREE_{t,i,k} <= 1
    for i in range(1, n + 1):
        tot = np.zeros(n, int)
        for k in inst.USERS[i]:
            tot += FREE[(i, k)].astype(int)
        assert (tot <= 1).all()
    # 5. FREE = 1 <=> num_hazards = 0  (Lemma 1)
    for (i, k), f in FREE.items():
        for t in range(1, n + 1):
            hz = (1 - int(R[t, k])) + int(S[t + 1, i]) + sum(int(R[t, j]) for j in inst.USERS[i] if j > k)
            assert bool(f[t - 1]) == (hz == 0)
    # 6. Alg. 1 plan simulated with stage-boundary drop == U peak; without drop >= (caveat)
    plan = generate_plan(inst, R, FREE)
    peak_plan, cost_plan = simulate_plan(inst, plan, S, drop_at_boundary=True)
    assert (peak_plan, cost_plan) == (out["peak"], out["cost"])
    peak_nodrop, _ = simulate_plan(inst, plan, S, drop_at_boundary=False)
    assert peak_nodrop >= out["peak"]
    # statement count = sum R + sum FREE  (SPEC plan examples)
    assert len(plan) == out["counters"]["sum_R"] + out["counters"]["free_events"]
    # greedy set-based simulation (no FREE matrix)
    assert simulate_greedy(inst, R, S) == (out["peak"], out["cost"])
    # 7. floor
    floor = g.ovh + max(int(g.mem[k]) + sum(int(g.mem[i]) for i in inst_deps0(g, k)) for k in range(n))
    assert out["peak"] >= floor
    # max attained at a compute step (Q9): U_{t,0} <= max_k U_{t,k}
    assert (U[:, 0] <= U[:, 1:].max(axis=1)).all()


def inst_deps0(g, k):
    return [i for (i, j) in g.edges if j == k]


@pytest.mark.parametrize("g,sstar,theta", CASES[:60])
def test_linearity(g, sstar, theta):
    """peak(B*M) - ovh = B*(peak(M) - ovh); cost linear in C (SURVEY invariant 8)."""
    inst = Instance.from_graph(g)
    base = evaluate(inst, sstar, theta)
    for B in (2, 7):
        inst2 = Instance(g.n, g.edges, g.cost * B, g.mem * B, g.ovh)
        o = evaluate(inst2, sstar, theta)
        assert o["peak"] - g.ovh == B * (base["peak"] - g.ovh)
        assert o["cost"] == B * base["cost"]


@pytest.mark.parametrize("g,sstar,theta", [c for c in CASES if c[0].n <= 5][:40])
def test_brute_force_min_R(g, sstar, theta):
    """Alg. 2's R is the cheapest R satisfying (2), (3), (12a-c) for the rounded S
    ('optimal up to the choice of S')."""
    inst = Instance(g.n, g.edges, np.asarray(g.cost) + 1, g.mem, g.ovh)   # C > 0
    S = round_S(inst, sstar, theta)
    R = two_phase_R(inst, S)
    Rb = brute_force_min_R(inst, S)
    assert (R == Rb).all()


@pytest.mark.parametrize("seed", range(40))
def test_repair_order_irrelevant(seed):
    """Horn least model is unique: random-order fixpoint == oracle's R."""
    g = G.random_dag(3 + seed % 6, 0.4, seed)
    inst = Instance.from_graph(g)
    sstar = gen_sstar(g, "g2", seed=7, s_begin=seed, count=1)[0]
    S = round_S(inst, sstar, 0.5)
    R = two_phase_R(inst, S)
    n = g.n
    rng = random.Random(seed)
    R2 = np.zeros_like(R)
    for t in range(1, n + 1):
        R2[t, t] = True
    rules = [("3", t, i) for t in range(2, n + 1) for i in range(1, n + 1)] + \
            [("2", t, e) for t in range(1, n + 1) for e in inst.E]
    changed = True
    while changed:
        changed = False
        rng.shuffle(rules)
        for r in rules:
            if r[0] == "3":
                _, t, i = r
                if S[t, i] and not R2[t - 1, i] and not S[t - 1, i]:
                    R2[t - 1, i] = True
                    changed = True
            else:
                _, t, (i, j) = r
                if R2[t, j] and not R2[t, i] and not S[t, i]:
                    R2[t, i] = True
                    changed = True
    assert (R == R2).all()


def test_rounding_edges():
    """Strict '>' (Q1): exact ties round to 0; NaN rounds to 0 (Q6); entries i >= t are
    never read (Q5); theta in {0, 1}."""
    g = G.random_dag(6, 0.5, 3)
    inst = Instance.from_graph(g)
    n = g.n
    x = np.full((n, 8), np.nan, np.float32)          # upper triangle garbage
    for r in range(n):
        x[r, :r] = [0.5, 0.25, np.nan, 1.0, 0.0, 0.75][:r]
    S = round_S(inst, x, 0.5)
    for t in range(1, n + 1):
        want = [v > 0.5 for v in [0.5, 0.25, np.nan, 1.0, 0.0, 0.75][:t - 1]]
        assert list(S[t, 1:t]) == want
        assert not S[t, t:].any()
    assert not round_S(inst, x, 1.0)[1:n + 1].any()
    S0 = round_S(inst, x, 0.0)
    assert S0[4, 1] == (np.float32(0.5) > 0) and S0[5, 5 - 1] == (np.float32(1.0) > 0)
    assert not S[n + 1].any()


def test_upper_triangle_never_read():
    g = G.random_training(3, 0.5, 1)
    a = gen_sstar(g, "g1", 5, 0, 1, upper=0.0)[0]
    b = gen_sstar(g, "g1", 5, 0, 1, upper=np.nan)[0]
    inst = Instance.from_graph(g)
    oa, ob = evaluate(inst, a, 0.5), evaluate(inst, b, 0.5)
    assert (oa["peak"], oa["cost"]) == (ob["peak"], ob["cost"])
