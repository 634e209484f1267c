"""Pins of execution-plan emission and hoisting (Alg. 1 PAPER.md:331-356,
code motion PAPER.md:328).

The hoisted plan must simulate cleanly (every used value resident, no double free), never
raise the peak, and its peak must equal the closed form max_t max_k (U_{t,k} - H_t) with H_t
the memory of stage t's spurious checkpoints (they are resident for the whole stage under
Eq. 9, so hoisting lowers every U_{t,k} of the stage by exactly H_t)."""
import numpy as np

from oracle import (Instance, evaluate, generate_plan, hoisted_plan, simulate_plan,
                    spurious_checkpoints)
from workloads import graphs as G
from workloads.sstar import from_binary, gen_sstar


def cases():
    rng = np.random.default_rng(11)
    for trial in range(40):
        g = G.random_dag(int(rng.integers(3, 12)), 0.35, trial) if trial % 2 else \
            G.random_training(int(rng.integers(3, 8)), 0.2, trial)
        if trial % 3 == 0:      # binary S with spurious checkpoints on purpose
            x = from_binary(np.tril(rng.random((g.n, g.n)) < 0.3, -1))
        else:
            x = gen_sstar(g, "mix", 3, trial, 1)[0]
        yield g, x


def test_hoisted_plan_properties():
    seen_hoist = 0
    for g, x in cases():
        inst = Instance.from_graph(g)
        o = evaluate(inst, x, 0.5, keep=True)
        R, S, FREE, U = o["R"], o["S"], o["FREE"], o["U"]
        plain = generate_plan(inst, R, FREE)
        hoist = hoisted_plan(inst, R, S, FREE)
        p0, c0 = simulate_plan(inst, plain, S)
        p1, c1 = simulate_plan(inst, hoist, S)
        assert (p0, c0) == (o["peak"], o["cost"])                    # invariant 6
        assert c1 == c0 and p1 <= p0
        H = {t: sum(int(inst.M[i]) for i in spurious_checkpoints(inst, R, S, t)) for t in range(1, g.n + 1)}
        closed = max(int(U[t - 1, k]) - H[t] for t in range(1, g.n + 1) for k in range(1, g.n + 1) if R[t, k])
        assert p1 == closed
        n_hoisted = sum(len(spurious_checkpoints(inst, R, S, t)) for t in range(1, g.n + 1))
        assert len(hoist) == len(plain) + n_hoisted
        assert len(plain) == int(R[1:g.n + 1, 1:].sum()) + sum(int(v.sum()) for v in FREE.values())
        seen_hoist += n_hoisted > 0 and p1 < p0
    assert seen_hoist >= 3                                         # hoisting actually mattered


def test_no_spurious_checkpoints_in_liveness_schedule():
    """The liveness schedule keeps a value exactly while it has a later user: nothing to hoist."""
    from tests.oracle_helpers import S_liveness
    g = G.training_chain(6)
    inst = Instance.from_graph(g)
    o = evaluate(inst, from_binary(S_liveness(g)), 0.5, keep=True)
    assert all(not spurious_checkpoints(inst, o["R"], o["S"], t) for t in range(1, g.n + 1))
