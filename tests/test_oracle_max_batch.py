"""Pins of the max-batch epilogue (Eq. 13).

B_max is checked against a direct re-evaluation of the schedule (Eqs. 6-9) with every M_i
scaled by the batch: B_max fits the budget, B_max + 1 does not."""
import numpy as np

from oracle import B_CAP, Instance, b_max, evaluate, max_batch_per_budget
from workloads import graphs as G
from workloads.sstar import gen_sstar


def scaled(g, B):
    return Instance.from_graph(g.scaled(B))


def test_b_max_against_scaled_evaluation():
    rng = np.random.default_rng(3)
    for trial in range(12):
        g = G.random_training(6 + trial % 5, 0.2, trial)
        x = gen_sstar(g, "mix", 9, trial, 1)[0]
        base = evaluate(Instance.from_graph(g), x, 0.5)
        span = base["peak"] - g.ovh
        budget = base["peak"] + int(rng.integers(0, 6 * span))
        bm = b_max(base["peak"], budget, g.ovh)
        assert 1 <= bm < B_CAP
        assert evaluate(scaled(g, bm), x, 0.5)["peak"] <= budget
        assert evaluate(scaled(g, bm + 1), x, 0.5)["peak"] > budget
        # cost does not depend on M (Eq. 13's left side is batch-independent under the model)
        assert evaluate(scaled(g, bm), x, 0.5)["cost"] == base["cost"]


def test_special_cases():
    assert b_max(10, 5, 7) == 0            # budget below the fixed overhead
    assert b_max(7, 100, 7) == B_CAP       # no activation memory at all
    assert b_max(17, 27, 7) == 2


def test_per_budget_selection():
    peaks = [20, 15, 15, 40]
    costs = [5, 9, 6, 1]
    ovh = 10
    # budget 40: B = 3, 6, 6, 1 -> candidates 1 and 2 tie at 6; cost limit 8 excludes 1
    assert max_batch_per_budget(peaks, costs, [40], ovh, 8) == [(6, 2)]
    assert max_batch_per_budget(peaks, costs, [40], ovh, 100) == [(6, 1)]
    assert max_batch_per_budget(peaks, costs, [14], ovh, 100) == [(0, -1)]
    assert max_batch_per_budget(peaks, costs, [40], ovh, 0) == [(0, -1)]
    assert max_batch_per_budget(peaks, costs, [40], ovh, 100, index_base=7) == [(6, 8)]
