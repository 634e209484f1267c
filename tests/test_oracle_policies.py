"""Pins of the baseline checkpoint policies (R3-R5)."""
import numpy as np

from oracle import Instance, S_from_K, articulation_points, evaluate, evaluate_policy, policy_K
from tests.oracle_helpers import S_all, S_chen, S_liveness
from workloads import graphs as G
from workloads.sstar import from_binary


def test_chen_sqrt_closed_form():
    """SPEC chen_sqrt: L = 16 -> {4, 8, 12}; on the training chain S from K is the
    Chen-segmented pattern of SURVEY §8(c), whose cost / peak are closed forms (46, 9)."""
    L = 16
    g = G.training_chain(L)
    inst = Instance.from_graph(g)
    K = policy_K(inst, L, "chen_sqrt")
    assert K == {4, 8, 12}
    S = S_from_K(inst, L, K)
    assert np.array_equal(S[1:g.n + 1, 1:], S_chen(L, sorted(K)))
    o = evaluate_policy(inst, L, "chen_sqrt")
    assert (o["cost"], o["peak"]) == (46, 9)


def test_chen_segmented_table():
    """SURVEY §8(c) Chen-segmented closed forms through S_from_K on the training chain."""
    for L, K, cost, peak in [(10, {5, 9}, 29, 6), (12, {2, 7}, 35, 9), (8, {3, 6}, 23, 6),
                             (9, {3, 6}, 26, 7), (5, set(), 16, 7)]:
        g = G.training_chain(L)
        inst = Instance.from_graph(g)
        o = evaluate(inst, from_binary(S_from_K(inst, L, K)[1:g.n + 1, 1:]), 0.5)
        assert (o["cost"], o["peak"]) == (cost, peak), (L, K)


def test_checkpoint_all_is_liveness():
    """Table 1 'Checkpoint all': every value kept until its last use, cost sum C."""
    for seed in range(4):
        g = G.random_training(7, 0.3, seed)
        inst = Instance.from_graph(g)
        S = S_from_K(inst, g.L, set(range(1, g.L + 1)))
        assert np.array_equal(S[1:g.n + 1, 1:], S_liveness(g))
        o = evaluate_policy(inst, g.L, "all")
        assert o["cost"] == int(g.cost.sum())


def test_greedy_unit_chain():
    """SPEC chen_greedy: unit memory, b = 4, L = 16 -> a checkpoint every 4 nodes; b >= sum M
    -> no checkpoint."""
    g = G.training_chain(16)
    inst = Instance.from_graph(g)
    assert policy_K(inst, 16, "chen_greedy", 4) == {4, 8, 12}
    assert policy_K(inst, 16, "chen_greedy", 100) == set()


def test_articulation_points():
    """Path: every interior node; a diamond's interior is not; reductions on linear graphs
    ('all proposed generalizations exactly reproduce the original heuristics on
    linear networks')."""
    g = G.training_chain(9)
    inst = Instance.from_graph(g)
    assert articulation_points(inst, 9) == list(range(2, 9))
    for pol in ("sqrt", "greedy"):
        for b in (2, 3, 5):
            assert policy_K(inst, 9, f"ap_{pol}", b) == policy_K(inst, 9, f"chen_{pol}", b)
    # residual block 1 -> {2, 3} -> 4 -> 5: only the block's exit 4 is an AP (the block's
    # interior 2, 3 is not; the input 1 is a candidate anyway, R5)
    inst2 = Instance(5, [(0, 1), (0, 2), (1, 3), (2, 3), (3, 4)], np.ones(5), np.ones(5), 0)
    assert articulation_points(inst2, 5) == [4]


def test_resnet_aps_are_block_boundaries():
    g = G.resnet50()
    inst = Instance.from_graph(g)
    aps = articulation_points(inst, g.L)
    assert 10 <= len(aps) < g.L // 2                                   # boundaries, not interiors
    # every AP separates: no forward edge jumps over it
    for v in aps:
        assert not any(i < v < j for (i, j) in inst.E if j <= g.L)


def test_policies_are_feasible_and_ordered():
    """Every policy's schedule satisfies the constraints (phase 2 repairs nothing it needs) and
    checkpoint-all is the cheapest (cost sum C) with the highest peak among them."""
    g = G.random_training(12, 0.2, 7)
    inst = Instance.from_graph(g)
    res = {}
    for pol in ("all", "chen_sqrt", "ap_sqrt", "chen_greedy", "ap_greedy"):
        res[pol] = evaluate_policy(inst, g.L, pol, int(g.mem.sum()) // 4)
    assert res["all"]["cost"] == int(g.cost.sum())
    assert all(r["cost"] >= res["all"]["cost"] for r in res.values())
    assert all(r["peak"] <= res["all"]["peak"] for r in res.values())
