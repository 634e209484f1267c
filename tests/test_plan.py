"""Execution-plan emission in the library (cm_emit_plan, host code)
against the oracle's Alg. 1 and hoisted plans, statement by statement (CPU only)."""
import numpy as np
import pytest

from oracle import Instance, evaluate, generate_plan, hoisted_plan, masks_u64, simulate_plan
from workloads import graphs as G
from workloads.sstar import from_binary, gen_sstar


def to0(plan):
    """oracle statements (1-based) -> the ABI's (op, stage, node, reg), 0-based."""
    out = []
    for st in plan:
        if st[0] == "compute":
            out.append((0, st[1] - 1, st[2] - 1, st[3]))
        else:
            out.append((1, st[1] - 1, st[3] - 1, st[2]))
    return out


@pytest.mark.parametrize("trial", range(24))
def test_plan_matches_oracle(trial):
    import paper_1910_02653_b200 as cm
    rng = np.random.default_rng(100 + trial)
    g = G.random_dag(int(rng.integers(2, 14)), 0.3, trial) if trial % 2 else \
        G.random_training(int(rng.integers(2, 9)), 0.2, trial)
    x = from_binary(np.tril(rng.random((g.n, g.n)) < 0.3, -1)) if trial % 3 == 0 else gen_sstar(g, "mix", 7, trial, 1)[0]
    inst = Instance.from_graph(g)
    o = evaluate(inst, x, 0.5, keep=True)
    rr, ss = masks_u64(inst, o["R"]), masks_u64(inst, o["S"])
    ptr, idx = g.pred_csr()
    for hoist, ref in ((False, generate_plan(inst, o["R"], o["FREE"])),
                       (True, hoisted_plan(inst, o["R"], o["S"], o["FREE"]))):
        stmts, peak = cm.emit_plan(g.n, ptr, idx, g.mem, g.ovh, rr, ss, hoist=hoist)
        assert stmts == to0(ref)
        assert peak == simulate_plan(inst, ref, o["S"])[0]
        if not hoist:
            assert peak == o["peak"]


def test_plan_rejects_infeasible_masks():
    import paper_1910_02653_b200 as cm
    g = G.path(5)
    inst = Instance.from_graph(g)
    o = evaluate(inst, from_binary(np.zeros((5, 5), bool)), 0.5, keep=True)
    rr, ss = masks_u64(inst, o["R"]), masks_u64(inst, o["S"])
    rr[4, 0] &= ~np.uint64(1 << 2)          # stage 5 no longer recomputes v3, which v4 needs
    ptr, idx = g.pred_csr()
    with pytest.raises(cm.CMError):
        cm.emit_plan(g.n, ptr, idx, g.mem, g.ovh, rr, ss)
