"""a8 in the reduce step through an NVLink multicast buffer (cm_mc_*, cm_eval_args
.best_key_mc): the fused kernel's keys go out as multimem.red.min to the multicast view; the
local replica must then hold exactly the keys of the atomic path and of the oracle
(best_per_budget, max_batch_per_budget).  One GPU: a multicast object with one device -- the
instruction and the mapping are the ones an N-GPU run uses; only the team size differs.
Skipped where the driver creates no multicast object (the single-GPU boxes of this run:
cuMulticastCreate -> CUDA_ERROR_INVALID_VALUE for every handle type, size and team size,
profiles/r2aq_nvls_probe.json).  The epilogue's code path itself is exercised on a unicast
address below (multimem.red compiles to REDG.E.MIN.S64.STRONG.SYS: on plain memory it is the
atomic MIN -- a diagnostic of the kernel wiring, not of NVLS)."""
import numpy as np
import pytest

from oracle import Instance, best_per_budget, evaluate
from oracle.max_batch import max_batch_per_budget
from workloads import budgets as B
from workloads import graphs as G
from workloads.budgets import eq13_cost_limit
from workloads.sstar import dense_to_blk, gen_sstar

pytestmark = pytest.mark.gpu

KEY_NONE = (1 << 63) - 1


@pytest.fixture
def env_var():
    """Set library tuning variables for one test (read by the library at every call)."""
    import os
    saved = {}

    def setter(**kv):
        for k, v in kv.items():
            saved.setdefault(k, os.environ.get(k))
            os.environ[k] = str(v)
    yield setter
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _supported():
    import paper_1910_02653_b200 as cm
    return bool(cm._lib.cm_mc_supported())


@pytest.mark.parametrize("fused", ["1", "0"])
def test_multicast_keys_equal_atomics_and_oracle(env_var, fused):
    import torch
    import paper_1910_02653_b200 as cm
    from paper_1910_02653_b200.dist import MulticastKeys, decode_keys
    if not _supported():
        pytest.skip("no NVLink multicast on this device")
    env_var(CM_FUSED=fused)
    g = G.random_training(40, 0.12, 5)
    n_s = 70
    x = np.stack([gen_sstar(g, "mix", 11, s, 1)[0] for s in range(n_s)])
    budgets = list(B.geometric_grid(g, 8))
    limit = eq13_cost_limit(g)
    dev = torch.device("cuda:0")
    graph = cm.Graph.from_workload(g)
    xs = torch.from_numpy(np.ascontiguousarray(dense_to_blk(x, upper=np.nan))).to(dev)
    th = torch.tensor([0.5, 0.35], dtype=torch.float32, device=dev)
    bu = torch.tensor(np.asarray(budgets, np.int64), device=dev)
    try:
        mk = MulticastKeys(len(budgets))
        mb = MulticastKeys(len(budgets))
    except cm.CMError as ex:
        graph.close()
        pytest.skip(f"no multicast object on this box: {ex}")
    try:
        mk.reset()
        mb.reset()
        torch.cuda.synchronize()
        total = 3 * n_s * 2
        out = cm.round_and_evaluate(graph, xs, th, bu, layout="blk", index_base=2 * n_s, total_candidates=total,
                                    best_key=mk.local, best_key_mc=mk.mc, cost_limit=limit,
                                    best_batch_key=mb.local, best_batch_key_mc=mb.mc)
        ref = cm.round_and_evaluate(graph, xs, th, bu, layout="blk", index_base=2 * n_s, total_candidates=total,
                                    cost_limit=limit)
        torch.cuda.synchronize()
        assert mk.local.tolist() == ref["best_key"].tolist()
        assert mb.local.tolist() == ref["best_batch_key"].tolist()
        inst = Instance.from_graph(g)
        outs = [evaluate(inst, x[s], t) for s in range(n_s) for t in (0.5, 0.35)]
        peaks, costs = [o["peak"] for o in outs], [o["cost"] for o in outs]
        want = best_per_budget(peaks, costs, budgets, 2 * n_s)
        got = decode_keys(mk.local, out["idx_bits"])
        assert [(i, c) for (c, i) in got] == [(i, -1 if c is None else c) for (i, c) in want]
        wb = max_batch_per_budget(peaks, costs, budgets, g.ovh, limit, 2 * n_s)
        gb = [cm.decode_batch_key(int(k), out["idx_bits"]) for k in mb.local.tolist()]
        assert gb == [(b, i) for (b, i) in wb]
        # keys only decrease: a second call over the same candidates changes nothing
        cm.round_and_evaluate(graph, xs, th, bu, layout="blk", index_base=2 * n_s, total_candidates=total,
                              best_key=mk.local, best_key_mc=mk.mc)
        torch.cuda.synchronize()
        assert mk.local.tolist() == ref["best_key"].tolist()
    finally:
        mk.close()
        mb.close()
        graph.close()


def test_multicast_keys_reject_init_keys():
    import torch
    import paper_1910_02653_b200 as cm
    g = G.random_training(12, 0.2, 1)
    graph = cm.Graph.from_workload(g)
    dev = torch.device("cuda:0")
    x = torch.zeros((2, cm.sstar_floats(g.n, "blk")), dtype=torch.float32, device=dev)
    th = torch.tensor([0.5], dtype=torch.float32, device=dev)
    bu = torch.tensor([1 << 40], dtype=torch.int64, device=dev)
    key = torch.full((1,), KEY_NONE, dtype=torch.int64, device=dev)
    with pytest.raises(cm.CMError):
        cm.round_and_evaluate(graph, x, th, bu, layout="blk", best_key=key, best_key_mc=key.data_ptr(),
                              init_keys=True)
    graph.close()


@pytest.mark.parametrize("fused", ["1", "0"])
def test_multimem_epilogue_wiring_on_unicast_address(env_var, fused):
    """best_key_mc / best_batch_key_mc pointing at plain device buffers: the keys land there (and
    not in the filter buffers), equal to the atomic path's and the oracle's."""
    import torch
    import paper_1910_02653_b200 as cm
    env_var(CM_FUSED=fused)
    g = G.random_training(40, 0.12, 5)
    n_s = 70
    x = np.stack([gen_sstar(g, "mix", 11, s, 1)[0] for s in range(n_s)])
    budgets = list(B.geometric_grid(g, 8))
    limit = eq13_cost_limit(g)
    dev = torch.device("cuda:0")
    graph = cm.Graph.from_workload(g)
    xs = torch.from_numpy(np.ascontiguousarray(dense_to_blk(x, upper=np.nan))).to(dev)
    th = torch.tensor([0.5, 0.35], dtype=torch.float32, device=dev)
    bu = torch.tensor(np.asarray(budgets, np.int64), device=dev)
    filt = torch.full((len(budgets),), KEY_NONE, dtype=torch.int64, device=dev)
    bfilt = torch.full((len(budgets),), KEY_NONE, dtype=torch.int64, device=dev)
    dst = torch.full((len(budgets),), KEY_NONE, dtype=torch.int64, device=dev)
    bdst = torch.full((len(budgets),), KEY_NONE, dtype=torch.int64, device=dev)
    out = cm.round_and_evaluate(graph, xs, th, bu, layout="blk", best_key=filt, best_key_mc=dst.data_ptr(),
                                cost_limit=limit, best_batch_key=bfilt, best_batch_key_mc=bdst.data_ptr())
    ref = cm.round_and_evaluate(graph, xs, th, bu, layout="blk", cost_limit=limit)
    torch.cuda.synchronize()
    assert dst.tolist() == ref["best_key"].tolist()
    assert bdst.tolist() == ref["best_batch_key"].tolist()
    assert filt.tolist() == [KEY_NONE] * len(budgets) and bfilt.tolist() == [KEY_NONE] * len(budgets)
    inst = Instance.from_graph(g)
    outs = [evaluate(inst, x[s], t) for s in range(n_s) for t in (0.5, 0.35)]
    peaks, costs = [o["peak"] for o in outs], [o["cost"] for o in outs]
    want = best_per_budget(peaks, costs, budgets, 0)
    got = [cm.decode_key(int(k), out["idx_bits"]) for k in dst.tolist()]
    assert [(i, c) for (c, i) in got] == [(i, -1 if c is None else c) for (i, c) in want]
    graph.close()
