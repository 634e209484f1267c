"""GPU parity of back-to-back calls with CM_EVAL_OVERLAP | CM_EVAL_INIT_KEYS: each call may
start while the previous one drains (programmatic dependent launch, alternating workspace
halves whose control words the kernel clears on exit) and initialises its own keys.  Every
call's outputs must equal the oracle's, whatever ran before it on the stream."""
import numpy as np
import pytest

from oracle import Instance, evaluate
from workloads import budgets as B
from workloads import graphs as G
from workloads.sstar import gen_sstar

pytestmark = pytest.mark.gpu

KEY_NONE = (1 << 63) - 1


@pytest.fixture
def env_var():
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


def check_keys(key, peak, cost, budgets, bits, index_base):
    """best_key against the call's own (oracle-checked) peaks and costs: (cost, idx) argmin."""
    for b, k in enumerate(key):
        feas = np.nonzero(peak <= budgets[b])[0]
        if len(feas) == 0:
            assert k == KEY_NONE
            continue
        c = cost[feas].min()
        assert (int(k) >> bits, int(k) & ((1 << bits) - 1)) == (c, index_base + feas[cost[feas] == c].min())


def run_chain(g, layout, n_calls, N, before=None):
    """n_calls overlapped calls, call i on its own S* batch (generator seed 100 + i, N[i] S*,
    or N for all) and its own outputs, keys pre-filled with 0 (a value INIT_KEYS must
    overwrite).  `before(i)` may enqueue other work between calls."""
    Ns = list(N) if isinstance(N, (list, tuple)) else [N] * n_calls
    import torch
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    dev = torch.device("cuda:0")
    graph = cm.Graph.from_workload(g)
    budgets = B.geometric_grid(g, 6)
    th = torch.tensor([0.5, 0.3], device=dev)
    bu = torch.tensor(budgets, device=dev)
    ins, outs = [], []
    for i in range(n_calls):
        dg = DeviceGenerator(g, "g1", 100 + i, layout=layout)
        x = torch.empty(dg.shape(Ns[i]), dtype=torch.float32, device=dev)
        dg.fill(x, 0)
        ins.append(x)
    torch.cuda.synchronize()
    for i in range(n_calls):
        if before:
            before(i)
        key = torch.zeros(len(budgets), dtype=torch.int64, device=dev)
        outs.append(cm.round_and_evaluate(graph, ins[i], th, bu, layout=layout, best_key=key,
                                          index_base=2000 * i, total_candidates=2000 * n_calls,
                                          init_keys=True, overlap=True))
    torch.cuda.synchronize()
    inst = Instance.from_graph(g)
    for i, out in enumerate(outs):
        N = Ns[i]
        peak, cost = out["peak"].cpu().numpy(), out["cost"].cpu().numpy()
        for s in sorted(v for v in {0, 31, 32, N // 2, N - 1} if v < N):
            x = gen_sstar(g, "g1", 100 + i, s, 1)[0]
            for j, t in enumerate([0.5, 0.3]):
                o = evaluate(inst, x, t)
                assert (peak[2 * s + j], cost[2 * s + j]) == (o["peak"], o["cost"]), (i, s, j)
        check_keys(out["best_key"].cpu().numpy(), peak, cost, budgets, out["idx_bits"], 2000 * i)
    graph.close()
    return outs


@pytest.mark.timeout(240)
@pytest.mark.parametrize("ring", [768, 3])
@pytest.mark.parametrize("layout", ["dense", "tri4"])
def test_overlapped_calls(env_var, layout, ring):
    """Six overlapped fused calls on ResNet-50 (ring 3: every slot of both halves reused)."""
    import paper_1910_02653_b200 as cm
    env_var(CM_RING=ring)
    run_chain(G.resnet50(), layout, 6, 400)
    assert cm.debug_last_launches() == 1


@pytest.mark.timeout(240)
def test_overlap_after_other_paths(env_var):
    """Overlapped calls interleaved with two-kernel-pipeline calls (which overwrite the
    workspace halves' control words: the next fused call must clear them again) and with
    an unrelated kernel between two calls."""
    import os
    import torch
    import paper_1910_02653_b200 as cm
    scratch = torch.zeros(1 << 20, device="cuda")

    def before(i):
        os.environ["CM_FUSED"] = "0" if i in (1, 2) else "1"
        if i == 4:
            scratch.add_(1.0)
    env_var(CM_FUSED=1)
    run_chain(G.vgg16(), "dense", 6, 300, before)
    assert cm.debug_last_launches() == 1


@pytest.mark.timeout(240)
def test_overlap_ring_sizes_change():
    """Batches of 2 to 1000 S* (rings of 1 to 32 slots): a half's previous call had a smaller
    ring, so its ring data lies where the next call's control words go (they must be cleared)."""
    run_chain(G.resnet50(), "dense", 8, [40, 60, 1000, 700, 2, 33, 900, 64])


@pytest.mark.parametrize("kernel", ["fused", "pipeline", "v1"])
def test_init_keys_all_paths(env_var, kernel):
    """CM_EVAL_INIT_KEYS on every launch path, including an empty batch."""
    import torch
    import paper_1910_02653_b200 as cm
    if kernel == "pipeline":
        env_var(CM_FUSED=0)
    elif kernel == "v1":
        env_var(CM_KERNEL="v1")
    g = G.unet()
    x = gen_sstar(g, "mix", 5, 0, 40)
    graph = cm.Graph.from_workload(g)
    budgets = B.geometric_grid(g, 5)
    th = torch.tensor([0.5, 0.25], device="cuda")
    bu = torch.tensor(budgets, device="cuda")
    key = torch.zeros(len(budgets), dtype=torch.int64, device="cuda")
    out = cm.round_and_evaluate(graph, torch.from_numpy(x).cuda(), th, bu, best_key=key, init_keys=True)
    torch.cuda.synchronize()
    inst = Instance.from_graph(g)
    want = [evaluate(inst, x[s], t) for s in range(40) for t in (0.5, 0.25)]
    peak, cost = out["peak"].cpu().numpy(), out["cost"].cpu().numpy()
    assert list(peak) == [o["peak"] for o in want] and list(cost) == [o["cost"] for o in want]
    check_keys(key.cpu().numpy(), peak, cost, budgets, out["idx_bits"], 0)
    key.zero_()
    cm.round_and_evaluate(graph, torch.from_numpy(x[:0]).cuda(), th, bu, best_key=key, init_keys=True,
                          peak=out["peak"], cost=out["cost"])
    torch.cuda.synchronize()
    assert (key.cpu().numpy() == KEY_NONE).all()
    graph.close()


@pytest.mark.timeout(240)
def test_overlap_randomized_and_max_batch():
    """Overlapped calls with randomized rounding (2 samples per S*) and the max-batch epilogue,
    keys and batch keys initialised in-kernel over pre-filled zeros, equal to serial calls with
    caller-initialised keys (the serial path is checked against the oracle elsewhere)."""
    import torch
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    g = G.resnet50()
    budgets = B.geometric_grid(g, 6)
    bu = torch.tensor(budgets, device="cuda")
    limit = 1 << 62                              # every candidate competes (Eq. 13's limit is the caller's)
    graph = cm.Graph.from_workload(g)
    ins = []
    for i in range(4):
        dg = DeviceGenerator(g, "g1", 300 + i, layout="dense")
        x = torch.empty(dg.shape(250), dtype=torch.float32, device="cuda")
        dg.fill(x, 0)
        ins.append(x)

    def call(i, overlap):
        z = (lambda: torch.zeros(len(budgets), dtype=torch.int64, device="cuda")) if overlap else \
            (lambda: torch.full((len(budgets),), KEY_NONE, dtype=torch.int64, device="cuda"))
        return cm.round_and_evaluate(graph, ins[i], None, bu, samples=2, seed=99, index_base=500 * i,
                                     total_candidates=2000, best_key=z(), best_batch_key=z(),
                                     cost_limit=limit, init_keys=overlap, overlap=overlap)
    over = [call(i, True) for i in range(4)]
    torch.cuda.synchronize()
    serial = []
    for i in range(4):
        serial.append(call(i, False))
        torch.cuda.synchronize()
    for a, b in zip(over, serial):
        for k in ("peak", "cost", "best_key", "best_batch_key"):
            assert torch.equal(a[k], b[k]), k
    assert any(int(k) != KEY_NONE for k in over[0]["best_batch_key"].cpu())
    graph.close()
