"""GPU parity of back-to-back calls with CM_EVAL_OVERLAP | CM_EVAL_INIT_KEYS: each call may
start while the previous one drains (programmatic dependent launch, alternating workspace
halves whose control words the kernel clears on exit) and initialises its own keys.  Every
call's outputs must equal the oracle's, whatever ran before it on the stream."""
import os

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
    # every output allocated (and its key pre-filled with 0) before the first call, so nothing
    # but `before(i)` is enqueued between two calls
    res = [{k: torch.zeros(m, dtype=torch.int64, device=dev) for k, m in
            (("peak", 2 * Ns[i]), ("cost", 2 * Ns[i]), ("key", len(budgets)))} for i in range(n_calls)]
    torch.cuda.synchronize()
    for i in range(n_calls):
        if before:
            before(i)
        outs.append(cm.round_and_evaluate(graph, ins[i], th, bu, layout=layout, best_key=res[i]["key"],
                                          peak=res[i]["peak"], cost=res[i]["cost"],
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


@pytest.mark.timeout(600)
def test_overlap_randomized_and_max_batch():
    """Overlapped calls with randomized rounding (2 samples per S*) and the max-batch epilogue,
    keys and batch keys initialised in-kernel over pre-filled zeros (every output allocated
    before the first call): call 0 against the oracle (randomized rounding R1, A2-A7, Eq. 13),
    and every call equal to a serial call with caller-initialised keys."""
    import torch
    import paper_1910_02653_b200 as cm
    from oracle import max_batch_per_budget
    from tests.oracle_pool import oracle_many
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

    def outputs(overlap):
        fill = 0 if overlap else KEY_NONE
        return [{"peak": torch.zeros(500, dtype=torch.int64, device="cuda"),
                 "cost": torch.zeros(500, dtype=torch.int64, device="cuda"),
                 "best_key": torch.full((len(budgets),), fill, dtype=torch.int64, device="cuda"),
                 "best_batch_key": torch.full((len(budgets),), fill, dtype=torch.int64, device="cuda")}
                for _ in range(4)]

    def call(i, o, overlap):
        return cm.round_and_evaluate(graph, ins[i], None, bu, samples=2, seed=99, index_base=500 * i,
                                     total_candidates=2000, cost_limit=limit, init_keys=overlap,
                                     overlap=overlap, **o)
    oo = outputs(True)
    torch.cuda.synchronize()
    over = [call(i, oo[i], True) for i in range(4)]
    torch.cuda.synchronize()
    so = outputs(False)
    serial = []
    for i in range(4):
        serial.append(call(i, so[i], False))
        torch.cuda.synchronize()
    for a, b in zip(over, serial):
        for k in ("peak", "cost", "best_key", "best_batch_key"):
            assert torch.equal(a[k], b[k]), k
    assert any(int(k) != KEY_NONE for k in over[0]["best_batch_key"].cpu())
    # call 0 against the oracle: S* #s of generator seed 300, global S* index s (index_base 0)
    want = oracle_many(g, "g1", 300, range(250), samples=2, rseed=99)
    peaks = [want[s][j][0] for s in range(250) for j in range(2)]
    costs = [want[s][j][1] for s in range(250) for j in range(2)]
    assert list(over[0]["peak"].cpu().numpy()) == peaks and list(over[0]["cost"].cpu().numpy()) == costs
    bits = over[0]["idx_bits"]
    check_keys(over[0]["best_key"].cpu().numpy(), np.array(peaks), np.array(costs), budgets, bits, 0)
    mb = max_batch_per_budget(peaks, costs, budgets, g.ovh, limit, index_base=0)
    got = [cm.decode_batch_key(int(k), bits) for k in over[0]["best_batch_key"].cpu().numpy()]
    assert got == [(b, i) for (b, i) in mb]
    graph.close()


@pytest.mark.timeout(600)
@pytest.mark.skipif(os.environ.get("CM_UNDER_SANITIZER") == "1",
                    reason="compute-sanitizer serialises kernels: no overlap to observe")
def test_overlap_is_concurrent(env_var):
    """consecutive overlapped calls really run concurrently.  Four bench-size calls
    (ResNet-50, 125 000 S*) with every output allocated before the first one (nothing enqueued
    between calls); the CM_TRACE=2 per-CTA %globaltimer stamps show call i+1's first CTA
    starting before call i's last scan warp finished (at least 2 of the 3 pairs: a trace-buffer
    clear may fall between one pair); every call's keys equal the (oracle-checked, sampled)
    per-candidate outputs' argmin."""
    import torch
    import paper_1910_02653_b200 as cm
    from tests.oracle_pool import oracle_many
    from workloads.device_gen import DeviceGenerator
    env_var(CM_TRACE=2)
    g = G.resnet50()
    N = 125000
    dg = DeviceGenerator(g, "g1", 515, layout="dense", ld=384)
    x = torch.empty(dg.shape(N), dtype=torch.float32, device="cuda")
    dg.fill(x, 0)
    graph = cm.Graph.from_workload(g)
    budgets = B.geometric_grid(g, 16)
    th = torch.tensor([0.5], device="cuda")
    bu = torch.tensor(budgets, device="cuda")
    sets = [{"peak": torch.zeros(N, dtype=torch.int64, device="cuda"),
             "cost": torch.zeros(N, dtype=torch.int64, device="cuda")} for _ in range(2)]
    keys = [torch.zeros(len(budgets), dtype=torch.int64, device="cuda") for _ in range(4)]
    torch.cuda.synchronize()
    outs = [cm.round_and_evaluate(graph, x, th, bu, best_key=keys[i], init_keys=True, overlap=True, **sets[i % 2])
            for i in range(4)]
    torch.cuda.synchronize()
    tr = [cm.debug_cta_trace(back=3 - i) for i in range(4)]
    assert all(t.shape[0] == tr[0].shape[0] > 0 for t in tr)
    overlapped = [int(tr[i + 1][:, 0].min()) < int(tr[i][:, 3].max()) for i in range(3)]
    assert sum(overlapped) >= 2, [(int(tr[i + 1][:, 0].min()) - int(tr[i][:, 3].max())) for i in range(3)]
    bits = outs[0]["idx_bits"]
    p0, c0 = sets[0]["peak"].cpu().numpy(), sets[0]["cost"].cpu().numpy()
    p1, c1 = sets[1]["peak"].cpu().numpy(), sets[1]["cost"].cpu().numpy()
    assert np.array_equal(p0, p1) and np.array_equal(c0, c1)       # same input, both sets
    for k in keys:
        check_keys(k.cpu().numpy(), p0, c0, budgets, bits, 0)
    sample = [0, 31, 32, 1000, 62499, 62500, N - 33, N - 32, N - 1] + list(range(7, N, 4999))
    want = oracle_many(g, "g1", 515, sample)
    for s in sample:
        assert (int(p0[s]), int(c0[s])) == want[s][0][:2], s
    graph.close()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("path", ["fused", "pipeline"])
def test_stream_wait_call(env_var, path):
    """cm_stream_wait_call: a second stream that waits for call `seq` through the device-side
    completion word sees every output of the call final (a copy taken on it equals the result
    after a full synchronisation), with nothing enqueued on the calling stream; the numbers
    count calls per graph."""
    import torch
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    if path == "pipeline":
        env_var(CM_FUSED=0)
    g = G.resnet50()
    N = 60000
    dg = DeviceGenerator(g, "g1", 616, layout="dense", ld=384)
    x = torch.empty(dg.shape(N), dtype=torch.float32, device="cuda")
    dg.fill(x, 0)
    graph = cm.Graph.from_workload(g)
    budgets = B.geometric_grid(g, 16)
    th = torch.tensor([0.5], device="cuda")
    bu = torch.tensor(budgets, device="cuda")
    side = torch.cuda.Stream()
    assert cm.last_call_seq(graph) == 0
    for i in range(3):
        o = {"peak": torch.zeros(N, dtype=torch.int64, device="cuda"),
             "cost": torch.zeros(N, dtype=torch.int64, device="cuda"),
             "best_key": torch.zeros(len(budgets), dtype=torch.int64, device="cuda")}
        torch.cuda.synchronize()
        cm.round_and_evaluate(graph, x, th, bu, init_keys=True, overlap=(path == "fused"), **o)
        seq = cm.last_call_seq(graph)
        assert seq == i + 1
        cm.stream_wait_call(graph, seq, side.cuda_stream)
        with torch.cuda.stream(side):
            snap = {k: v.clone() for k, v in o.items()}
        torch.cuda.synchronize()
        for k in o:
            assert torch.equal(snap[k], o[k]), k
        assert int(o["best_key"].max()) > 0
    graph.close()
