"""GPU parity of randomized two-phase rounding (R1):
the CUDA path against the oracle's Philox-driven rounding, bit-exact."""
import numpy as np
import pytest

from oracle import Instance, best_per_budget, evaluate, evaluate_randomized, masks_u64
from oracle.randomized import round_S_randomized
from workloads import budgets as B
from workloads import graphs as G
from workloads.sstar import dense_to_blk, dense_to_tri4, from_binary, gen_sstar

pytestmark = pytest.mark.gpu
KEY_NONE = (1 << 63) - 1


def run_rand(g, x_dense, samples, seed, budgets=None, layout="dense", masks=False, index_base=0, total=None):
    import torch
    import paper_1910_02653_b200 as cm
    dev = torch.device("cuda:0")
    graph = cm.Graph.from_workload(g)
    src = {"dense": lambda x: x, "tri4": dense_to_tri4, "blk": dense_to_blk}[layout](x_dense)
    x = torch.from_numpy(np.ascontiguousarray(src)).to(dev)
    bu = None if budgets is None else torch.tensor(np.asarray(budgets, np.int64), device=dev)
    out = cm.round_and_evaluate(graph, x, None, bu, layout=layout, masks=masks, samples=samples, seed=seed,
                                index_base=index_base, total_candidates=total,
                                ld=x_dense.shape[2] if layout == "dense" else None)
    torch.cuda.synchronize()
    res = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}
    graph.close()
    return res


def check(g, x, samples, seed, budgets=None, layout="dense", masks=False, index_base=0, total=None):
    res = run_rand(g, x, samples, seed, budgets, layout, masks, index_base, total)
    inst = Instance.from_graph(g)
    s_base = index_base // samples
    peaks, costs = [], []
    for s in range(x.shape[0]):
        for j in range(samples):
            c = s * samples + j
            o = evaluate_randomized(inst, x[s], s_base + s, j, seed, keep=masks)
            assert (res["peak"][c], res["cost"][c]) == (o["peak"], o["cost"]), (s, j)
            if masks:
                assert np.array_equal(res["s_mask"][c].view(np.uint64), masks_u64(inst, o["S"])), (s, j)
                assert np.array_equal(res["r_mask"][c].view(np.uint64), masks_u64(inst, o["R"])), (s, j)
            peaks.append(o["peak"])
            costs.append(o["cost"])
    if budgets is not None:
        want = best_per_budget(peaks, costs, budgets, index_base)
        bits = res["idx_bits"]
        for b, key in enumerate(res["best_key"]):
            if want[b][0] < 0:
                assert key == KEY_NONE
            else:
                assert (int(key) >> bits, int(key) & ((1 << bits) - 1) if bits else 0) == (want[b][1], want[b][0])
    return res


@pytest.mark.parametrize("layout", ["dense", "tri4", "blk"])
@pytest.mark.parametrize("samples", [1, 3, 4, 6])
def test_small_randomized(layout, samples):
    """samples <= 4: the fused kernel (one Philox block per element gives four samples);
    6: the two-kernel pipeline with two rounding passes."""
    g = G.random_training(20, 0.1, samples)
    x = gen_sstar(g, "mix", 21, 0, 5)
    check(g, x, samples, 0x1234_5678_9ABC_DEF0 + samples, B.geometric_grid(g, 5), layout=layout, masks=True)


@pytest.mark.parametrize("n", [2, 33, 65, 130])
def test_word_boundaries_randomized(n):
    g = G.random_dag(n, 0.05, n)
    x = gen_sstar(g, "g2", 3, 0, 3)
    check(g, x, 4, 77, [B.p_floor(g), B.p_live(g)], masks=True)


def test_index_base_sets_the_counter():
    """The global S* index (index_base / samples + s) is part of the Philox counter."""
    g = G.vgg16()
    x = gen_sstar(g, "g1", 4, 0, 3)
    a = check(g, x, 2, 5, index_base=2 * 1000, total=10 ** 6)
    b = check(g, x, 2, 5)
    assert not (np.array_equal(a["peak"], b["peak"]) and np.array_equal(a["cost"], b["cost"]))


def test_binary_sstar_matches_deterministic():
    """Binary S*: randomized rounding must reproduce the deterministic path exactly."""
    import torch
    import paper_1910_02653_b200 as cm
    g = G.training_chain(12)
    rng = np.random.default_rng(5)
    x = np.stack([from_binary(np.tril(rng.random((g.n, g.n)) < 0.3, -1)) for _ in range(6)])
    res = run_rand(g, x, 3, 99)
    graph = cm.Graph.from_workload(g)
    det = cm.round_and_evaluate(graph, torch.from_numpy(x).cuda(), torch.tensor([0.5], device="cuda"))
    torch.cuda.synchronize()
    assert np.array_equal(res["peak"], np.repeat(det["peak"].cpu().numpy(), 3))
    assert np.array_equal(res["cost"], np.repeat(det["cost"].cpu().numpy(), 3))


def test_full_size_randomized_sampled():
    """ResNet-50 shape, device-generated G1 S*, 4 samples each (the fused kernel), sampled
    candidates against the oracle."""
    import torch
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    g = G.resnet50()
    N = 1500
    dg = DeviceGenerator(g, "g1", 31, layout="dense")
    buf = torch.empty(dg.shape(N), dtype=torch.float32, device="cuda")
    dg.fill(buf, 0)
    graph = cm.Graph.from_workload(g)
    out = cm.round_and_evaluate(graph, buf, None, torch.tensor(B.geometric_grid(g, 4), device="cuda"),
                                samples=4, seed=2024)
    torch.cuda.synchronize()
    assert cm.debug_last_launches() == 1
    peak, cost = out["peak"].cpu().numpy(), out["cost"].cpu().numpy()
    inst = Instance.from_graph(g)
    for s in [0, 777, N - 1]:
        x = gen_sstar(g, "g1", 31, s, 1)[0]
        for j in range(4):
            o = evaluate_randomized(inst, x, s, j, 2024)
            assert (peak[4 * s + j], cost[4 * s + j]) == (o["peak"], o["cost"]), (s, j)
