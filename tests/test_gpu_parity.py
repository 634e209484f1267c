"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element on the same seeded inputs.  Integer outputs must be bit-exact."""
import numpy as np
import pytest

from oracle import Instance, best_per_budget, evaluate, masks_u64
from workloads import budgets as B
from workloads import graphs as G
from workloads.sstar import dense_to_blk, dense_to_tri4, from_binary, gen_sstar, roundup4

pytestmark = pytest.mark.gpu

KEY_NONE = (1 << 63) - 1
# dense: K1 reads 32x32 blocks by tensor-map TMA; tri4: by tile::gather4 (per-row 1-D bulk copies
# for a batch's last S*); blk (CM_LAYOUT_BLK): one 1-D bulk copy per block
LAYOUTS = ["dense", "tri4", "blk"]


def gpu_run(g, sstar, thetas, budgets=None, layout="dense", masks=False, index_base=0,
            total=None, ld=None):
    import torch
    import paper_1910_02653_b200 as cm
    dev = torch.device("cuda:0")
    graph = cm.Graph.from_workload(g)
    x = torch.from_numpy(np.ascontiguousarray(sstar)).to(dev)
    th = torch.tensor(np.asarray(thetas, np.float32), device=dev)
    bu = None if budgets is None else torch.tensor(np.asarray(budgets, np.int64), device=dev)
    out = cm.round_and_evaluate(graph, x, th, bu, layout=layout, masks=masks, index_base=index_base,
                                total_candidates=total, ld=ld)
    torch.cuda.synchronize()
    res = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}
    graph.close()
    return res


def oracle_run(g, sstar_dense, thetas, keep=False):
    inst = Instance.from_graph(g)
    outs = []
    for s in range(sstar_dense.shape[0]):
        for th in thetas:
            outs.append(evaluate(inst, sstar_dense[s], th, keep=keep))
    return inst, outs


def compare(g, sstar_dense, thetas, budgets=None, masks=False, layout="dense", index_base=0,
            total=None):
    src = {"dense": lambda x: x, "tri4": dense_to_tri4, "blk": lambda x: dense_to_blk(x, upper=np.nan)}[layout](sstar_dense)
    res = gpu_run(g, src, thetas, budgets, layout=layout, masks=masks, index_base=index_base,
                  total=total, ld=sstar_dense.shape[2] if layout == "dense" else None)
    inst, outs = oracle_run(g, sstar_dense, thetas, keep=masks)
    peaks = [o["peak"] for o in outs]
    costs = [o["cost"] for o in outs]
    assert list(res["peak"]) == peaks
    assert list(res["cost"]) == costs
    if masks:
        for c, o in enumerate(outs):
            assert np.array_equal(res["r_mask"][c].view(np.uint64), masks_u64(inst, o["R"])), c
            assert np.array_equal(res["s_mask"][c].view(np.uint64), masks_u64(inst, o["S"])), c
    if budgets is not None:
        want = best_per_budget(peaks, costs, budgets, index_base)
        bits = res["idx_bits"]
        for b, key in enumerate(res["best_key"]):
            if want[b][0] < 0:
                assert key == KEY_NONE
            else:
                assert (int(key) >> bits, int(key) & ((1 << bits) - 1) if bits else 0) == \
                    (want[b][1], want[b][0])
    return res, outs


@pytest.mark.parametrize("layout", LAYOUTS)
def test_config1_path8(layout):
    """BASELINE config 1: path n=8, unit C/M, 64 S* x 4 thresholds x 3 budgets."""
    g = G.path(8)
    x = gen_sstar(g, "mix", 1, 0, 64)
    compare(g, x, [0.3, 0.4, 0.5, 0.6], [2, 4, 8], masks=True, layout=layout)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13])
@pytest.mark.parametrize("fam", ["g1", "g2"])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_small_random(n, fam, layout):
    g = G.random_dag(n, 0.4, 10 + n)
    x = gen_sstar(g, fam, 3, 0, 8)
    compare(g, x, [0.5, 0.2], [g.ovh + 5, g.ovh + 20, 10 ** 9], masks=True, layout=layout)


@pytest.mark.parametrize("n", [31, 32, 33, 63, 64, 65, 95, 96, 97, 127, 128, 129, 191, 257])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_word_boundaries(n, layout):
    g = G.random_dag(n, 0.05, n)
    x = gen_sstar(g, "g1" if n % 2 else "g2", 5, 0, 3)
    compare(g, x, [0.5, 0.8], [B.p_floor(g), B.p_live(g)], masks=True, layout=layout)


@pytest.mark.parametrize("L", [15, 16, 17, 31, 32, 33, 48])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_training_random(L, layout):
    g = G.random_training(L, 0.05, L)
    x = gen_sstar(g, "mix", 7, 0, 4)
    compare(g, x, [0.5], B.geometric_grid(g, 5), masks=True, layout=layout)


@pytest.mark.parametrize("name", ["vgg16", "resnet50", "unet", "mobilenet", "fcn8"])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_paper_shaped(name, layout):
    g = G.NETWORKS[name]()
    if name == "unet":
        base = g
        g = g.scaled(5)
        budgets = B.unet_grid(base)
    else:
        budgets = B.geometric_grid(g, 16)
    x = gen_sstar(g, "mix", 11, 100, 3)
    compare(g, x, [0.5, 0.35], budgets, masks=(name == "resnet50"), layout=layout)


def test_layouts_and_ld():
    g = G.resnet50()
    x = gen_sstar(g, "g1", 2, 0, 3)
    r1, _ = compare(g, x, [0.5], layout="tri4")
    wide = gen_sstar(g, "g1", 2, 0, 3, ld=roundup4(g.n) + 64, upper=np.nan)
    r2, _ = compare(g, wide, [0.5])
    assert np.array_equal(r1["peak"], r2["peak"]) and np.array_equal(r1["cost"], r2["cost"])


@pytest.mark.parametrize("layout", LAYOUTS)
def test_rounding_edge_values(layout):
    """Exact 0.5 ties, NaN, theta 0 and 1, garbage in the never-read upper triangle."""
    g = G.random_training(10, 0.2, 4)
    x = gen_sstar(g, "g2", 9, 0, 4, upper=np.nan)
    x[0][np.tril(np.ones_like(x[0], bool), -1)] = 0.5
    x[1][3, 1] = np.nan
    x[1][7, 2:5] = np.nan
    x[2] = np.where(np.tril(np.ones_like(x[2], bool), -1), np.float32(1.0), np.float32(7.0))
    compare(g, x, [0.5, 0.0, 1.0, np.nextafter(np.float32(0.5), np.float32(0))], masks=True, layout=layout)


@pytest.mark.parametrize("layout", LAYOUTS)
def test_rounding_ieee_corners(layout):
    """The packed-fp32 compare (sign of theta - x) against IEEE '>' on the corners:
    +-0 with theta = +-0, denormals next to a denormal / zero theta, +-inf, quiet and signalling
    NaNs of both signs, values one ulp either side of theta."""
    g = G.random_training(12, 0.2, 6)
    n = g.n
    bits = np.array([0x00000000, 0x80000000, 0x00000001, 0x80000001, 0x00000002, 0x7F800000, 0xFF800000,
                     0x7FC00000, 0xFFC00000, 0x7F800001, 0xFF800001, 0x3F000000, 0x3EFFFFFF, 0x3F000001,
                     0x3F800000, 0x00800000, 0x007FFFFF], np.uint32)
    vals = bits.view(np.float32)
    ld = roundup4(n)
    x = np.zeros((4, n, ld), np.float32)
    rng = np.random.default_rng(3)
    for s in range(4):
        x[s] = vals[rng.integers(0, len(vals), (n, ld))]
    thetas = np.array([0x00000000, 0x80000000, 0x00000001, 0x3F000000], np.uint32).view(np.float32)
    compare(g, x, list(thetas), masks=True, layout=layout)


def test_binary_patterns_closed_forms():
    from tests.oracle_helpers import S_all, S_chen, S_liveness, S_zero
    L = 16
    g = G.training_chain(L)
    pats = [S_zero(g.n), S_all(g.n), S_liveness(g), S_chen(L, [4, 8, 12])]
    x = np.stack([from_binary(S) for S in pats])
    res, _ = compare(g, x, [0.5])
    n = g.n
    assert list(res["cost"]) == [n * (n + 1) // 2, n, n, 46]
    assert list(res["peak"]) == [L + 2, n, L + 2, 9]


def test_index_base_and_total():
    g = G.vgg16()
    x = gen_sstar(g, "mix", 3, 0, 5)
    compare(g, x, [0.5, 0.6], B.geometric_grid(g, 4), index_base=1000, total=5000)


def test_empty_batch():
    import torch
    import paper_1910_02653_b200 as cm
    g = G.path(8)
    graph = cm.Graph.from_workload(g)
    x = torch.zeros((0, 8, 8), device="cuda")
    out = cm.round_and_evaluate(graph, x, torch.tensor([0.5], device="cuda"),
                                torch.tensor([4], dtype=torch.int64, device="cuda"))
    torch.cuda.synchronize()
    assert out["peak"].numel() == 0 and int(out["best_key"][0]) == KEY_NONE


def test_error_paths_on_device():
    import torch
    import paper_1910_02653_b200 as cm
    g = G.path(8)
    graph = cm.Graph.from_workload(g)
    x = torch.zeros((2, 8, 8), device="cuda")
    th = torch.tensor([0.5], device="cuda")
    with pytest.raises(cm.CMError):
        cm.round_and_evaluate(graph, x, th, ld=6)                   # ld < n
    with pytest.raises(cm.CMError):
        cm.round_and_evaluate(graph, x, th, ld=8, stride=60)        # stride < n*ld
    with pytest.raises(cm.CMError):
        cm.round_and_evaluate(graph, x, th, index_base=5, total_candidates=3)
    big = G.path(64, cost=[1 << 40] * 64)
    gb = cm.Graph.from_workload(big)
    xb = torch.zeros((1, 64, 64), device="cuda")
    with pytest.raises(cm.CMError):                                 # key cannot hold cost bound
        cm.round_and_evaluate(gb, xb, th, total_candidates=1 << 20)


@pytest.mark.parametrize("layout", LAYOUTS)
def test_max_n(layout):
    """n = CM_NMAX = 1024 (32 words per row, 1024 threads)."""
    g = G.random_dag(1024, 0.0015, 77)
    x = gen_sstar(g, "g1", 3, 0, 2)
    compare(g, x, [0.5], [B.p_live(g)], layout=layout)


def test_device_generator_matches_host():
    import torch
    from workloads.device_gen import DeviceGenerator
    for name, fam, layout in [("resnet50", "mix", "dense"), ("unet", "g1", "tri4"), ("vgg16", "g2", "dense"),
                              ("resnet50", "g1", "blk"), ("fcn8", "mix", "blk")]:
        g = G.NETWORKS[name]()
        dg = DeviceGenerator(g, fam, 1234, layout=layout)
        buf = torch.empty(dg.shape(6), dtype=torch.float32, device="cuda")
        dg.fill(buf, s_begin=500, upper=0.0)
        host = gen_sstar(g, fam, 1234, 500, 6, layout=layout)
        assert np.array_equal(buf.cpu().numpy().view(np.uint32), host.view(np.uint32)), name


def test_full_size_sampled():
    """The bench launch configuration (ResNet-50, n=353, G1 LP-like S*, theta 0.5, 16 budgets,
    device-generated batch) checked on sampled candidates against the oracle, plus the
    per-budget keys against the GPU's own per-candidate outputs."""
    import torch
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    g = G.resnet50()
    N = 8192
    dg = DeviceGenerator(g, "g1", 2024, layout="tri4")
    buf = torch.empty(dg.shape(N), dtype=torch.float32, device="cuda")
    dg.fill(buf, 0)
    graph = cm.Graph.from_workload(g)
    budgets = B.geometric_grid(g, 16)
    bu = torch.tensor(budgets, device="cuda")
    th = torch.tensor([0.5], device="cuda")
    out = cm.round_and_evaluate(graph, buf, th, bu, layout="tri4")
    torch.cuda.synchronize()
    peak = out["peak"].cpu().numpy()
    cost = out["cost"].cpu().numpy()
    inst = Instance.from_graph(g)
    rng = np.random.default_rng(0)
    sample = sorted(set(rng.integers(0, N, 20).tolist()) | {0, N - 1})
    for s in sample:
        x = gen_sstar(g, "g1", 2024, s, 1)[0]
        o = evaluate(inst, x, 0.5)
        assert (peak[s], cost[s]) == (o["peak"], o["cost"]), s
    bits = out["idx_bits"]
    for b, key in enumerate(out["best_key"].cpu().numpy()):
        feas = np.nonzero(peak <= budgets[b])[0]
        if len(feas) == 0:
            assert key == KEY_NONE
            continue
        c = cost[feas].min()
        idx = feas[cost[feas] == c].min()
        assert (int(key) >> bits, int(key) & ((1 << bits) - 1)) == (c, idx)
    # the winner of the loosest budget re-checked by the oracle
    wi = int(out["best_key"][-1].item()) & ((1 << bits) - 1)
    o = evaluate(inst, gen_sstar(g, "g1", 2024, wi, 1)[0], 0.5)
    assert (o["peak"], o["cost"]) == (peak[wi], cost[wi])


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_int64_state_path(seed, layout):
    """M values too large for the int32 scan state (sum M / gcd >= 2^30): int64 kernels."""
    g = G.random_training(20, 0.1, seed)
    g.mem = g.mem * (1 << 35) + np.arange(g.n, dtype=np.int64) * 7 + 3    # gcd 1, huge sums
    x = gen_sstar(g, "mix", 4, 0, 6)
    compare(g, x, [0.5, 0.7], [B.p_floor(g), B.p_live(g)], masks=True, layout=layout)


def test_scaled_int32_path():
    """All M share a large common factor: the scan runs in units of gcd(M) exactly."""
    g = G.resnet50()
    g.mem = g.mem * 1000                                   # sum M >> 2^31, sum M / gcd small
    x = gen_sstar(g, "g1", 8, 0, 3)
    compare(g, x, [0.5], B.geometric_grid(g, 8))


@pytest.mark.parametrize("layout", LAYOUTS)
def test_many_thresholds(layout):
    """Six thresholds: two K1 passes per S* (4 + 2 thresholds)."""
    g = G.random_training(24, 0.1, 5)
    x = gen_sstar(g, "mix", 12, 0, 5)
    compare(g, x, [0.5, 0.1, 0.9, 0.3, 0.7, 0.45], B.geometric_grid(g, 4), masks=True, layout=layout)


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


@pytest.mark.timeout(240)
@pytest.mark.parametrize("win", [0, 16])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_fused_ring_wraparound(env_var, layout, win):
    """Fused path with a 3-slot ring: 1000 S* = 32 units, every slot reused ~10 times
    (producer / consumer hand-off, slot release after the in-kernel reduce); with ticket
    windows requested (clamped to R / 2 so the hand-off cannot deadlock)."""
    import torch
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    env_var(CM_RING=3, CM_WIN=win)
    g = G.resnet50()
    N = 1000
    dg = DeviceGenerator(g, "g1", 77, layout=layout)
    buf = torch.empty(dg.shape(N), dtype=torch.float32, device="cuda")
    dg.fill(buf, 0)
    graph = cm.Graph.from_workload(g)
    budgets = B.geometric_grid(g, 6)
    th = torch.tensor([0.5, 0.3], device="cuda")
    out = cm.round_and_evaluate(graph, buf, th, torch.tensor(budgets, device="cuda"), layout=layout)
    torch.cuda.synchronize()
    assert cm.debug_last_launches() == 1                           # the fused kernel ran
    peak, cost = out["peak"].cpu().numpy(), out["cost"].cpu().numpy()
    inst = Instance.from_graph(g)
    for s in [0, 31, 32, 500, 777, N - 1]:
        x = gen_sstar(g, "g1", 77, s, 1)[0]
        for j, t in enumerate([0.5, 0.3]):
            o = evaluate(inst, x, t)
            assert (peak[2 * s + j], cost[2 * s + j]) == (o["peak"], o["cost"]), (s, j)
    bits = out["idx_bits"]
    for b, key in enumerate(out["best_key"].cpu().numpy()):
        feas = np.nonzero(peak <= budgets[b])[0]
        if len(feas) == 0:
            assert key == KEY_NONE
            continue
        c = cost[feas].min()
        assert (int(key) >> bits, int(key) & ((1 << bits) - 1)) == (c, feas[cost[feas] == c].min())


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("name", ["vgg16", "resnet50", "fcn8"])
def test_two_kernel_pipeline(env_var, name, layout):
    """The two-kernel chunked pipeline (used for > 4 thresholds, the int64 state, or without
    TMEM) forced on the paper-shaped graphs, with a workspace small enough for several chunks."""
    import paper_1910_02653_b200 as cm
    env_var(CM_FUSED=0, CM_WS_MB=1)                                 # minimum workspace: 1024 candidates
    g = G.NETWORKS[name]()
    x = gen_sstar(g, "mix", 13, 40, 700 if name == "vgg16" else 70)   # vgg16: 2 chunks
    compare(g, x, [0.5, 0.25], B.geometric_grid(g, 8), layout=layout)
    assert cm.debug_last_launches() >= 3


@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("name", ["resnet50", "training"])
def test_max_batch_epilogue(env_var, name, fused):
    """Max-batch epilogue (Eq. 13, NEXT #4) against the oracle on the oracle's own peaks/costs,
    on the fused kernel and the two-kernel pipeline."""
    import torch
    import paper_1910_02653_b200 as cm
    from oracle import max_batch_per_budget
    env_var(CM_FUSED=fused)
    from tests.oracle_helpers import S_all, S_liveness
    g = G.resnet50() if name == "resnet50" else G.random_training(30, 0.1, 4)
    # LP-like S* plus two cheap binary schedules (keep-all, liveness: cost sum C <= Eq. 13's
    # limit) with different peaks, so the epilogue has real choices
    x = np.concatenate([gen_sstar(g, "g1", 17, 0, 38), from_binary(S_all(g.n))[None],
                        from_binary(S_liveness(g))[None]])
    budgets = [int(B.p_live(g) * f) for f in (0.5, 1, 2, 3.5, 8)]   # up to 8x the live peak
    limit = B.eq13_cost_limit(g)
    graph = cm.Graph.from_workload(g)
    thetas = [0.5, 0.3]
    out = cm.round_and_evaluate(graph, torch.from_numpy(x).cuda(), torch.tensor(thetas, device="cuda"),
                                torch.tensor(budgets, device="cuda"), cost_limit=limit, index_base=64,
                                total_candidates=64 + 80)
    torch.cuda.synchronize()
    inst, outs = oracle_run(g, x, thetas)
    peaks = [o["peak"] for o in outs]
    costs = [o["cost"] for o in outs]
    assert list(out["peak"].cpu().numpy()) == peaks and list(out["cost"].cpu().numpy()) == costs
    want = max_batch_per_budget(peaks, costs, budgets, g.ovh, limit, index_base=64)
    got = [cm.decode_batch_key(int(k), out["idx_bits"]) for k in out["best_batch_key"].cpu().numpy()]
    assert got == [(b, i) for (b, i) in want]
    assert any(b > 1 for b, _ in want)                              # a non-trivial instance


def test_plan_for_gpu_winners():
    """NEXT #3 end to end: the GPU picks the per-budget winners and writes their R / S masks;
    cm_emit_plan turns them into Alg. 1 plans (hoisted), equal to the oracle's."""
    import torch
    import paper_1910_02653_b200 as cm
    from oracle import hoisted_plan
    g = G.vgg16()
    x = gen_sstar(g, "g1", 23, 0, 24)
    budgets = B.geometric_grid(g, 4)
    graph = cm.Graph.from_workload(g)
    out = cm.round_and_evaluate(graph, torch.from_numpy(x).cuda(), torch.tensor([0.5], device="cuda"),
                                torch.tensor(budgets, device="cuda"), masks=True)
    torch.cuda.synchronize()
    inst = Instance.from_graph(g)
    ptr, idx = g.pred_csr()
    checked = 0
    for key in out["best_key"].cpu().numpy():
        c, i = cm.decode_key(int(key), out["idx_bits"])
        if i < 0:
            continue
        stmts, peak = cm.emit_plan(g.n, ptr, idx, g.mem, g.ovh, out["r_mask"][i].cpu().numpy(),
                                   out["s_mask"][i].cpu().numpy(), hoist=True)
        o = evaluate(inst, x[i], 0.5, keep=True)
        ref = hoisted_plan(inst, o["R"], o["S"], o["FREE"])
        assert len(stmts) == len(ref) and peak <= o["peak"] and c == o["cost"]
        assert [(s[0], s[1], s[2]) for s in stmts] == [
            ((0, t - 1, a - 1) if op == "compute" else (1, t - 1, b - 1)) for (op, t, a, b) in ref]
        checked += 1
    assert checked >= 2


@pytest.mark.parametrize("name", ["chain", "resnet50", "unet"])
def test_baseline_policies_on_device(name):
    """NEXT #2: every policy of Table 1's generalisations with a b-sweep, S written on the
    device from the checkpoint sets and evaluated in one batch, against the oracle."""
    import torch
    import paper_1910_02653_b200 as cm
    from oracle import S_from_K, evaluate_policy
    g = {"chain": lambda: G.training_chain(20), "resnet50": G.resnet50, "unet": G.unet}[name]()
    graph = cm.Graph.from_workload(g)
    fwd = int(g.mem[: g.L].sum())
    specs = [("all", 0), ("sqrt", 0), ("ap_sqrt", 0)] + \
            [(p, b) for p in ("greedy", "ap_greedy") for b in (fwd // 40, fwd // 12, fwd // 4)]
    budgets = B.geometric_grid(g, 6)
    out = cm.baseline_sweep(graph, g.L, specs, torch.tensor(budgets, device="cuda"))
    torch.cuda.synchronize()
    inst = Instance.from_graph(g)
    names = {"all": "all", "sqrt": "chen_sqrt", "greedy": "chen_greedy", "ap_sqrt": "ap_sqrt",
             "ap_greedy": "ap_greedy"}
    sstar = out["sstar"].cpu().numpy()
    peaks, costs = [], []
    for c, (p, b) in enumerate(specs):
        o = evaluate_policy(inst, g.L, names[p], b)
        S = S_from_K(inst, g.L, o["K"])[1:g.n + 1, 1:]
        assert np.array_equal(sstar[c][:, :g.n] > 0.5, S), (p, b)
        assert (int(out["peak"][c]), int(out["cost"][c])) == (o["peak"], o["cost"]), (p, b)
        peaks.append(o["peak"])
        costs.append(o["cost"])
    want = best_per_budget(peaks, costs, budgets)
    got = [cm.decode_key(int(k), out["idx_bits"]) for k in out["best_key"].cpu().numpy()]
    assert got == [((w[1], w[0]) if w[0] >= 0 else (-1, -1)) for w in want]


@pytest.mark.parametrize("layout", LAYOUTS)
def test_int32_state_near_limit(layout):
    """sum M / gcd(M) just below 2^31: still the int32 scan state (E <= sum M, every
    intermediate within [-sum M, sum M]); exact against the oracle."""
    g = G.random_training(24, 0.15, 8)
    rng = np.random.default_rng(8)
    w = rng.integers(1, 1000, g.n).astype(np.int64)
    g.mem = (w * ((2 ** 31 - 1) // int(w.sum()))) * 3           # gcd 3 (or a multiple), sum/gcd < 2^31
    assert int(g.mem.sum()) // 3 < 2 ** 31
    x = gen_sstar(g, "mix", 19, 0, 8)
    compare(g, x, [0.5, 0.2], [B.p_floor(g), B.p_live(g)], masks=True, layout=layout)


def test_bench_launch_configuration_sampled():
    """The exact launches bench.py times: ResNet-50 (n=353), 125 000 device-generated G1 S* in
    the dense layout with 128-byte rows (ld = 384), theta 0.5, 16 budgets, one fused launch per
    step, consecutive steps overlapped (CM_EVAL_OVERLAP | CM_EVAL_INIT_KEYS) on two alternating
    output sets whose keys start at 0; three steps, the last two checked: sampled candidates
    against the oracle, every per-budget key against the GPU's own per-candidate outputs."""
    import torch
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    g = G.resnet50()
    N = 125000
    dg = DeviceGenerator(g, "g1", 20250101, layout="dense", ld=384)
    buf = torch.empty(dg.shape(N), dtype=torch.float32, device="cuda")
    dg.fill(buf, 0)
    graph = cm.Graph.from_workload(g)
    budgets = B.geometric_grid(g, 16)
    th = torch.tensor([0.5], device="cuda")
    bu = torch.tensor(budgets, device="cuda")
    sets = [{k: torch.zeros(n, dtype=torch.int64, device="cuda") for k, n in
             (("peak", N), ("cost", N), ("key", len(budgets)))} for _ in range(2)]
    for step in range(3):
        o = sets[step % 2]                                         # keys start at 0 (allocation)
        out = cm.round_and_evaluate(graph, buf, th, bu, best_key=o["key"], peak=o["peak"], cost=o["cost"],
                                    init_keys=True, overlap=True)
        assert cm.debug_last_launches() == 1
    torch.cuda.synchronize()
    del buf
    inst = Instance.from_graph(g)
    rng = np.random.default_rng(7)
    samples = sorted(set(rng.integers(0, N, 14).tolist()) | {0, 31, 32, N - 1})
    want = {s: evaluate(inst, gen_sstar(g, "g1", 20250101, s, 1)[0], 0.5) for s in samples}
    bits = out["idx_bits"]
    for o in sets:
        peak, cost = o["peak"].cpu().numpy(), o["cost"].cpu().numpy()
        for s in samples:
            assert (peak[s], cost[s]) == (want[s]["peak"], want[s]["cost"]), s
        for b, key in enumerate(o["key"].cpu().numpy()):
            feas = np.nonzero(peak <= budgets[b])[0]
            if len(feas) == 0:
                assert key == KEY_NONE
                continue
            c = cost[feas].min()
            assert (int(key) >> bits, int(key) & ((1 << bits) - 1)) == (c, feas[cost[feas] == c].min())


@pytest.mark.timeout(240)
@pytest.mark.parametrize("ring", [1, 2])
def test_fused_tiny_ring_small_graph(env_var, ring):
    """VGG16 (producers claim 8 consecutive S* per ticket) through a 1- or 2-slot ring: every
    unit waits for its predecessor's release; 700 S* = 22 units, one partial."""
    import torch
    import paper_1910_02653_b200 as cm
    env_var(CM_RING=ring)
    g = G.vgg16()
    x = gen_sstar(g, "mix", 29, 0, 700)
    budgets = B.geometric_grid(g, 6)
    res, outs = compare(g, x, [0.5], budgets)
    assert cm.debug_last_launches() == 1


@pytest.mark.parametrize("name", ["random", "vgg16", "resnet50"])
def test_row_form_kernel(env_var, name):
    """The row-form fallback (one CTA per S*, used when the stage-sliced layout does not fit
    shared memory), forced with CM_KERNEL=v1."""
    import paper_1910_02653_b200 as cm
    env_var(CM_KERNEL="v1")
    g = {"random": lambda: G.random_training(18, 0.2, 3), "vgg16": G.vgg16, "resnet50": G.resnet50}[name]()
    x = gen_sstar(g, "mix", 31, 0, 6)
    compare(g, x, [0.5, 0.3], B.geometric_grid(g, 5), masks=(name != "resnet50"))
    assert cm.debug_last_launches() == 1
