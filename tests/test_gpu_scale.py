"""GPU parity at scale and the cross-GPU argmin (a8) on CUDA-produced keys.

- Each of bench.py's five configs at its exact bench launch (device-generated S* in the
  blocked layout bench.py times, and in the dense layout with 128-byte rows; bench's seed, fused persistent kernel, consecutive calls overlapped on two
  alternating output sets with in-kernel key init): >= 2 000 candidates per config checked
  against the CPU oracle -- the first 1 000, unit boundaries, the last unit and 1 000 random
  ones -- and every per-budget key against the call's own per-candidate outputs.  A second
  check compares ALL candidates of the fused launch with the two-kernel pipeline
  (CM_FUSED=0): a detector for ring hand-off races, not a parity claim.  The same for
  randomized rounding at bench.py --samples 1 / 4's launch.
- a8: the CUDA path over P contiguous index_base shards,
  MIN-reduced, equals the unsharded call and the oracle's best_per_budget (Alg. 2 +
  budget row; SURVEY invariant 9, shard invariance); the winners'
  R / S masks gathered from the shards equal the oracle's.  The same through a real
  world-size-2 process group (gloo; both ranks on cuda:0) and paper_1910_02653_b200.dist.
"""
import os
import socket

import numpy as np
import pytest

import bench
from tests.oracle_pool import boundary_sample, oracle_many
from workloads import budgets as B
from workloads import graphs as G

pytestmark = pytest.mark.gpu

KEY_NONE = (1 << 63) - 1
BENCH_SEED = 20250101


@pytest.fixture
def env_var():
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


def keys_of(peak, cost, budgets, bits, index_base=0):
    """The a7 keys a call must produce from its own per-candidate (peak, cost)."""
    out = []
    for b in budgets:
        feas = np.nonzero(peak <= b)[0]
        if len(feas) == 0:
            out.append(KEY_NONE)
            continue
        c = int(cost[feas].min())
        out.append((c << bits) | (index_base + int(feas[cost[feas] == c].min())))
    return out


def oracle_keys(peaks, costs, budgets, bits, index_base=0):
    from oracle import best_per_budget
    return [KEY_NONE if i < 0 else (c << bits) | i
            for (i, c) in best_per_budget(peaks, costs, budgets, index_base)]


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("layout,ring", [("blk", None), ("dense", None), ("blk", 256)])
@pytest.mark.parametrize("cfg", ["resnet50", "vgg16", "unet", "mobilenet", "fcn8"])
def test_bench_config_full_launch(cfg, layout, ring, env_var):
    """ring: CM_RING slots (None: the library's default, ~300 MB of slots -- every unit of a
    VGG16 call, so only the forced 256-slot ring makes its claim-8 producers wrap)."""
    import torch
    if ring is not None:
        if cfg not in ("vgg16", "unet"):
            pytest.skip("forced ring depth: small graphs only (the default already wraps at n >= 353)")
        env_var(CM_RING=ring)
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    g, fam, thetas, budgets, N = bench.build_workload(cfg)
    nt = len(thetas)
    dev = torch.device("cuda:0")
    ld = -(-g.n // 32) * 32 if layout == "dense" else None          # bench.py's dense rows: 128 bytes
    dg = DeviceGenerator(g, fam, BENCH_SEED, layout=layout, ld=ld)
    buf = torch.empty(dg.shape(N), dtype=torch.float32, device=dev)
    dg.fill(buf, 0)
    graph = cm.Graph.from_workload(g)
    th = torch.tensor(thetas, dtype=torch.float32, device=dev)
    bu = torch.tensor(budgets, dtype=torch.int64, device=dev)
    sets = [{k: torch.zeros(m, dtype=torch.int64, device=dev) for k, m in
             (("peak", N * nt), ("cost", N * nt), ("key", len(budgets)))} for _ in range(2)]
    torch.cuda.synchronize()
    for step in range(3):                                           # bench's step, 3 calls back to back
        o = sets[step % 2]
        out = cm.round_and_evaluate(graph, buf, th, bu, best_key=o["key"], peak=o["peak"], cost=o["cost"],
                                    index_base=0, total_candidates=N * nt, init_keys=True, overlap=True,
                                    layout=layout)
        assert cm.debug_last_launches() == 1                        # the fused persistent kernel
    torch.cuda.synchronize()
    bits = out["idx_bits"]
    got = [(o["peak"].cpu().numpy(), o["cost"].cpu().numpy(), o["key"].cpu().numpy()) for o in sets]
    # ring-race detector: every candidate of the fused launch equals the two-kernel pipeline
    env_var(CM_FUSED=0)
    ref = cm.round_and_evaluate(graph, buf, th, bu, total_candidates=N * nt, layout=layout)
    torch.cuda.synchronize()
    assert cm.debug_last_launches() >= 3
    env_var(CM_FUSED=1)
    rp, rc = ref["peak"].cpu().numpy(), ref["cost"].cpu().numpy()
    del buf, ref
    torch.cuda.empty_cache()
    for peak, cost, key in got:
        assert np.array_equal(peak, rp) and np.array_equal(cost, rc)
        assert list(key) == keys_of(peak, cost, budgets, bits)
    # >= 2 000 candidates against the oracle
    sample = boundary_sample(N)
    assert len(sample) >= 2000
    want = oracle_many(g, fam, BENCH_SEED, sample, thetas)
    bad = []
    for s in sample:
        for j in range(nt):
            c = s * nt + j
            w = want[s][j]
            for peak, cost, _ in got:
                if (int(peak[c]), int(cost[c])) != (w[0], w[1]):
                    bad.append((s, j, int(peak[c]), int(cost[c]), w[0], w[1]))
    assert not bad, bad[:10]
    graph.close()


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("thetas", [[0.2, 0.4, 0.5, 0.7], [0.5, 0.3]])
def test_bench_launch_multi_threshold(thetas, env_var):
    """bench.py --thetas launch (the fused instances with 2-4 thresholds run 12 scan warps,
    setmaxnreg-rebalanced, 4-quad Sn rings): ResNet-50, 125 000 device-generated G1 S*, blocked
    layout, three overlapped calls; >= 2 000 S* x N_theta against the oracle, every candidate
    against the two-kernel pipeline, keys against the call's own outputs."""
    import torch
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    g, fam, _, budgets, N = bench.build_workload("resnet50")
    nt = len(thetas)
    dev = torch.device("cuda:0")
    dg = DeviceGenerator(g, fam, BENCH_SEED, layout="blk")
    buf = torch.empty(dg.shape(N), dtype=torch.float32, device=dev)
    dg.fill(buf, 0)
    graph = cm.Graph.from_workload(g)
    th = torch.tensor(thetas, dtype=torch.float32, device=dev)
    bu = torch.tensor(budgets, dtype=torch.int64, device=dev)
    nc = N * nt
    sets = [{k: torch.zeros(m, dtype=torch.int64, device=dev) for k, m in
             (("peak", nc), ("cost", nc), ("key", len(budgets)))} for _ in range(2)]
    torch.cuda.synchronize()
    for step in range(3):
        o = sets[step % 2]
        out = cm.round_and_evaluate(graph, buf, th, bu, best_key=o["key"], peak=o["peak"], cost=o["cost"],
                                    total_candidates=nc, init_keys=True, overlap=True, layout="blk")
        assert cm.debug_last_launches() == 1
    torch.cuda.synchronize()
    bits = out["idx_bits"]
    got = [(o["peak"].cpu().numpy(), o["cost"].cpu().numpy(), o["key"].cpu().numpy()) for o in sets]
    env_var(CM_FUSED=0)
    ref = cm.round_and_evaluate(graph, buf, th, bu, total_candidates=nc, layout="blk")
    torch.cuda.synchronize()
    env_var(CM_FUSED=1)
    rp, rc = ref["peak"].cpu().numpy(), ref["cost"].cpu().numpy()
    del buf, ref
    torch.cuda.empty_cache()
    for peak, cost, key in got:
        assert np.array_equal(peak, rp) and np.array_equal(cost, rc)
        assert list(key) == keys_of(peak, cost, budgets, bits)
    sample = boundary_sample(N)
    want = oracle_many(g, fam, BENCH_SEED, sample, thetas)
    bad = []
    for s in sample:
        for j in range(nt):
            c = s * nt + j
            w = want[s][j]
            for peak, cost, _ in got:
                if (int(peak[c]), int(cost[c])) != (w[0], w[1]):
                    bad.append((s, j, int(peak[c]), int(cost[c]), w[0], w[1]))
    assert not bad, bad[:10]
    graph.close()


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("samples,N", [(1, 125000), (4, 31250)])
def test_bench_launch_randomized(samples, N, env_var):
    """Randomized rounding (R1) at bench.py --samples K's launch: ResNet-50, device-
    generated G1 S* in the blocked layout, bench's seed (also the Philox key), three overlapped
    calls on two alternating output sets with in-kernel key init.  >= 2 000 S* (x K samples)
    against the oracle's evaluate_randomized; every candidate of the fused launch against the
    two-kernel pipeline (ring-race detector); keys against the call's own outputs."""
    import torch
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    g, fam, _, budgets, _ = bench.build_workload("resnet50")
    dev = torch.device("cuda:0")
    dg = DeviceGenerator(g, fam, BENCH_SEED, layout="blk")
    buf = torch.empty(dg.shape(N), dtype=torch.float32, device=dev)
    dg.fill(buf, 0)
    graph = cm.Graph.from_workload(g)
    bu = torch.tensor(budgets, dtype=torch.int64, device=dev)
    nc = N * samples
    sets = [{k: torch.zeros(m, dtype=torch.int64, device=dev) for k, m in
             (("peak", nc), ("cost", nc), ("key", len(budgets)))} for _ in range(2)]
    torch.cuda.synchronize()
    for step in range(3):
        o = sets[step % 2]
        out = cm.round_and_evaluate(graph, buf, None, bu, best_key=o["key"], peak=o["peak"], cost=o["cost"],
                                    total_candidates=nc, init_keys=True, overlap=True, layout="blk",
                                    samples=samples, seed=BENCH_SEED)
        assert cm.debug_last_launches() == 1
    torch.cuda.synchronize()
    bits = out["idx_bits"]
    got = [(o["peak"].cpu().numpy(), o["cost"].cpu().numpy(), o["key"].cpu().numpy()) for o in sets]
    env_var(CM_FUSED=0)
    ref = cm.round_and_evaluate(graph, buf, None, bu, total_candidates=nc, layout="blk", samples=samples,
                                seed=BENCH_SEED)
    torch.cuda.synchronize()
    env_var(CM_FUSED=1)
    rp, rc = ref["peak"].cpu().numpy(), ref["cost"].cpu().numpy()
    del buf, ref
    torch.cuda.empty_cache()
    for peak, cost, key in got:
        assert np.array_equal(peak, rp) and np.array_equal(cost, rc)
        assert list(key) == keys_of(peak, cost, budgets, bits)
    sample = boundary_sample(N)
    assert len(sample) >= 2000
    want = oracle_many(g, fam, BENCH_SEED, sample, samples=samples, rseed=BENCH_SEED)
    bad = []
    for s in sample:
        for j in range(samples):
            c = s * samples + j
            w = want[s][j]
            for peak, cost, _ in got:
                if (int(peak[c]), int(cost[c])) != (w[0], w[1]):
                    bad.append((s, j, int(peak[c]), int(cost[c]), w[0], w[1]))
    assert not bad, bad[:10]
    graph.close()


def _oracle_all(g, fam, seed, N, thetas):
    want = oracle_many(g, fam, seed, range(N), thetas)
    peaks = [want[s][j][0] for s in range(N) for j in range(len(thetas))]
    costs = [want[s][j][1] for s in range(N) for j in range(len(thetas))]
    return np.array(peaks, np.int64), np.array(costs, np.int64)


def _winner_masks_oracle(g, fam, seed, key, bits, nt, thetas):
    """Oracle R / S masks (the C-ABI's u64 row layout) of each budget's winner."""
    from oracle import Instance, evaluate, masks_u64
    from workloads.sstar import gen_sstar
    inst = Instance.from_graph(g)
    out = {}
    for b, k in enumerate(key):
        if k == KEY_NONE:
            continue
        idx = int(k) & ((1 << bits) - 1)
        s, j = divmod(idx, nt)
        o = evaluate(inst, gen_sstar(g, fam, seed, s, 1)[0], thetas[j], keep=True)
        out[b] = (masks_u64(inst, o["R"]), masks_u64(inst, o["S"]))
    return out


@pytest.mark.timeout(1800)
def test_virtual_shards_resnet50():
    """ResNet-50, 4 096 S* x 2 thresholds x 16 budgets, as P in {2, 3, 8} contiguous shards
    (dist.shard_range), one library call per shard with its global index_base: the MIN of
    the shards' keys equals the unsharded call and the oracle's best_per_budget over all
    8 192 candidates; the winners' masks gathered from the shards (dist.gather_winner_masks
    on each shard's GPU-written masks, summed) equal the oracle's."""
    import torch
    import paper_1910_02653_b200 as cm
    from paper_1910_02653_b200.dist import gather_winner_masks, shard_range
    from workloads.device_gen import DeviceGenerator
    g = G.resnet50()
    N, thetas, fam, seed = 4096, [0.5, 0.35], "g1", 4242
    nt = len(thetas)
    budgets = B.geometric_grid(g, 16)
    dev = torch.device("cuda:0")
    dg = DeviceGenerator(g, fam, seed, layout="dense", ld=384)
    buf = torch.empty(dg.shape(N), dtype=torch.float32, device=dev)
    dg.fill(buf, 0)
    graph = cm.Graph.from_workload(g)
    th = torch.tensor(thetas, dtype=torch.float32, device=dev)
    bu = torch.tensor(budgets, dtype=torch.int64, device=dev)
    total = N * nt
    full = cm.round_and_evaluate(graph, buf, th, bu, total_candidates=total)
    torch.cuda.synchronize()
    bits = full["idx_bits"]
    fkey = [int(k) for k in full["best_key"].cpu().numpy()]
    fpeak, fcost = full["peak"].cpu().numpy(), full["cost"].cpu().numpy()
    opeak, ocost = _oracle_all(g, fam, seed, N, thetas)
    assert np.array_equal(fpeak, opeak) and np.array_equal(fcost, ocost)
    okey = oracle_keys(list(opeak), list(ocost), budgets, bits)
    assert fkey == okey
    masks_want = _winner_masks_oracle(g, fam, seed, okey, bits, nt, thetas)
    assert len(masks_want) >= 2
    for P in (2, 3, 8):
        kmin = torch.full((len(budgets),), KEY_NONE, dtype=torch.int64, device=dev)
        shards = []
        for r in range(P):
            lo, hi = shard_range(N, r, P)
            o = cm.round_and_evaluate(graph, buf[lo:hi], th, bu, index_base=lo * nt, total_candidates=total,
                                      masks=True)
            torch.cuda.synchronize()
            assert np.array_equal(o["peak"].cpu().numpy(), fpeak[lo * nt:hi * nt])
            assert np.array_equal(o["cost"].cpu().numpy(), fcost[lo * nt:hi * nt])
            kmin = torch.minimum(kmin, o["best_key"])               # dist.global_best's MIN
            shards.append((lo, o["r_mask"], o["s_mask"]))
        assert [int(k) for k in kmin.cpu().numpy()] == okey, P
        gathered = sum(gather_winner_masks(kmin, bits, lo * nt, rm, sm) for (lo, rm, sm) in shards)
        gathered = gathered.cpu().numpy()
        for b in range(len(budgets)):
            if b in masks_want:
                r_want, s_want = masks_want[b]
                assert np.array_equal(gathered[b, 0].view(np.uint64), r_want), (P, b)
                assert np.array_equal(gathered[b, 1].view(np.uint64), s_want), (P, b)
            else:
                assert not gathered[b].any()
        del shards
    graph.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SHARD_N, SHARD_THETAS, SHARD_SEED = 700, [0.5, 0.4], 99


def _gloo_rank(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1910_02653_b200 as cm
        from paper_1910_02653_b200.dist import gather_winner_masks, global_best, shard_range
        from workloads.device_gen import DeviceGenerator
        g = G.resnet50()
        nt = len(SHARD_THETAS)
        dev = torch.device("cuda:0")
        lo, hi = shard_range(SHARD_N, rank, world)
        dg = DeviceGenerator(g, "g1", SHARD_SEED, layout="dense", ld=384)
        buf = torch.empty(dg.shape(hi - lo), dtype=torch.float32, device=dev)
        dg.fill(buf, lo)                                            # this rank's S* only
        graph = cm.Graph.from_workload(g)
        o = cm.round_and_evaluate(graph, buf, torch.tensor(SHARD_THETAS, device=dev),
                                  torch.tensor(B.geometric_grid(g, 16), device=dev),
                                  index_base=lo * nt, total_candidates=SHARD_N * nt, masks=True)
        torch.cuda.synchronize()
        key = o["best_key"].cpu()
        global_best(key)                                            # all-reduce MIN over the group
        masks = gather_winner_masks(key, o["idx_bits"], lo * nt, o["r_mask"].cpu(), o["s_mask"].cpu())
        if rank == 0:
            q.put((key.tolist(), masks.numpy(), o["idx_bits"]))
        graph.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(900)
def test_global_best_gloo_two_ranks_cuda_keys():
    """a8 through a real process group: two ranks on cuda:0, each running the CUDA path on its
    own device-generated shard with its global index_base; dist.global_best (all-reduce MIN)
    and dist.gather_winner_masks (all-reduce SUM) over gloo.  Result = the oracle's."""
    import torch.multiprocessing as mp
    g = G.resnet50()
    nt = len(SHARD_THETAS)
    budgets = B.geometric_grid(g, 16)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    keys, masks, bits = q.get(timeout=600)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    opeak, ocost = _oracle_all(g, "g1", SHARD_SEED, SHARD_N, SHARD_THETAS)
    okey = oracle_keys(list(opeak), list(ocost), budgets, bits)
    assert keys == okey
    want = _winner_masks_oracle(g, "g1", SHARD_SEED, okey, bits, nt, SHARD_THETAS)
    assert len(want) >= 2
    for b, (r_want, s_want) in want.items():
        assert np.array_equal(masks[b, 0].view(np.uint64), r_want), b
        assert np.array_equal(masks[b, 1].view(np.uint64), s_want), b
