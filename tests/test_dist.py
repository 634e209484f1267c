"""Multi-process (world size 2, gloo, CPU) tests of the cross-rank argmin (a8): contiguous
S* shards with global candidate indices, packed (cost << idx_bits | idx) keys, all-reduce
MIN.  The per-candidate results come from the CPU oracle; the reduction under test is
paper_1910_02653_b200.dist (no CUDA needed)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

KEY_NONE = (1 << 63) - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _keys_for(peaks, costs, budgets, index_base, idx_bits):
    keys = []
    for b in budgets:
        best = KEY_NONE
        for c, (p, q) in enumerate(zip(peaks, costs)):
            if p <= b:
                best = min(best, (q << idx_bits) | (index_base + c))
        keys.append(best)
    return keys


def _worker(rank, world, port, n_sstar, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import importlib.util
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        spec = importlib.util.spec_from_file_location("cm_dist", os.path.join(root, "paper_1910_02653_b200", "dist.py"))
        D = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(D)
        from oracle import Instance, evaluate
        from workloads import budgets as B
        from workloads import graphs as G
        from workloads.sstar import gen_sstar
        g = G.random_training(6, 0.2, 3)
        inst = Instance.from_graph(g)
        budgets = list(B.geometric_grid(g, 6))
        lo, hi = D.shard_range(n_sstar, rank, world)
        thetas = [0.5, 0.6]
        total = n_sstar * len(thetas)
        idx_bits = max(1, (total - 1).bit_length())
        peaks, costs = [], []
        for s in range(lo, hi):
            x = gen_sstar(g, "mix", 17, s, 1)[0]
            for th in thetas:
                o = evaluate(inst, x, th)
                peaks.append(o["peak"])
                costs.append(o["cost"])
        keys = torch.tensor(_keys_for(peaks, costs, budgets, lo * len(thetas), idx_bits), dtype=torch.int64)
        D.global_best(keys)
        if rank == 0:
            out_q.put((keys.tolist(), D.decode_keys(keys, idx_bits), idx_bits))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_sstar", [5, 8])
def test_global_best_two_ranks(n_sstar):
    from oracle import Instance, best_per_budget, evaluate
    from workloads import budgets as B
    from workloads import graphs as G
    from workloads.sstar import gen_sstar
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_sstar, q)) for r in range(2)]
    for p in procs:
        p.start()
    keys, decoded, idx_bits = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single-process reference over all candidates
    g = G.random_training(6, 0.2, 3)
    inst = Instance.from_graph(g)
    budgets = list(B.geometric_grid(g, 6))
    peaks, costs = [], []
    for s in range(n_sstar):
        x = gen_sstar(g, "mix", 17, s, 1)[0]
        for th in [0.5, 0.6]:
            o = evaluate(inst, x, th)
            peaks.append(o["peak"])
            costs.append(o["cost"])
    want = best_per_budget(peaks, costs, budgets)
    for (widx, wcost), (cost, idx) in zip(want, decoded):
        if widx < 0:
            assert (cost, idx) == (-1, -1)
        else:
            assert (cost, idx) == (wcost, widx)


def test_shard_ranges_cover():
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("cm_dist", os.path.join(root, "paper_1910_02653_b200", "dist.py"))
    D = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(D)
    for N in [0, 1, 7, 125000, 10 ** 6]:
        for P in [1, 2, 3, 8]:
            rs = [D.shard_range(N, r, P) for r in range(P)]
            assert rs[0][0] == 0 and rs[-1][1] == N
            assert all(rs[i][1] == rs[i + 1][0] for i in range(P - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def _mask_worker(rank, world, port, n_sstar, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import importlib.util
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        spec = importlib.util.spec_from_file_location("cm_dist", os.path.join(root, "paper_1910_02653_b200", "dist.py"))
        D = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(D)
        import numpy as np
        from oracle import Instance, evaluate, masks_u64
        from workloads import budgets as B
        from workloads import graphs as G
        from workloads.sstar import gen_sstar
        g = G.random_training(6, 0.2, 3)
        inst = Instance.from_graph(g)
        budgets = list(B.geometric_grid(g, 6))
        lo, hi = D.shard_range(n_sstar, rank, world)
        idx_bits = max(1, (n_sstar - 1).bit_length())
        peaks, costs, rm, sm = [], [], [], []
        for s in range(lo, hi):
            o = evaluate(inst, gen_sstar(g, "mix", 17, s, 1)[0], 0.5, keep=True)
            peaks.append(o["peak"])
            costs.append(o["cost"])
            rm.append(masks_u64(inst, o["R"]).view(np.int64))
            sm.append(masks_u64(inst, o["S"]).view(np.int64))
        keys = torch.tensor(_keys_for(peaks, costs, budgets, lo, idx_bits), dtype=torch.int64)
        D.global_best(keys)
        got = D.gather_winner_masks(keys, idx_bits, lo, torch.from_numpy(np.stack(rm)), torch.from_numpy(np.stack(sm)))
        out_q.put((rank, keys.tolist(), got.numpy()))
    finally:
        dist.destroy_process_group()


def test_winner_masks_two_ranks():
    """Every rank ends with the R / S masks of every budget's global winner."""
    import numpy as np
    from oracle import Instance, evaluate, masks_u64
    from workloads import graphs as G
    from workloads.sstar import gen_sstar
    n_sstar = 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mask_worker, args=(r, 2, port, n_sstar, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = G.random_training(6, 0.2, 3)
    inst = Instance.from_graph(g)
    idx_bits = max(1, (n_sstar - 1).bit_length())
    (_, keys, m0), (_, keys1, m1) = res
    assert keys == keys1 and np.array_equal(m0, m1)
    seen = 0
    for b, k in enumerate(keys):
        if k == KEY_NONE:
            assert not m0[b].any()
            continue
        i = k & ((1 << idx_bits) - 1)
        o = evaluate(inst, gen_sstar(g, "mix", 17, i, 1)[0], 0.5, keep=True)
        assert np.array_equal(m0[b, 0].view(np.uint64), masks_u64(inst, o["R"]))
        assert np.array_equal(m0[b, 1].view(np.uint64), masks_u64(inst, o["S"]))
        seen += 1
    assert seen >= 2


def _fd_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import importlib.util
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        spec = importlib.util.spec_from_file_location("cm_dist", os.path.join(root, "paper_1910_02653_b200", "dist.py"))
        D = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(D)
        fd = -1
        if rank == 0:
            r, w = os.pipe()
            os.write(w, b"multicast handle of rank 0")
            os.close(w)
            fd = r
        got = D.share_fd(fd, None)
        data = os.read(got, 64) if rank != 0 else b""
        out_q.put((rank, got >= 0, data))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_share_fd_over_unix_socket(world):
    """The NVLS multicast handle's plumbing (dist.MulticastKeys): rank 0's file descriptor
    reaches every other rank (SCM_RIGHTS over an abstract Unix socket whose name travels in the
    process group) -- here a pipe whose contents the other ranks read back."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fd_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    # every non-zero rank reads the whole message through its own duplicate: the pipe is shared,
    # so the reads split it; together they return it exactly once
    got = b"".join(d for r, _, d in res if r != 0)
    assert got == b"multicast handle of rank 0"


def _mc_fail_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1910_02653_b200 as cm
        from paper_1910_02653_b200.dist import MulticastKeys
        try:
            MulticastKeys(16)
            out_q.put((rank, "created"))
        except cm.CMError as ex:
            out_q.put((rank, "raised: " + str(ex)[:200]))
    finally:
        dist.destroy_process_group()


def test_multicast_keys_fail_together_without_gpu():
    """dist.MulticastKeys is collective: where rank 0 cannot create the multicast object (here:
    no GPU at all), every rank raises CMError -- none is left waiting in the next collective."""
    if torch.cuda.is_available():
        pytest.skip("CPU-only check of the failure path")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mc_fail_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(msg.startswith("raised") and "cm_mc_create" in msg for _, msg in res), res
