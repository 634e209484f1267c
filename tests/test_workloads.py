"""Input generators: shapes of the paper-like DAGs, the G1 anchor's
structure, layouts and determinism.  CPU only."""
import numpy as np
import pytest

from tests.oracle_helpers import S_chen
from workloads import budgets as B
from workloads import graphs as G
from workloads.sstar import (dense_to_tri4, g1_anchor_row, g1_params, gen_sstar, tri4_offset,
                             tri4_size)

SHAPES = {"vgg16": (89, 132), "resnet50": (353, 560), "unet": (213, 328),
          "mobilenet": (401, 600), "fcn8": (563, 847)}


@pytest.mark.parametrize("name", sorted(SHAPES))
def test_network_shapes(name):
    g = G.NETWORKS[name]()
    assert (g.n, len(g.edges)) == SHAPES[name]
    assert g.n == 2 * g.L + 1
    assert all(0 <= i < j < g.n for (i, j) in g.edges)
    assert len(set(g.edges)) == len(g.edges)
    assert (g.cost > 0).all() and (g.mem > 0).all() and g.ovh > 0
    ptr, idx = g.pred_csr()
    assert ptr[-1] == len(g.edges)
    for k in range(g.n):
        lst = list(idx[ptr[k]:ptr[k + 1]])
        assert lst == sorted(lst)


def test_unet_skips():
    g = G.unet()
    skips = {(9, 96), (18, 86), (27, 76), (36, 66), (45, 56)}
    got = {(i + 1, j + 1) for (i, j) in g.edges if j < g.L and j - i > 1}
    assert got == skips


def test_resnet_max_indegree():
    g = G.resnet50()
    ptr, _ = g.pred_csr()
    assert (np.diff(ptr)).max() == 3


@pytest.mark.parametrize("L,K", [(16, [4, 8, 12]), (10, [5, 9]), (8, [3, 6]), (5, []), (6, [1, 2, 3, 4, 5, 6])])
def test_g1_anchor_is_chen_on_chain(L, K):
    """On the training chain the G1 anchor equals the Chen-segmented pattern."""
    g = G.training_chain(L)
    Kmask = np.zeros(L, bool)
    for c in K:
        Kmask[c - 1] = True
    from workloads.sstar import segment_tops
    tau = segment_tops(L, Kmask)
    want = S_chen(L, K)
    last, lastF = g.last_use(), g.last_forward_use()
    for r in range(g.n):
        a = g1_anchor_row(r, L, Kmask, tau, last, lastF)
        assert list(a) == list(want[r, :r]), r


def test_tri4_layout():
    for r in range(40):
        assert tri4_offset(r) % 4 == 0
        assert tri4_offset(r + 1) - tri4_offset(r) == (r + 3) // 4 * 4
    g = G.random_training(4, 0.3, 2)
    d = gen_sstar(g, "mix", 3, 10, 3)
    t = gen_sstar(g, "mix", 3, 10, 3, layout="tri4")
    assert t.shape == (3, tri4_size(g.n))
    assert (dense_to_tri4(d) == t).all()


def test_generator_determinism_and_ranges():
    g = G.resnet50()
    a = gen_sstar(g, "g1", 42, 5, 2)
    b = gen_sstar(g, "g1", 42, 5, 2)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    c = gen_sstar(g, "g1", 42, 6, 1)
    assert np.array_equal(a[1].view(np.uint32), c[0].view(np.uint32))
    lo = np.tril(np.ones((g.n, a.shape[2]), bool), -1)
    vals = a[0][lo[:, :a.shape[2]]]
    assert vals.min() >= 0 and vals.max() <= 1
    assert (vals == 0.5).sum() > 0            # PSI: exact ties present
    u = gen_sstar(g, "g2", 1, 0, 1)[0][lo]
    assert 0.45 < u.mean() < 0.55


def test_g1_params_rho():
    L = 176
    rhos = set()
    for s in range(30):
        K, tau = g1_params(9, s, L)
        rhos.add(round(K.mean(), 1))
        for v in range(L):
            if not K[v]:
                assert tau[v] >= v and not K[tau[v]]
                assert tau[v] == L - 1 or K[tau[v] + 1]
    assert len(rhos) >= 2


def test_budget_grid():
    g = G.resnet50()
    grid = B.geometric_grid(g, 16)
    assert len(grid) == 16 and (np.diff(grid) > 0).all()
    assert grid[-1] == B.p_live(g) and grid[0] >= B.p_floor(g)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 32, 33, 34, 64, 65, 89, 213, 353, 401, 563, 1024])
def test_blk_layout_is_a_bijection(n):
    """CM_LAYOUT_BLK: every strict-lower entry (r, i) has its own float position inside the
    S*'s blk_size(n) floats; the size agrees with the library's cm_sstar_floats."""
    import ctypes
    from paper_1910_02653_b200 import _abi
    from workloads.sstar import blk_positions, blk_size
    lib = _abi.load()
    assert lib.cm_sstar_floats(n, 2, 0) == blk_size(n)
    r, i, pos = blk_positions(n)
    assert len(pos) == n * (n - 1) // 2
    assert len(np.unique(pos)) == len(pos)
    assert (pos >= 0).all() and (pos < max(1, blk_size(n))).all()
    assert blk_size(n) % 4 == 0
    del ctypes


def test_blk_layout_small_case_by_hand():
    """n = 6 (one group of h = 5 rows, one diagonal block, chunk-major): chunk 0 of rows
    l = 0..4 at chunks 0..4, chunk 1 (nodes 4..7) of row l = 4 (r = 5) at chunk 5."""
    from workloads.sstar import blk_positions, blk_size, dense_to_blk
    assert blk_size(6) == 4 * (5 + 1)
    x = np.zeros((1, 6, 8), np.float32)
    for r in range(6):
        for i in range(r):
            x[0, r, i] = 10 * r + i
    b = dense_to_blk(x, upper=-1.0)[0]
    assert list(b[0:4]) == [10, -1, -1, -1]                   # row 1: node 0
    assert list(b[16:20]) == [50, 51, 52, 53]                 # row 5 (l = 4), chunk 0
    assert list(b[20:24]) == [54, -1, -1, -1]                 # row 5, chunk 1 (node 4)
    r, i, pos = blk_positions(6)
    assert dict(zip(zip(r.tolist(), i.tolist()), pos.tolist()))[(3, 2)] == 4 * 2 + 2


def test_blk_layout_offdiagonal_chunk_major():
    """n = 40: group 1 holds rows 33..39 (h = 7); its block w = 0 is chunk-major, chunk c of row
    l at chunk 7 c + l; group 0's 32 x 32 diagonal block (576 floats) precedes it."""
    from workloads.sstar import dense_to_blk
    x = np.zeros((1, 40, 40), np.float32)
    for r in range(40):
        for i in range(r):
            x[0, r, i] = 1000 * r + i
    b = dense_to_blk(x)[0]
    base = 576
    for l in range(7):
        for c in range(8):
            o = base + 4 * (7 * c + l)
            assert list(b[o:o + 4]) == [1000 * (33 + l) + 4 * c + e for e in range(4)]
