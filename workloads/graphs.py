"""Synthetic computation DAGs shaped like the paper's benchmark networks.

Shared, seeded INPUT generators only: this module holds none of the method's
arithmetic (no rounding, no closure, no memory accounting).  Both the CPU
oracle tests and the CUDA path consume what it produces.

Graph model (§4.1): nodes v_1..v_n numbered in a
topological order, every edge (i, j) has i < j, node v carries a compute cost
C_v and an output size M_v.  Here indices are 0-based (node v_i <-> index i-1)
and C/M are int64 (ns / bytes), the north_star's bit-exact units (SURVEY §8(c)
Q15).

Training graphs follow SURVEY §8(d): a forward DAG f_1..f_L, loss = L+1,
b_v = 2L+2-v, edges: forward edges u->v, f_L->loss->b_L, b_v->b_u for each
forward edge u->v, and f_v->b_v.  n = 2L+1.  This generalises SPEC.md:51-59
(make_linear_training).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from .rng import mix64, u24


@dataclasses.dataclass
class Graph:
    name: str
    n: int
    edges: list            # list of (i, j), 0-based, i < j, no duplicates
    cost: np.ndarray       # int64 [n]  C_i (ns)
    mem: np.ndarray        # int64 [n]  M_i (bytes)
    ovh: int               # M_input + 2 M_param (Eq. 6 constant term)
    L: int                 # forward-node count (nodes 0..L-1 forward); L == n for non-training graphs

    # ---- plain CSR views (plumbing for the C-ABI; no method arithmetic) ----
    def pred_csr(self):
        """DEPS(k) = {i : (i,k) in E} as CSR, each list sorted ascending."""
        ptr = np.zeros(self.n + 1, np.int32)
        for (_, j) in self.edges:
            ptr[j + 1] += 1
        ptr = np.cumsum(ptr).astype(np.int32)
        idx = np.zeros(len(self.edges), np.int32)
        fill = ptr[:-1].copy()
        for (i, j) in sorted(self.edges, key=lambda e: (e[1], e[0])):
            idx[fill[j]] = i
            fill[j] += 1
        return ptr, idx

    def succ_csr(self):
        """USERS(i) = {j : (i,j) in E} as CSR, each list sorted ascending."""
        ptr = np.zeros(self.n + 1, np.int32)
        for (i, _) in self.edges:
            ptr[i + 1] += 1
        ptr = np.cumsum(ptr).astype(np.int32)
        idx = np.zeros(len(self.edges), np.int32)
        fill = ptr[:-1].copy()
        for (i, j) in sorted(self.edges):
            idx[fill[i]] = j
            fill[i] += 1
        return ptr, idx

    def last_use(self):
        """last(i) = max USERS(i), or i itself if none (SURVEY §8(d) G1 anchor)."""
        last = np.arange(self.n, dtype=np.int64)
        for (i, j) in self.edges:
            last[i] = max(last[i], j)
        return last

    def last_forward_use(self):
        """lastF(i) = max USERS(i) within the forward part + loss (0-based <= L), else i."""
        last = np.arange(self.n, dtype=np.int64)
        for (i, j) in self.edges:
            if j <= self.L:
                last[i] = max(last[i], j)
        return last

    def scaled(self, mem_factor: int) -> "Graph":
        """B·M_i in place of M_i (SPEC scale_memory); ovh unchanged."""
        return dataclasses.replace(self, mem=self.mem * int(mem_factor),
                                   name=f"{self.name}x{mem_factor}")


def _check(n, edges):
    seen = set()
    for (i, j) in edges:
        assert 0 <= i < j < n, (i, j, n)
        assert (i, j) not in seen, (i, j)
        seen.add((i, j))


# --------------------------------------------------------------------------
# Small fixtures
# --------------------------------------------------------------------------

def path(n: int, cost=None, mem=None, ovh: int = 0) -> Graph:
    """Path v_1 -> v_2 -> ... -> v_n (SURVEY §8(c) closed forms)."""
    edges = [(i, i + 1) for i in range(n - 1)]
    c = np.ones(n, np.int64) if cost is None else np.asarray(cost, np.int64)
    m = np.ones(n, np.int64) if mem is None else np.asarray(mem, np.int64)
    return Graph(f"path{n}", n, edges, c, m, int(ovh), n)


def training_from_forward(L: int, fwd_edges, cost_f=None, mem_f=None,
                          loss_cost: int = 1, loss_mem: int = 1, ovh: int = 0,
                          bwd_cost_factor=None, name="train") -> Graph:
    """Forward DAG on f_1..f_L (0-based 0..L-1) -> training graph.

    loss = index L, b_v = index 2L - v (0-based; 1-based b_v = 2L+2-v).
    Edges: forward u->v; f_L->loss; loss->b_L; b_v->b_u for each forward u->v;
    f_v->b_v.  Backward M_b = M_f; backward C_b = factor_v * C_f.
    """
    n = 2 * L + 1
    b = lambda v: 2 * L - v          # noqa: E731  (0-based backward index of forward v)
    edges = list(fwd_edges)
    edges.append((L - 1, L))
    edges.append((L, b(L - 1)))
    for (u, v) in fwd_edges:
        edges.append((b(v), b(u)))
    for v in range(L):
        edges.append((v, b(v)))
    _check(n, edges)
    cf = np.ones(L, np.int64) if cost_f is None else np.asarray(cost_f, np.int64)
    mf = np.ones(L, np.int64) if mem_f is None else np.asarray(mem_f, np.int64)
    fac = np.ones(L, np.int64) if bwd_cost_factor is None else np.asarray(bwd_cost_factor, np.int64)
    cost = np.zeros(n, np.int64)
    mem = np.zeros(n, np.int64)
    cost[:L] = cf
    mem[:L] = mf
    cost[L] = loss_cost
    mem[L] = loss_mem
    for v in range(L):
        cost[b(v)] = cf[v] * fac[v]
        mem[b(v)] = mf[v]
    return Graph(name, n, sorted(edges), cost, mem, int(ovh), L)


def training_chain(L: int, cost: int = 1, mem: int = 1) -> Graph:
    """SPEC.md:51-59 make_linear_training: n = 2L+1, |E| = 3L; unit C/M by default."""
    g = training_from_forward(L, [(i, i + 1) for i in range(L - 1)],
                              cost_f=[cost] * L, mem_f=[mem] * L,
                              loss_cost=cost, loss_mem=mem, name=f"chain{L}")
    return g


def fig4_fixture() -> Graph:
    """Fig. 4: a=1, b=2, c=3, k=4, j=5; a->k, b->k, c->k, a->j, k->j,
    plus b->c to keep the numbering realistic (SURVEY §8(c) invariant 10)."""
    edges = [(0, 3), (1, 3), (2, 3), (0, 4), (3, 4), (1, 2)]
    _check(5, edges)
    return Graph("fig4", 5, sorted(edges), np.ones(5, np.int64), np.ones(5, np.int64), 0, 5)


def random_dag(n: int, p: float, seed: int, cmax: int = 9, mmax: int = 9, ovh_max: int = 5) -> Graph:
    """Random DAG on n nodes: edge (i,j), i<j, present w.p. p; every node j>0 gets
    at least one predecessor so the graph is connected.  Seeded by splitmix64."""
    edges = []
    for j in range(1, n):
        preds = [i for i in range(j) if u24(mix64(seed, 11, i, j)) < p * (1 << 24)]
        if not preds:
            preds = [int(mix64(seed, 12, j, 0) % j)]
        edges += [(i, j) for i in preds]
    c = np.array([1 + mix64(seed, 13, v, 0) % cmax for v in range(n)], np.int64)
    m = np.array([1 + mix64(seed, 14, v, 0) % mmax for v in range(n)], np.int64)
    ovh = int(mix64(seed, 15, 0, 0) % (ovh_max + 1))
    _check(n, edges)
    return Graph(f"rand{n}_{seed}", n, edges, c, m, ovh, n)


def random_training(L: int, p_skip: float, seed: int) -> Graph:
    """Random forward DAG (chain + random skip edges) turned into a training graph."""
    fwd = [(i, i + 1) for i in range(L - 1)]
    for j in range(2, L):
        for i in range(j - 1):
            if u24(mix64(seed, 21, i, j)) < p_skip * (1 << 24):
                fwd.append((i, j))
    cf = [1 + mix64(seed, 22, v, 0) % 9 for v in range(L)]
    mf = [1 + mix64(seed, 23, v, 0) % 9 for v in range(L)]
    return training_from_forward(L, fwd, cf, mf, loss_cost=1, loss_mem=1,
                                 ovh=int(mix64(seed, 24, 0, 0) % 6),
                                 bwd_cost_factor=[1 + (mix64(seed, 25, v, 0) % 2) for v in range(L)],
                                 name=f"rtrain{L}_{seed}")


# --------------------------------------------------------------------------
# Paper-shaped networks with profiled-style int64 C/M
# --------------------------------------------------------------------------
# Layer record: (kind, out_elems_per_image, flops_per_image, params)
#   kind in {"input","conv","fc","elem","pool","reshape","softmax","add","concat","upconv"}
# C_v (ns) = ceil(batch*FLOPs/15700) + ceil(2*M_v/900) + 5000  (V100-like roofline + launch,
# echoing PAPER.md:360-361, 84); M_v = 4*batch*elements; backward C = 2x for
# conv/fc/upconv, 1x otherwise; loss C = 5000, M = 4*batch; ovh = 4*(input + 2*params);
# +-10% multiplicative jitter on C per node, seeded.

class _Net:
    def __init__(self):
        self.layers = []   # (kind, elems, flops, params)
        self.edges = []

    def add(self, kind, elems, flops=0, params=0, inputs=None):
        idx = len(self.layers)
        self.layers.append((kind, int(elems), int(flops), int(params)))
        if inputs is None:
            inputs = [idx - 1] if idx > 0 else []
        for u in inputs:
            self.edges.append((u, idx))
        return idx

    def conv(self, cin, cout, h, w, k=3, stride=1, inputs=None, kind="conv"):
        ho, wo = h // stride, w // stride
        e = cout * ho * wo
        return self.add(kind, e, 2 * e * cin * k * k, cout * cin * k * k + cout, inputs), ho, wo

    def elem(self, c, h, w, ops=1, inputs=None, kind="elem"):
        e = c * h * w
        return self.add(kind, e, ops * e, 0, inputs)


def _finish(net: _Net, name: str, batch: int, seed: int, input_elems: int) -> Graph:
    L = len(net.layers)
    cf = np.zeros(L, np.int64)
    mf = np.zeros(L, np.int64)
    fac = np.ones(L, np.int64)
    params = 0
    for v, (kind, elems, flops, prm) in enumerate(net.layers):
        m = 4 * batch * elems
        c = math.ceil(batch * flops / 15700) + math.ceil(2 * m / 900) + 5000
        jit = 0.9 + 0.2 * (u24(mix64(seed, 31, v, 0)) / float(1 << 24))
        cf[v] = int(c * jit)
        mf[v] = m
        if kind in ("conv", "fc", "upconv"):
            fac[v] = 2
        params += prm
    ovh = 4 * (batch * input_elems + 2 * params)
    return training_from_forward(L, net.edges, cf, mf, loss_cost=5000, loss_mem=4 * batch,
                                 ovh=ovh, bwd_cost_factor=fac, name=name)


def vgg16(batch: int = 64, seed: int = 1) -> Graph:
    """VGG16-shaped linear DAG: the 41-node sequence (input, 13x(conv, relu), 5xpool, flatten,
    2x(fc, relu, dropout), fc, softmax) + 3 zero-FLOP reshape nodes (after pool3/4/5) -> L=44,
    n=89, |E|=132."""
    net = _Net()
    h = w = 224
    c = 3
    net.add("input", c * h * w)
    cfg = [(64, 2), (128, 2), (256, 3), (512, 3), (512, 3)]
    for bi, (co, reps) in enumerate(cfg):
        for _ in range(reps):
            net.conv(c, co, h, w)
            c = co
            net.elem(c, h, w)                      # relu
        h //= 2
        w //= 2
        net.add("pool", c * h * w, 4 * c * h * w)
        if bi >= 2:
            net.add("reshape", c * h * w, 0)
    net.add("reshape", c * h * w, 0)               # flatten
    d = c * h * w
    for _ in range(2):
        net.add("fc", 4096, 2 * 4096 * d, 4096 * d + 4096)
        d = 4096
        net.elem(4096, 1, 1)
        net.elem(4096, 1, 1)                       # dropout
    net.add("fc", 1000, 2 * 1000 * d, 1000 * d + 1000)
    net.add("softmax", 1000, 5 * 1000)
    assert len(net.layers) == 44, len(net.layers)
    return _finish(net, "vgg16", batch, seed, 3 * 224 * 224)


def resnet50(batch: int = 32, seed: int = 2) -> Graph:
    """ResNet-50-shaped residual DAG: stem (pad, conv, bn, relu, pool) + [3,4,6,3] bottlenecks
    (8 main nodes; projection conv+bn on the first block of each stage; add, relu) + (avgpool,
    fc, softmax) -> L=176, n=353, |E|=560 (the headline)."""
    net = _Net()
    h = w = 224
    net.add("elem", 3 * 230 * 230)                 # pad (graph starts here)
    _, h, w = net.conv(3, 64, 224, 224, k=7, stride=2)
    net.elem(64, h, w, 2)                          # bn
    net.elem(64, h, w)                             # relu
    h //= 2
    w //= 2
    x = net.add("pool", 64 * h * w, 9 * 64 * h * w)
    cin = 64
    for s, blocks in enumerate([3, 4, 6, 3]):
        mid = 64 << s
        out = 256 << s
        for bidx in range(blocks):
            stride = 2 if (bidx == 0 and s > 0) else 1
            c1, _, _ = net.conv(cin, mid, h, w, k=1, inputs=[x])
            net.elem(mid, h, w, 2)
            net.elem(mid, h, w)
            _, h2, w2 = net.conv(mid, mid, h, w, k=3, stride=stride)
            net.elem(mid, h2, w2, 2)
            net.elem(mid, h2, w2)
            net.conv(mid, out, h2, w2, k=1)
            b3 = net.elem(out, h2, w2, 2)
            if bidx == 0:
                net.conv(cin, out, h, w, k=1, stride=stride, inputs=[x])
                pb = net.elem(out, h2, w2, 2)
                sc = pb
            else:
                sc = x
            net.add("add", out * h2 * w2, out * h2 * w2, inputs=[b3, sc])
            x = net.elem(out, h2, w2)              # relu
            h, w, cin = h2, w2, out
    net.add("pool", cin, cin * h * w)              # avgpool
    net.add("fc", 1000, 2 * 1000 * cin, 1000 * cin + 1000)
    net.add("softmax", 1000, 5 * 1000)
    assert len(net.layers) == 176, len(net.layers)
    return _finish(net, "resnet50", batch, seed, 3 * 224 * 224)


def unet(batch: int = 8, seed: int = 3) -> Graph:
    """U-Net-shaped DAG with long skip edges: input, 5 encoder levels x ([pad, conv, bn, relu]x2
    + pool) with the skip taken before the pool, an 8-node bottleneck, 5 decoder levels x
    (upconv, concat <- skip, [pad, conv, bn, relu]x2), head (conv1x1, sigmoid) -> L=106,
    n=213, |E|=328; skips 9->96, 18->86, 27->76, 36->66, 45->56 (1-based)."""
    net = _Net()
    h, w = 416, 608
    c = 3
    net.add("input", c * h * w)
    skips = []
    chans = [64, 128, 256, 512, 1024]
    for lvl in range(5):
        co = chans[lvl] // 2 if lvl == 4 else chans[lvl]
        for _ in range(2):
            net.elem(c, h + 2, w + 2)              # pad
            net.conv(c, co, h, w)
            c = co
            net.elem(c, h, w, 2)                   # bn
            r = net.elem(c, h, w)                  # relu
        skips.append((r, c, h, w))
        h //= 2
        w //= 2
        net.add("pool", c * h * w, 4 * c * h * w)
    # bottleneck: 8 nodes (pad, conv, bn, relu, pad, conv, bn, relu)
    for _ in range(2):
        net.elem(c, h + 2, w + 2)
        net.conv(c, c, h, w)
        net.elem(c, h, w, 2)
        net.elem(c, h, w)
    for lvl in range(5):
        sk, sc, sh, sw = skips[4 - lvl]
        up, _, _ = net.conv(c, sc, h, w, k=2, kind="upconv")
        h, w = sh, sw
        net.layers[up] = ("upconv", sc * h * w, 2 * sc * h * w * c * 4, sc * c * 4)
        cat = net.add("concat", 2 * sc * h * w, 2 * sc * h * w, inputs=[up, sk])
        c = 2 * sc
        for _ in range(2):
            net.elem(c, h + 2, w + 2)
            net.conv(c, sc, h, w)
            c = sc
            net.elem(c, h, w, 2)
            net.elem(c, h, w)
        del cat
    net.conv(c, 1, h, w, k=1)
    net.elem(1, h, w, 4, kind="softmax")           # sigmoid
    assert len(net.layers) == 106, len(net.layers)
    g = _finish(net, "unet", batch, seed, 3 * 416 * 608)
    return g


def mobilenet(batch: int = 64, seed: int = 4) -> Graph:
    """MobileNet chain: input, stem conv, 33 x (dw, bn, relu, pw, bn, relu) -> L=200, n=401,
    |E|=600 (the block count is inflated to reach n~400)."""
    net = _Net()
    net.add("input", 3 * 224 * 224)
    _, h, w = net.conv(3, 32, 224, 224, stride=2)
    c = 32
    # channel / stride schedule: MobileNet v1's 13 blocks stretched to 33
    plan = [(64, 1)] * 3 + [(128, 2)] + [(128, 1)] * 4 + [(256, 2)] + [(256, 1)] * 5 + \
           [(512, 2)] + [(512, 1)] * 14 + [(1024, 2)] + [(1024, 1)] * 3
    assert len(plan) == 33
    for co, st in plan:
        e = c * (h // st) * (w // st)
        net.add("conv", e, 2 * e * 9, c * 9)       # depthwise 3x3
        h //= st
        w //= st
        net.elem(c, h, w, 2)
        net.elem(c, h, w)
        net.conv(c, co, h, w, k=1)
        c = co
        net.elem(c, h, w, 2)
        net.elem(c, h, w)
    assert len(net.layers) == 200, len(net.layers)
    return _finish(net, "mobilenet", batch, seed, 3 * 224 * 224)


def fcn8(batch: int = 4, seed: int = 5) -> Graph:
    """FCN8 segmentation DAG: input, a VGG16 backbone whose 13 convs are each unrolled into 20
    elementwise-chained nodes (conv + 19 elementwise), 5 pools, fc6/fc7 head (conv, relu,
    dropout, conv, relu, dropout, score) and the FCN-8s skip head (upsample, score_pool4 <-
    pool4, add, upsample, score_pool3 <- pool3, add, upsample, softmax) -> L=281, n=563,
    |E|=847."""
    net = _Net()
    h, w = 416, 608
    c = 3
    net.add("input", c * h * w)
    pools = []
    for co, reps in [(64, 2), (128, 2), (256, 3), (512, 3), (512, 3)]:
        for _ in range(reps):
            net.conv(c, co, h, w)
            c = co
            for _ in range(19):
                net.elem(c, h, w)
        h //= 2
        w //= 2
        pools.append((net.add("pool", c * h * w, 4 * c * h * w), c, h, w))
    net.conv(c, 4096, h, w, k=7)
    net.elem(4096, h, w)
    net.elem(4096, h, w)
    net.conv(4096, 4096, h, w, k=1)
    net.elem(4096, h, w)
    net.elem(4096, h, w)
    score, _, _ = net.conv(4096, 21, h, w, k=1)
    p3, c3, h3, w3 = pools[2]
    p4, c4, h4, w4 = pools[3]
    up1 = net.add("upconv", 21 * h4 * w4, 2 * 21 * 21 * 16 * h4 * w4, 21 * 21 * 16, inputs=[score])
    sp4 = net.add("conv", 21 * h4 * w4, 2 * 21 * c4 * h4 * w4, 21 * c4, inputs=[p4])
    a1 = net.add("add", 21 * h4 * w4, 21 * h4 * w4, inputs=[up1, sp4])
    up2 = net.add("upconv", 21 * h3 * w3, 2 * 21 * 21 * 16 * h3 * w3, 21 * 21 * 16, inputs=[a1])
    sp3 = net.add("conv", 21 * h3 * w3, 2 * 21 * c3 * h3 * w3, 21 * c3, inputs=[p3])
    a2 = net.add("add", 21 * h3 * w3, 21 * h3 * w3, inputs=[up2, sp3])
    up3 = net.add("upconv", 21 * 416 * 608, 2 * 21 * 21 * 256 * 416 * 608 // 64, 21 * 21 * 256,
                  inputs=[a2])
    net.add("softmax", 21 * 416 * 608, 5 * 21 * 416 * 608, inputs=[up3])
    assert len(net.layers) == 281, len(net.layers)
    return _finish(net, "fcn8", batch, seed, 3 * 416 * 608)


NETWORKS = {"vgg16": vgg16, "resnet50": resnet50, "unet": unet,
            "mobilenet": mobilenet, "fcn8": fcn8}
