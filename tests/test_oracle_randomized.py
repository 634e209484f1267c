"""Pins of the oracle's randomized two-phase rounding (R1).

The generator is pinned by the published Philox4x32-10 known-answer vectors; the rounding
rule by the cases where it must reduce to deterministic rounding, by its mean, and by the
paper's Appendix D comparison (deterministic rounding is not beaten on average)."""
import json
import os

import numpy as np

from oracle import Instance, evaluate, evaluate_randomized, philox4x32_10, round_S, round_S_randomized, uniforms
from oracle.randomized import philox4x32_10_np, uniform32
from workloads import graphs as G
from workloads.sstar import from_binary, gen_sstar

HERE = os.path.dirname(os.path.abspath(__file__))


def test_philox_known_answers():
    kat = json.load(open(os.path.join(HERE, "golden", "philox4x32_10_kat.json")))
    for v in kat["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        want = [int(x, 16) for x in v["out"]]
        assert list(philox4x32_10(ctr, key)) == want
        got = philox4x32_10_np(*[np.array([c], np.uint64) for c in ctr], key[0], key[1])
        assert [int(g[0]) for g in got] == want


def test_uniform_mapping_exact():
    w = np.array([0, 1, 255, 256, 0xFFFFFFFF, 0x80000000], np.uint32)
    u = uniform32(w)
    assert u.dtype == np.float64
    assert list(u) == [0.0, 2.0 ** -32, 255 * 2.0 ** -32, 2.0 ** -24, 1.0 - 2.0 ** -32, 0.5]


def test_compare_is_exact_at_the_boundary():
    """S = 1[u < S*] on the real values (R1): S* equal to a uniform never fires,
    one fp32 ulp above it does, whatever the word's low bits; S* = 1 always fires, 0 never."""
    n = 6
    inst = Instance(n, [], np.zeros(n, np.int64), np.zeros(n, np.int64), 0)
    U = uniforms(n, 5, 1, 77)
    x = np.zeros((n, n), np.float32)
    for t in range(2, n + 1):
        for i in range(1, t):
            u = U[t - 1, i - 1]
            # the fp32 nearest below / at-or-above u: [u < x] is 0 and 1 respectively
            lo = np.float32(u)
            lo = lo if float(lo) <= u else np.nextafter(lo, np.float32(0))
            hi = lo if float(lo) == u else np.nextafter(lo, np.float32(1))
            hi = hi if float(hi) > u else np.nextafter(hi, np.float32(1))
            x[t - 1, i - 1] = hi if (t + i) % 2 else lo
    S = round_S_randomized(inst, x, 5, 1, 77)
    for t in range(2, n + 1):
        for i in range(1, t):
            assert S[t, i] == bool((t + i) % 2), (t, i)
    assert round_S_randomized(inst, np.ones((n, n), np.float32), 5, 1, 77)[1:n + 1, 1:].sum() == n * (n - 1) // 2
    assert not round_S_randomized(inst, np.zeros((n, n), np.float32), 5, 1, 77).any()


def test_binary_sstar_equals_deterministic():
    """S* in {0, 1}: u in [0, 1) gives u < 1 always and u < 0 never, so every sample equals
    the deterministic rounding at theta = 0.5 (and the whole candidate does)."""
    g = G.random_training(6, 0.2, 3)
    inst = Instance.from_graph(g)
    rng = np.random.default_rng(1)
    for trial in range(4):
        S0 = np.tril(rng.random((g.n, g.n)) < 0.4, -1)
        x = from_binary(S0)
        det = evaluate(inst, x, 0.5)
        for j in range(3):
            assert np.array_equal(round_S_randomized(inst, x, trial, j, 99), round_S(inst, x, 0.5))
            r = evaluate_randomized(inst, x, trial, j, 99)
            assert (r["peak"], r["cost"]) == (det["peak"], det["cost"])


def test_mean_and_independence():
    """Pr[S = 1] = S* (PAPER.md:383): constant S* = p gives a fraction p of ones (5 sigma),
    different samples / S* numbers / seeds give different S, NaN never sets a bit."""
    n = 96
    inst = Instance(n, [], np.zeros(n, np.int64), np.zeros(n, np.int64), 0)
    tri = n * (n - 1) // 2
    for p in (0.1, 0.5, 0.9):
        x = np.full((n, n), p, np.float32)
        S = round_S_randomized(inst, x, 7, 2, 12345)
        frac = S[1:n + 1, 1:].sum() / tri
        assert abs(frac - p) < 5 * np.sqrt(p * (1 - p) / tri)
        assert not np.triu(S[1:n + 1, 1:]).any()          # only i < t
    x = np.full((n, n), 0.5, np.float32)
    base = round_S_randomized(inst, x, 7, 0, 1)
    for s, j, seed in [(7, 1, 1), (8, 0, 1), (7, 0, 2), (7, 4, 1)]:
        assert not np.array_equal(base, round_S_randomized(inst, x, s, j, seed))
    x[:] = np.nan
    assert not round_S_randomized(inst, x, 7, 0, 1).any()


def test_uniforms_layout():
    """u(s, j, t, i) uses counter ((i-1) div 4, t-1, s, j) and output word (i-1) mod 4
    (R1): written out with the scalar Philox block for every (t, i) of n = 9."""
    U = uniforms(9, 3, 6, (7 << 32) | 11)
    for t in range(1, 10):
        for i in range(1, 10):
            w = philox4x32_10(((i - 1) // 4, t - 1, 3, 6), (11, 7))[(i - 1) % 4]
            assert U[t - 1, i - 1] == w / 2.0 ** 32
    # one block serves four consecutive nodes: nodes 1..4 of a row are its four words
    blk = philox4x32_10((0, 2, 3, 6), (11, 7))
    assert [U[2, q] for q in range(4)] == [w / 2.0 ** 32 for w in blk]


def test_appendix_d_deterministic_not_worse():
    """App. D: 'two-phase deterministic rounding produces consistently lower
    cost schedules' than the mean of randomized ones.  On LP-like S* of the training chain
    the deterministic cost is at most the mean sampled cost."""
    g = G.training_chain(8)
    inst = Instance.from_graph(g)
    for s in range(3):
        x = gen_sstar(g, "g1", 5, s, 1)[0]
        det = evaluate(inst, x, 0.5)["cost"]
        costs = [evaluate_randomized(inst, x, s, j, 2024)["cost"] for j in range(24)]
        assert det <= np.mean(costs)
