#!/usr/bin/env python
"""Algorithmic integer ops per candidate from the CPU oracle's A8 counters.

    python tools/ops_alg.py [--count 64] > profiles/ops_alg.json

Ops_alg = tri (threshold compares) + n*W (phase-2a words) + V (closure edge visits)
        + F (free events) + sum R (compute / cost events) + sum S (U_{t,0} terms),
W = ceil(n/64), averaged over S* #0..count-1 of bench.py's seeded workload of each config
(bench seed, family).  Randomized rounding (key "rand_<family>", --rand-samples K): the same
counters of the randomized candidates (oracle evaluate_randomized, samples 0..K-1 of each S*,
the bench seed), whose S -- and so closure, frees, sum R, sum S -- differ from the
deterministic ones; the generator's own work is added by bench.py per element and sample.
Calls only oracle/ (a stored value written by a committed script)."""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _one(job):
    cfg, fam, seed, s, j = job
    import bench
    from oracle import Instance, evaluate, evaluate_randomized
    from workloads.sstar import gen_sstar
    g, _, thetas, _, _ = bench.build_workload(cfg, fam)
    inst = Instance.from_graph(g)
    x = gen_sstar(g, fam, seed, s, 1)[0]
    o = evaluate(inst, x, thetas[0]) if j is None else evaluate_randomized(inst, x, s, j, seed)
    return cfg, fam if j is None else "rand_" + fam, o["counters"]


def ops_of(n: int, c: dict) -> float:
    tri = n * (n - 1) // 2
    W = (n + 63) // 64
    return tri + n * W + c["closure_visits"] + c["free_events"] + c["sum_R"] + c["sum_S"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=64)
    ap.add_argument("--configs", default="resnet50,vgg16,unet,mobilenet,fcn8")
    ap.add_argument("--families", default="g1,g2,mix")
    ap.add_argument("--rand-samples", type=int, default=4, help="randomized samples per S* (resnet50, g1)")
    ap.add_argument("--rand-count", type=int, default=32)
    a = ap.parse_args()
    import bench
    jobs = [(cfg, fam, bench.BENCH_SEED, s, None) for cfg in a.configs.split(",") for fam in a.families.split(",")
            for s in range(a.count)]
    jobs += [("resnet50", "g1", bench.BENCH_SEED, s, j) for s in range(a.rand_count) for j in range(a.rand_samples)]
    with mp.get_context("spawn").Pool(len(os.sched_getaffinity(0))) as pool:
        res = pool.map(_one, jobs, chunksize=4)
    out = {}
    for cfg in a.configs.split(","):
        g = bench.build_workload(cfg)[0]
        fams = a.families.split(",") + (["rand_g1"] if cfg == "resnet50" and a.rand_samples else [])
        for fam in fams:
            cs = [c for (cf, fm, c) in res if cf == cfg and fm == fam]
            mean = {k: sum(c[k] for c in cs) / len(cs) for k in cs[0]}
            how = (f"S* #0..{a.rand_count - 1} x samples 0..{a.rand_samples - 1}, randomized (R1), bench seed "
                   f"{bench.BENCH_SEED}" if fam.startswith("rand_") else
                   f"S* #0..{a.count - 1}, bench seed {bench.BENCH_SEED}, theta {bench.CONFIGS[cfg][2][0]}")
            out.setdefault(cfg, {})[fam] = {
                "n": g.n, "ops_alg_per_candidate": sum(ops_of(g.n, c) for c in cs) / len(cs),
                "tri": g.n * (g.n - 1) // 2, "n_W": g.n * ((g.n + 63) // 64), "counters_mean": mean,
                "sample": how}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
