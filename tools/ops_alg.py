#!/usr/bin/env python
"""Algorithmic integer ops per candidate from the CPU oracle's A8 counters.

    python tools/ops_alg.py [--count 64] > profiles/ops_alg.json

Ops_alg = tri (threshold compares) + n*W (phase-2a words) + V (closure edge visits)
        + F (free events) + sum R (compute / cost events) + sum S (U_{t,0} terms),
W = ceil(n/64), averaged over S* #0..count-1 of bench.py's seeded workload of each config
(bench seed, family).  Calls only oracle/ (a stored value written by a committed script)."""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _one(job):
    cfg, fam, seed, s = job
    import bench
    from oracle import Instance, evaluate
    from workloads.sstar import gen_sstar
    g, _, thetas, _, _ = bench.build_workload(cfg, fam)
    inst = Instance.from_graph(g)
    o = evaluate(inst, gen_sstar(g, fam, seed, s, 1)[0], thetas[0])
    return cfg, fam, o["counters"]


def ops_of(n: int, c: dict) -> float:
    tri = n * (n - 1) // 2
    W = (n + 63) // 64
    return tri + n * W + c["closure_visits"] + c["free_events"] + c["sum_R"] + c["sum_S"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=64)
    ap.add_argument("--configs", default="resnet50,vgg16,unet,mobilenet,fcn8")
    ap.add_argument("--families", default="g1,g2,mix")
    a = ap.parse_args()
    import bench
    jobs = [(cfg, fam, bench.BENCH_SEED, s) for cfg in a.configs.split(",") for fam in a.families.split(",")
            for s in range(a.count)]
    with mp.get_context("spawn").Pool(len(os.sched_getaffinity(0))) as pool:
        res = pool.map(_one, jobs, chunksize=4)
    out = {}
    for cfg in a.configs.split(","):
        g = bench.build_workload(cfg)[0]
        for fam in a.families.split(","):
            cs = [c for (cf, fm, c) in res if cf == cfg and fm == fam]
            mean = {k: sum(c[k] for c in cs) / len(cs) for k in cs[0]}
            out.setdefault(cfg, {})[fam] = {
                "n": g.n, "ops_alg_per_candidate": sum(ops_of(g.n, c) for c in cs) / len(cs),
                "tri": g.n * (g.n - 1) // 2, "n_W": g.n * ((g.n + 63) // 64), "counters_mean": mean,
                "sample": f"S* #0..{a.count - 1}, bench seed {bench.BENCH_SEED}, theta {bench.CONFIGS[cfg][2][0]}"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
