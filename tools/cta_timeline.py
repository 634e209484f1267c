#!/usr/bin/env python
"""CM_TRACE=2 timeline of one fused call (timing diagnostic): per CTA, relative to the first
CTA start (ms): rounding warps done (K1 end), first unit-0 wait satisfied, scan warps done
(K2 end); min / median / max over CTAs.

    python tools/cta_timeline.py [--config resnet50] [--layout blk] [--batch N]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="resnet50")
    ap.add_argument("--layout", default="blk")
    ap.add_argument("--batch", type=int, default=None)
    a = ap.parse_args()
    os.environ["CM_TRACE"] = "2"
    import torch
    import bench
    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator
    g, fam, thetas, budgets, batch = bench.build_workload(a.config)
    batch = a.batch or batch
    ld = -(-g.n // 32) * 32 if a.layout == "dense" else None
    dg = DeviceGenerator(g, fam, bench.BENCH_SEED, layout=a.layout, ld=ld)
    x = torch.empty(dg.shape(batch), dtype=torch.float32, device="cuda")
    dg.fill(x, 0)
    graph = cm.Graph.from_workload(g)
    th = torch.tensor(thetas, device="cuda")
    bu = torch.tensor(budgets, device="cuda")
    for _ in range(3):
        cm.round_and_evaluate(graph, x, th, bu, layout=a.layout)
        torch.cuda.synchronize()
    t = cm.debug_cta_trace().astype(np.float64)
    t0 = t[:, 0].min()
    k1 = (t[:, 1] - t0) / 1e6
    first = (np.array([~int(v) & ((1 << 64) - 1) for v in t[:, 2].astype(np.uint64)], np.float64) - t0) / 1e6
    k2 = (t[:, 3] - t0) / 1e6
    q = lambda v: "%.3f / %.3f / %.3f" % (v.min(), np.median(v), v.max())
    print(f"{a.config} {a.layout} batch {batch}: CTAs {t.shape[0]}")
    print("  CTA start      ", q((t[:, 0] - t0) / 1e6))
    print("  K1 (rounding) end", q(k1))
    print("  first unit ready ", q(first[(first > -1) & (first < 1e3)]) if ((first > -1) & (first < 1e3)).any() else "-")
    print("  K2 (scan) end    ", q(k2))


if __name__ == "__main__":
    main()
