#!/usr/bin/env python
"""HBM probe (timing experiment, not a product path): read-only bandwidth of a large
fp32 buffer through torch's sum and amax (one pass), and a copy, with CUDA events."""
import json
import torch

dev = torch.device("cuda:0")
n = (16 << 30) // 4
x = torch.rand(n, device=dev)
y = torch.empty_like(x)
out = {}
for name, fn, bytes_ in [("sum", lambda: x.sum(), 4 * n), ("amax", lambda: x.amax(), 4 * n),
                         ("copy", lambda: y.copy_(x), 8 * n)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    out[name] = bytes_ / best / 1e6
print(json.dumps({"gbs": out}))
