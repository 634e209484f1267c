#!/usr/bin/env python
"""HBM read ceiling for the fused kernel's access pattern (measurement tool, not the product):
tools/csrc/bw_probe.cu streams a 32 GB buffer with 1-D bulk copies of `bytes`-sized chunks,
one CTA per SM, `warps` warps x `stages` stages each; GB/s from CUDA events (best of reps).

    python tools/bw_probe.py [--json out.json]
"""
from __future__ import annotations

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "tools", "libcm_bwprobe.so")


def main():
    import torch
    lib = ctypes.CDLL(LIB)
    lib.cmbw_launch.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    total = 32 << 30
    buf = torch.empty(total // 4, dtype=torch.float32, device=dev)
    buf.uniform_()
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    res = []
    for bytes_, warps, stages in [(4096, 8, 2), (4096, 8, 3), (4096, 8, 4), (4096, 8, 5), (4096, 16, 3),
                                  (4096, 16, 2), (2304, 8, 3), (8192, 8, 3), (8192, 8, 2), (16384, 4, 3),
                                  (4096, 12, 4)]:
        if warps * stages * bytes_ > 220 * 1024:
            continue
        times = []
        for r in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            rc = lib.cmbw_launch(buf.data_ptr(), total, bytes_, warps, stages, sms, sink.data_ptr(), st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            if rc:
                break
            times.append(e0.elapsed_time(e1))
        if not times:
            res.append({"bytes": bytes_, "warps": warps, "stages": stages, "error": rc})
            continue
        best = min(times[1:]) if len(times) > 1 else times[0]
        res.append({"bytes": bytes_, "warps": warps, "stages": stages,
                    "in_flight_kb_per_sm": warps * (stages - 1) * bytes_ / 1024, "gbs": total / best / 1e6})
    out = {"what": "1-D bulk-copy read stream, one CTA per SM, 32 GB buffer, best of 3 after a warm-up",
           "sms": sms, "results": res}
    s = json.dumps(out, indent=1)
    if len(sys.argv) > 2 and sys.argv[1] == "--json":
        open(sys.argv[2], "w").write(s)
    print(s)


if __name__ == "__main__":
    main()
