#!/usr/bin/env python
"""K-mu: the integer-pipe roofline denominator, MEASURED.

Runs tools/csrc/int_peak.cu (tools/libcm_intpeak.so, built by paper_1910_02653_b200/build.py)
on cuda:0: per instruction class, a full-chip grid of long independent chains; lane ops per
second from CUDA events, and the loaded SM clock the kernel itself saw (%clock64 over
%globaltimer per CTA, median).

    python tools/int_peak.py [--pipes] [--json out.json]
"""
from __future__ import annotations

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "tools", "libcm_intpeak.so")
CLASSES = {0: "lop3", 1: "iadd3", 2: "imad", 3: "lop3+imad", 4: "popc", 5: "flo", 6: "shfl", 7: "fsetp+or"}
# pipe probes (--pipes): which pipe the randomized-rounding K1 instructions issue to
PIPES = {8: "imad.wide", 9: "i2fp", 10: "shf.l.w", 11: "ffma2", 12: "imad.hi", 13: "lop3+i2fp",
         14: "lop3+imad.wide", 15: "lop3+imad.hi", 16: "carry-pack", 17: "lop3+ffma2", 18: "lop3+shf",
         19: "lop3+carry-pack"}


def _lib():
    if not os.path.exists(LIB):
        raise RuntimeError(f"{LIB} missing: run paper_1910_02653_b200/build.py")
    lib = ctypes.CDLL(LIB)
    lib.cmip_launch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p]
    lib.cmip_launch.restype = ctypes.c_int
    lib.cmip_ops_per_iter.argtypes = [ctypes.c_int]
    lib.cmip_ops_per_iter.restype = ctypes.c_int
    return lib


def measure(iters: int = 8192, reps: int = 3, device: int = 0, pipes: bool = False) -> dict:
    import numpy as np
    import torch
    lib = _lib()
    dev = torch.device("cuda", device)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks = 4 * sms
    sink = torch.zeros(4, dtype=torch.int32, device=dev)
    clk = torch.zeros(2 * blocks, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    out = {}
    for cls, name in ({**CLASSES, **PIPES} if pipes else CLASSES).items():
        rc = lib.cmip_launch(cls, blocks, 64, 1, sink.data_ptr(), clk.data_ptr(), st.cuda_stream)   # warm-up
        if rc != 0:
            raise RuntimeError(f"int_peak launch failed: cudaError {rc}")
        best, mhz = 1e30, []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            lib.cmip_launch(cls, blocks, iters, 12345, sink.data_ptr(), clk.data_ptr(), st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e1))
            c = clk.view(-1, 2).cpu().numpy().astype(np.float64)
            mhz.append(float(np.median(c[:, 0] / np.maximum(c[:, 1], 1)) * 1e3))
        ops = float(blocks) * 256 * iters * lib.cmip_ops_per_iter(cls)
        out[name] = {"tops": ops / (best / 1e3) / 1e12, "ms": best, "sm_mhz": float(np.median(mhz)),
                     "ops_per_sm_cycle": ops / (best / 1e3) / sms / (float(np.median(mhz)) * 1e6)}
    return {"sms": sms, "classes": out,
            "int_peak_tops": out["lop3+imad"]["tops"], "alu_tops": out["lop3"]["tops"],
            "how": "tools/csrc/int_peak.cu: 4 CTAs x 256 threads per SM, 8 independent chains per thread, "
                   "CUDA-event time (best of %d), SM clock from %%clock64 / %%globaltimer per CTA" % reps}


if __name__ == "__main__":
    r = measure(pipes="--pipes" in sys.argv)
    s = json.dumps(r, indent=1)
    if "--json" in sys.argv:
        open(sys.argv[sys.argv.index("--json") + 1], "w").write(s + "\n")
    print(s)
