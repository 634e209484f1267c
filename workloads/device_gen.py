"""Device-side S* generation (workloads/libcm_gen.so), bit-identical to
workloads/sstar.py.  Used by bench.py to fill HBM-sized batches without a host
round trip; tests check it byte for byte against the numpy generator."""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .sstar import FAMILY_IDS, SIGMA_SCALE, blk_size, roundup4, tri4_size

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcm_gen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1910_02653_b200.build`")
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        lib.cmgen_sstar.argtypes = [ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, ctypes.c_uint64,
                                    ctypes.c_int64, ctypes.c_int32, ctypes.c_int, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_float, ctypes.c_float, P, P]
        lib.cmgen_sstar.restype = ctypes.c_int
        _lib = lib
    return _lib


class DeviceGenerator:
    def __init__(self, graph, family: str, seed: int, layout: str = "dense", ld: int | None = None,
                 device="cuda"):
        import torch
        self.g = graph
        self.family = FAMILY_IDS[family]
        self.seed = int(seed)
        self.layout = layout
        n = graph.n
        if layout == "dense":
            self.ld = roundup4(n) if ld is None else int(ld)
            self.stride = n * self.ld
        elif layout == "tri4":
            self.ld = 0
            self.stride = tri4_size(n)
        elif layout == "blk":
            self.ld = 0
            self.stride = blk_size(n)
        else:
            raise ValueError(layout)
        self.last = torch.tensor(graph.last_use().astype(np.int32), device=device)
        self.lastF = torch.tensor(graph.last_forward_use().astype(np.int32), device=device)

    def shape(self, count):
        return (count, self.g.n, self.ld) if self.layout == "dense" else (count, self.stride)

    def fill(self, out, s_begin: int, upper: float = 0.0, stream=None):
        """Write S* #s_begin .. s_begin + out.shape[0] - 1 into the float32 CUDA tensor ``out``."""
        import torch
        lib = _load()
        count = out.shape[0]
        if stream is None:
            stream = torch.cuda.current_stream(out.device).cuda_stream
        with torch.cuda.nvtx.range("cm_generate_sstar"):
            rc = lib.cmgen_sstar(self.g.n, self.g.L, self.last.data_ptr(), self.lastF.data_ptr(),
                                 self.family, self.seed, int(s_begin), int(count),
                                 {"dense": 0, "tri4": 1, "blk": 2}[self.layout], self.ld, self.stride,
                                 float(upper), float(SIGMA_SCALE), out.data_ptr(), ctypes.c_void_p(stream))
        if rc != 0:
            raise RuntimeError(f"cmgen_sstar failed: cudaError {rc}")
        return out
