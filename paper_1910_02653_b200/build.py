"""In-tree build of the sm_100a shared libraries (nvcc; no JIT cache).

    python paper_1910_02653_b200/build.py [--force]   # builds both libraries if stale
    (run as a file: importing the package needs the library this produces)

libcheckmate_b200.so   the product: C ABI of include/cm.h
workloads/libcm_gen.so the device input generator (workloads/csrc/gen_sstar.cu)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]

LIBS = {
    os.path.join(PKG, "libcheckmate_b200.so"): (
        sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu"))),
        sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "cm.h")],
        ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc")],
    ),
    os.path.join(ROOT, "workloads", "libcm_gen.so"): (
        [os.path.join(ROOT, "workloads", "csrc", "gen_sstar.cu")],
        [],
        [],
    ),
}


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> list:
    built = []
    for out, (srcs, hdrs, inc) in LIBS.items():
        if not force and not _stale(out, srcs + hdrs):
            continue
        cmd = [NVCC] + ARCH + FLAGS + inc + ["-o", out] + srcs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {out}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        log = out + ".ptxas.txt"
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
        if verbose:
            print(r.stdout + r.stderr)
        built.append(out)
    return built


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
