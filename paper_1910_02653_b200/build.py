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
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
         "-static-global-template-stub=false"]   # kernel instances live in their own TUs (cm_inst.cuh)

LIBS = {
    os.path.join(PKG, "libcheckmate_b200.so"): (
        sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.cpp"))),
        sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "cm.h")],
        ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc")],
    ),
    os.path.join(ROOT, "workloads", "libcm_gen.so"): (
        [os.path.join(ROOT, "workloads", "csrc", "gen_sstar.cu")],
        [],
        [],
    ),
    # measurement tools (integer-pipe roofline, tools/int_peak.py; HBM read ceiling of the
    # bulk-copy pattern, tools/bw_probe.py), not the product
    os.path.join(ROOT, "tools", "libcm_bwprobe.so"): (
        [os.path.join(ROOT, "tools", "csrc", "bw_probe.cu")],
        [],
        [],
    ),
    os.path.join(ROOT, "tools", "libcm_intpeak.so"): (
        [os.path.join(ROOT, "tools", "csrc", "int_peak.cu")],
        [],
        [],
    ),
}


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile_one(src, obj, inc):
    cmd = [NVCC] + ARCH + [f for f in FLAGS if f != "-shared"] + inc + ["-c", "-o", obj, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return cmd, r


def build(force: bool = False, verbose: bool = False, extra=None, out_override=None) -> list:
    """Each .cu is compiled to an object in parallel (the kernel instances live in their own
    translation units), then linked into the shared library."""
    from concurrent.futures import ThreadPoolExecutor
    built = []
    for out, (srcs, hdrs, inc) in LIBS.items():
        if out_override and out.endswith("libcheckmate_b200.so"):
            out = out_override
        elif out_override:
            continue
        if not force and not extra and not _stale(out, srcs + hdrs):
            continue
        inc = inc + list(extra or [])
        objdir = os.path.join(os.path.dirname(out), "build", os.path.basename(out))
        os.makedirs(objdir, exist_ok=True)
        objs = [os.path.join(objdir, os.path.basename(sf) + ".o") for sf in srcs]
        with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 4))) as ex:
            res = list(ex.map(lambda a: _compile_one(*a), [(sf, ob, inc) for sf, ob in zip(srcs, objs)]))
        logs = []
        for cmd, r in res:
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
            logs.append(r.stdout + r.stderr)
        cmd = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", out] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc link failed for {out}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        with open(out + ".ptxas.txt", "w") as f:
            f.write("".join(logs))
        if verbose:
            print("".join(logs))
        built.append(out)
    return built


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
