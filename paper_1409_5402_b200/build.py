"""Build libsamelda_cuda.so in-tree for sm_100a (no torch extension machinery).

    python -m paper_1409_5402_b200.build

the kernels_*.cu units are compiled with -fmad=false (reference-identical f64 rounding:
the reference is an x86-64 build without FMA); capi.cu is host code.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libsamelda_cuda.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "-I", CSRC,
          "-I", os.path.join(ROOT, "include")]
UNITS = {
    "kernels_sample.cu": ["-fmad=false"],
    "kernels_mstep.cu": ["-fmad=false"],
    "kernels_eval.cu": ["-fmad=false"],
    "capi.cu": [],
    "synth.cpp": [],
    "corpus_io.cpp": [],
}
GXX = ["-O3", "-std=c++20", "-fPIC", "-pthread", "-I", CSRC, "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "samelda_cu.h"))
    objs = []
    for unit, flags in UNITS.items():
        src = os.path.join(CSRC, unit)
        if not os.path.exists(src):
            continue
        obj = os.path.join(BUILD, os.path.splitext(unit)[0] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            if unit.endswith(".cpp"):
                cmd = [os.environ.get("CXX", "g++"), *GXX, *flags, "-c", src, "-o", obj]
            else:
                cmd = [nvcc(), *ARCH, *COMMON, *flags, "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
