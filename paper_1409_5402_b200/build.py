"""Build the package's native libraries in-tree for sm_100a (no torch extension machinery).

    python -m paper_1409_5402_b200.build [--force]

libsamelda_cuda.so    the product: kernels_*.cu (compiled with -fmad=false:
                      reference-identical f64 rounding -- the reference is an
                      x86-64 build without FMA), capi.cu (context, C ABI,
                      multi-GPU group), corpus_io.cpp (data formats)
libsamelda_synth.so   the synthetic corpus generator (host C++, no CUDA): the
                      bench and the tests load it without mapping the product
                      library (the reference arm of bench.py uses it too)

Translation units compile in parallel.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libsamelda_cuda.so")
SYNTH_LIB = os.path.join(PKG, "libsamelda_synth.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "-I", CSRC,
          "-I", os.path.join(ROOT, "include")]
# extra nvcc / g++ flags per unit (SAMELDA_NVCC_EXTRA adds to every .cu unit,
# e.g. -DSAMELDA_AB_VARIANTS for the A/B tools)
UNITS = {
    "kernels_sample.cu": ["-fmad=false"],
    "kernels_mstep.cu": ["-fmad=false"],
    "kernels_eval.cu": ["-fmad=false"],
    "kernels_cgs.cu": ["-fmad=false"],
    "capi.cu": [],
    "group.cu": [],
    "corpus_io.cpp": [],
}
SYNTH_UNITS = {"synth.cpp": []}
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


def _compile_cmd(unit: str, flags: list[str], obj: str) -> list[str]:
    src = os.path.join(CSRC, unit)
    if unit.endswith(".cpp"):
        return [os.environ.get("CXX", "g++"), *GXX, *flags, "-c", src, "-o", obj]
    extra = os.environ.get("SAMELDA_NVCC_EXTRA", "").split()
    return [nvcc(), *ARCH, *COMMON, *flags, *extra, "-c", src, "-o", obj]


def _objects(units: dict, headers: list[str], force: bool, verbose: bool) -> list[str]:
    jobs, objs = [], []
    for unit, flags in units.items():
        src = os.path.join(CSRC, unit)
        if not os.path.exists(src):
            continue
        obj = os.path.join(BUILD, os.path.splitext(unit)[0] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            jobs.append(_compile_cmd(unit, flags, obj))

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(run, c) for c in jobs]:
            f.result()
    return objs


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers += [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    objs = _objects(UNITS, headers, force, verbose)
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lpthread", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    sobjs = _objects(SYNTH_UNITS, headers, force, verbose)
    if force or _stale(SYNTH_LIB, sobjs):
        cmd = [os.environ.get("CXX", "g++"), "-shared", "-o", SYNTH_LIB, *sobjs, "-pthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
