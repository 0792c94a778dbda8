"""Builds libgdx.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2311_06837_b200.build          # or via __graft_entry__.build()

The library is the whole product: CUDA kernels + the C ABI of include/gdx.h +
host C++.  It is written next to this file so the gpurun snapshot carries it.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libgdx.so")
OBJ = os.path.join(ROOT, "build", "gdx")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
CU_FLAGS = ARCH + COMMON + ["-Xcompiler", "-fPIC,-ffp-contract=off", "--expt-relaxed-constexpr",
                            "-Xptxas", "-v"] if os.environ.get("GDX_PTXAS_V") else \
    ARCH + COMMON + ["-Xcompiler", "-fPIC,-ffp-contract=off", "--expt-relaxed-constexpr"]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off",
             "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include"]

SOURCES_CU = ["aggregate.cu", "gemm_tcgen05.cu", "dense_ops.cu", "sampling.cu"]
SOURCES_CXX = ["host.cpp"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, "gdx_common.cuh"), os.path.join(ROOT, "include", "gdx.h")]
    objs = []
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        if force or _stale(o, [s] + headers):
            cmd = [NVCC] + CU_FLAGS + ["-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
        objs.append(o)
    for src in SOURCES_CXX:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        if force or _stale(o, [s] + headers):
            cmd = ["g++"] + CXX_FLAGS + ["-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
        objs.append(o)
    if force or _stale(OUT, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", OUT] + objs + ["-Xcompiler", "-fopenmp", "-lgomp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
