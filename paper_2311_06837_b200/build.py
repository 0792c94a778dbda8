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

SOURCES_CU = ["aggregate.cu", "gemm_tcgen05.cu", "dense_ops.cu", "sampling.cu", "exchange.cu",
              "cobatch_plan.cu", "trainer.cu", "aggregate_exchange.cu"]
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


API_OUT = os.path.join(HERE, "libgranndis_b200.so")
REF_TESTS = "/root/reference/proj/tests"
SUITE_OUT = os.path.join(ROOT, "build", "ref_suite_b200")


def build_cxx_api(verbose: bool = False, force: bool = False) -> str:
    """libgranndis_b200.so: the reference's C++ API (include/granndis_b200/granndis.hpp)
    over the engine, self-contained (libgdx objects linked in)."""
    build(verbose, force)
    src = os.path.join(CSRC, "granndis_api.cpp")
    obj = os.path.join(OBJ, "granndis_api.o")
    hdr = [os.path.join(ROOT, "include", "granndis_b200", "granndis.hpp"),
           os.path.join(ROOT, "include", "gdx.h")]
    if force or _stale(obj, [src] + hdr):
        cmd = ["g++", "-O2", "-std=c++20", "-fPIC", "-I" + os.path.join(ROOT, "include"),
               "-I/usr/local/cuda/include", "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    objs = [obj] + [os.path.join(OBJ, f + ".o") for f in SOURCES_CU + SOURCES_CXX]
    if force or _stale(API_OUT, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", API_OUT] + objs + ["-Xcompiler", "-fopenmp", "-lgomp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return API_OUT


def build_ref_suite(verbose: bool = False, force: bool = False):
    """Compile the reference's own doctest suites for the hot path (read in place from
    /root/reference, never copied) against libgranndis_b200.so -> build/ref_suite_b200.
    Skipped where /root/reference is absent (the GPU box uses the prebuilt binary)."""
    if not os.path.isdir(REF_TESTS):
        return None
    build_cxx_api(verbose, force)
    srcs = [os.path.join(REF_TESTS, "test_reference_gnn.cpp"), os.path.join(REF_TESTS, "test_extract.cpp"),
            os.path.join(REF_TESTS, "test_batch_plan.cpp"), os.path.join(ROOT, "tests", "cxx", "doctest_main.cpp")]
    if force or _stale(SUITE_OUT, srcs + [API_OUT]):
        cmd = ["g++", "-O2", "-std=c++20", "-I" + os.path.join(ROOT, "tests", "cxx"),
               "-I" + os.path.join(ROOT, "include", "granndis_compat"), "-I" + os.path.join(ROOT, "include"),
               *srcs, "-L" + HERE, "-lgranndis_b200", "-Wl,-rpath,$ORIGIN/../paper_2311_06837_b200",
               "-o", SUITE_OUT]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return SUITE_OUT


CXX_TESTS = {"trainer_epoch": os.path.join(ROOT, "tests", "cxx", "trainer_epoch.cpp")}


def build_cxx_tests(verbose: bool = False, force: bool = False) -> list:
    """C/C++ host programs that drive the engine through include/gdx.h only
    (no Python, no torch) -> build/<name>, linked against the in-tree libgdx.so."""
    build(verbose, force)
    out = []
    for name, src in CXX_TESTS.items():
        exe = os.path.join(ROOT, "build", name)
        if force or _stale(exe, [src, OUT, os.path.join(ROOT, "include", "gdx.h")]):
            cmd = ["g++", "-O2", "-std=c++17", "-I" + os.path.join(ROOT, "include"), src, "-L" + HERE, "-lgdx",
                   "-Wl,-rpath,$ORIGIN/../paper_2311_06837_b200", "-o", exe]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
        out.append(exe)
    return out


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
    build_cxx_api(verbose=True)
    build_ref_suite(verbose=True)
    build_cxx_tests(verbose=True)
