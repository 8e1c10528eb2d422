"""In-tree build of libfuzzyclust_cuda.so (sm_100a) with nvcc.

``--fmad=false`` is part of the numerical contract, not a tuning flag: the
reference is compiled without FMA contraction (proj/CMakeLists.txt:7-9, no
-march), and contracting ``acc + w*x`` into DFMA changes the bits
(SURVEY.md section 0.7).  The host compiler gets ``-ffp-contract=off`` for the
same reason (the few host-side reductions, e.g. ShareMatrix::frob_sq).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.environ.get("FC_LIB") or os.path.join(LIBDIR, "libfuzzyclust_cuda.so")
SOURCES = [os.path.join(CSRC, "fc_capi.cu"), os.path.join(CSRC, "fc_build.cu"), os.path.join(CSRC, "fc_ingest.cu"), os.path.join(CSRC, "fc_refine.cu"), os.path.join(CSRC, "generator.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, "fc_kernels.cuh"), os.path.join(CSRC, "fc_internal.h"),
                  os.path.join(ROOT, "include", "fuzzyclust_cuda.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "--fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
    "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = LIB + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, "-I" + os.path.join(ROOT, "include"), "-o", tmp, *SOURCES, "-lnccl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


DEBUG_LIB = os.path.join(LIBDIR, "libfuzzyclust_cuda_debug.so")


def build_debug(force: bool = False) -> str:
    """The same library with device-side bounds checks on every gathered / scattered row
    index (-DFC_DEBUG_CHECKS: FC_DCHECK in fc_kernels.cuh traps with the location).  Used
    by tests/test_gpu_debug_checks.py in place of compute-sanitizer, which the GPU pool
    does not allow."""
    if not force and os.path.exists(DEBUG_LIB) and all(os.path.getmtime(p) <= os.path.getmtime(DEBUG_LIB)
                                                       for p in DEPS):
        return DEBUG_LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = DEBUG_LIB + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, "-DFC_DEBUG_CHECKS", "-I" + os.path.join(ROOT, "include"), "-o", tmp, *SOURCES,
           "-lnccl"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, DEBUG_LIB)
    return DEBUG_LIB


DROPIN_SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
DROPIN_BIN = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_test")


def build_dropin_test(force: bool = False) -> str:
    """C++ caller of the drop-in headers (include/fuzzyclust/*.hpp) linked to the library."""
    deps = [DROPIN_SRC, LIB] + [os.path.join(ROOT, "include", "fuzzyclust", f)
                                for f in os.listdir(os.path.join(ROOT, "include", "fuzzyclust"))]
    if not force and os.path.exists(DROPIN_BIN) and all(os.path.getmtime(p) <= os.path.getmtime(DROPIN_BIN)
                                                         for p in deps):
        return DROPIN_BIN
    os.makedirs(os.path.dirname(DROPIN_BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.dirname(DROPIN_SRC), DROPIN_SRC, "-L" + LIBDIR, "-lfuzzyclust_cuda",
           "-Wl,-rpath," + LIBDIR, "-o", DROPIN_BIN]
    subprocess.run(cmd, check=True)
    return DROPIN_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))


REF_TESTS = os.environ.get("FC_REF_TESTS", "/root/reference/proj/tests")
REF_SUITES = ("simplex", "objective", "solver", "secondorder", "graph")
SHIM = os.path.join(ROOT, "tests", "cpp", "gtest_shim")


def ref_suite_bin(name: str) -> str:
    return os.path.join(ROOT, "tests", "cpp", "_build", f"ref_{name}_test")


def build_reference_suites(force: bool = False) -> list:
    """The reference's own GTest suites ({simplex,objective,solver,secondorder,graph}_test.cpp
    + support.hpp),
    compiled UNMODIFIED from where they lie under /root/reference against the drop-in
    headers (include/fuzzyclust) and the GoogleTest shim (tests/cpp/gtest_shim), linked to
    the CUDA library.  Nothing is copied into the repo; without /root/reference (the GPU
    box) the binaries built here are used as they are."""
    out = []
    if not os.path.isdir(REF_TESTS):
        return [ref_suite_bin(n) for n in REF_SUITES if os.path.exists(ref_suite_bin(n))]
    hdrs = [os.path.join(ROOT, "include", "fuzzyclust", f) for f in os.listdir(os.path.join(ROOT, "include", "fuzzyclust"))]
    hdrs += [os.path.join(SHIM, "gtest", "gtest.h"), os.path.join(SHIM, "gtest_main.cpp"), LIB]
    os.makedirs(os.path.join(ROOT, "tests", "cpp", "_build"), exist_ok=True)
    for name in REF_SUITES:
        src = os.path.join(REF_TESTS, f"{name}_test.cpp")
        dst = ref_suite_bin(name)
        deps = hdrs + [src, os.path.join(REF_TESTS, "support.hpp")]
        if force or not os.path.exists(dst) or any(os.path.getmtime(d) > os.path.getmtime(dst) for d in deps):
            cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I" + os.path.join(ROOT, "include"), "-I" + SHIM,
                   src, os.path.join(SHIM, "gtest_main.cpp"), "-L" + LIBDIR, "-lfuzzyclust_cuda",
                   "-Wl,-rpath," + LIBDIR, "-lpthread", "-o", dst]
            subprocess.run(cmd, check=True)
        out.append(dst)
    return out
