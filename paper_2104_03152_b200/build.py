"""Build the C-ABI shared library libhe_ckks.so in-tree for sm_100a.

    python -m paper_2104_03152_b200.build [--force]

nvcc compiles the CUDA translation units for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo (so ncu's source page maps to the code); g++ compiles the host
parameter code (needs libquadmath for the binary128 CDT table).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
# HE_LIB_OUT: build an experiment variant elsewhere (with HE_NVCC_EXTRA flags); the product is LIB
LIB = os.environ.get("HE_LIB_OUT") or os.path.join(HERE, "libhe_ckks.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU = ["he_ops.cu", "he_capi.cu"]
CPP = ["he_host.cpp"]
HEADERS = ["he_common.cuh", "he_ntt.cuh", "he_jobs.cuh", "he_internal.cuh", "he_ops.h", "he_host.h"]


def _sources():
    return ([os.path.join(CSRC, f) for f in CU + CPP + HEADERS]
            + [os.path.join(ROOT, "include", "he_ckks.h")])


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd[:3]) + " ...")
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build" if LIB.endswith("/libhe_ckks.so") and os.path.dirname(LIB) == HERE
                          else "build_" + os.path.basename(LIB).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    from concurrent.futures import ThreadPoolExecutor

    def cu(f):
        o = os.path.join(objdir, f + ".o")
        extra = os.environ.get("HE_NVCC_EXTRA", "").split()   # experiments only (e.g. -DHE_NTT32_MINB=2)
        out = _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-Xptxas", "-v" if verbose else "-O3", "--expt-relaxed-constexpr", *extra,
                    "-I", CSRC, "-c", os.path.join(CSRC, f), "-o", o])
        if verbose:
            sys.stderr.write(out)
        return o

    def cpp(f):
        o = os.path.join(objdir, f + ".o")
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-c", os.path.join(CSRC, f), "-o", o])
        return o

    with ThreadPoolExecutor(max_workers=4) as ex:
        futs = [ex.submit(cu, f) for f in CU] + [ex.submit(cpp, f) for f in CPP]
        objs = [f.result() for f in futs]
    tmp = LIB + f".tmp{os.getpid()}"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lquadmath", "-lcudart"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
