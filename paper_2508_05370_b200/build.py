"""Builds libhsim.so (the C-ABI library, include/hsim.h) in-tree with nvcc for sm_100a.

Flags that matter for exactness (DESIGN.md C.0): device ``-fmad=false`` (no
FMA contraction) and IEEE division (nvcc default ``-prec-div=true``, never
``--use_fast_math``); host ``-ffp-contract=off``.
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhsim.so")
SOURCES = [os.path.join(CSRC, f) for f in ("host.cu", "kernels.cu", "flow.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "hsim_core.cuh"), os.path.join(ROOT, "include", "hsim.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nvcc_cmd(out=LIB, extra=()):
    return [NVCC, "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
            "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
            "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
            "-I", os.path.join(ROOT, "include"), *extra, *SOURCES, "-o", out]


def build(force=False, verbose=False):
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return LIB
    cmd = nvcc_cmd(extra=("-Xptxas", "-v") if verbose else ())
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
