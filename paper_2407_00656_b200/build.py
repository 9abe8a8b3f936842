"""Build libhgks.so (CUDA sm_100a + host C++) in-tree with nvcc.

No CPU fallback exists: the product path needs this library and a B200.
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libhgks.so")
SOURCES = [os.path.join(PKG, "csrc", "solver.cu"), os.path.join(PKG, "csrc", "setup.cpp")]
DEPS = SOURCES + [os.path.join(PKG, "csrc", "kernels.cuh"), os.path.join(PKG, "csrc", "hot.cuh"),
                  os.path.join(PKG, "csrc", "common.cuh"), os.path.join(PKG, "csrc", "erfc_fit.h"),
                  os.path.join(PKG, "csrc", "moments_gen.cuh"), os.path.join(PKG, "csrc", "internal.h"),
                  os.path.join(ROOT, "include", "hgks.h")]

NVCC_FLAGS = ["-O3", "-std=c++17", "--split-compile=0", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC,-fopenmp,-O2", "-shared"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        nvcc = os.environ.get("NVCC", "nvcc")
        cmd = [nvcc, *NVCC_FLAGS, "-o", LIB + ".tmp", *SOURCES, "-ldl", "-lgomp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
