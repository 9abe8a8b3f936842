"""Build libhgks.so (CUDA sm_100a + host C++) in-tree with nvcc.

No CPU fallback exists: the product path needs this library and a B200.
"""
from __future__ import annotations

import os
import re
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


# nvcc --split-compile is not deterministic: the same sources give different SASS from build to
# build, and the fp64 tet reconstruction comes out either with a 32-byte stack frame (0.40 ms on
# C2) or with 56 / 64 bytes of spills (0.43 ms; profiles/r02/README.md, code-generation draws).
# A fresh build therefore compiles up to HGKS_BUILD_DRAWS times and keeps the draw whose
# k_recon<14, 4, 6> spills least.
RECON_KERNEL = "_ZN4hgks3p647k_reconILi14ELi4ELi6EEEvNS0_9ReconArgsE"


def recon_stack(path: str) -> int:
    """Stack frame (bytes) of the fp64 tet reconstruction kernel in a built library."""
    try:
        out = subprocess.run(["cuobjdump", "--dump-resource-usage", path], capture_output=True, text=True).stdout
    except OSError:
        return 0
    lines = out.splitlines()
    for i, line in enumerate(lines):
        if RECON_KERNEL in line and i + 1 < len(lines):
            m = re.search(r"STACK:(\d+)", lines[i + 1])
            return int(m.group(1)) if m else 0
    return 0


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        nvcc = os.environ.get("NVCC", "nvcc")
        draws = max(1, int(os.environ.get("HGKS_BUILD_DRAWS", "2")))
        best = None
        for k in range(draws):
            tmp = f"{LIB}.tmp{k}"
            cmd = [nvcc, *NVCC_FLAGS, "-o", tmp, *SOURCES, "-ldl", "-lgomp"]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
            st = recon_stack(tmp)
            if verbose:
                print(f"draw {k}: k_recon<14, 4, 6> stack {st} B", flush=True)
            if best is None or st < best[0]:
                if best is not None:
                    os.remove(best[1])
                best = (st, tmp)
            else:
                os.remove(tmp)
            if st <= 32:
                break
        os.replace(best[1], LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
