"""Build an experiment variant of libhgks.so with extra -D flags (A/B runs with HGKS_LIB):
    python scripts/build_variant.py var/libhgks_x.so -DHGKS_POLY_SPLIT=0"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00656_b200 import build as B  # noqa: E402

out, flags = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
cmd = [os.environ.get("NVCC", "nvcc"), *B.NVCC_FLAGS, *flags, "-o", out, *B.SOURCES, "-ldl", "-lgomp"]
print(" ".join(cmd), flush=True)
subprocess.check_call(cmd)
