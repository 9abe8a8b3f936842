"""examples/c_driver.c: a plain C program using only include/hgks.h and libhgks.so
(no Python on the path) builds against the library here; on a GPU it runs 20
steps of a periodic hex box and checks discrete conservation to 1e-12."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_example(tmp_path):
    from paper_2407_00656_b200 import hgks
    hgks.lib()  # make sure libhgks.so exists
    exe = str(tmp_path / "c_driver")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_driver.c"), "-L", os.path.join(ROOT, "paper_2407_00656_b200"), "-lhgks",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{os.path.join(ROOT, 'paper_2407_00656_b200')}",
           "-lm", "-o", exe]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def test_c_example_builds(tmp_path):
    build_example(tmp_path)


@pytest.mark.gpu
def test_c_example_runs(cuda_ok, tmp_path):
    exe = build_example(tmp_path)
    out = subprocess.run([exe, "12"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "-> OK" in out.stdout, out.stdout
