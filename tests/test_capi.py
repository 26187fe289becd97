"""The boundary is a plain C ABI: a C99 program (examples/acc_reduce.c) compiles against include/ipm.h with
-pedantic -Werror (CPU) and, on a GPU, links libipm.so and reproduces closed forms without Python or torch."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA_INC = "/usr/local/cuda/include"


def _compile(out):
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Werror", "-pedantic", "-I", os.path.join(ROOT, "include"),
           "-isystem", CUDA_INC, os.path.join(ROOT, "examples", "acc_reduce.c"), "-o", out,
           "-L", os.path.join(ROOT, "paper_1412_1127_b200"), "-l:libipm.so",
           f"-Wl,-rpath,{os.path.join(ROOT, 'paper_1412_1127_b200')}", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_header_is_c99_and_example_links(tmp_path):
    from tools import build
    build.build_ipm()
    _compile(str(tmp_path / "acc_reduce"))


@pytest.mark.gpu
def test_c_program_on_gpu(tmp_path):
    exe = str(tmp_path / "acc_reduce")
    _compile(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "acc_reduce: ok" in r.stdout
