"""The C++ mirror of the reference API (include/minsvd_gpu.hpp) compiles
against the C ABI (CPU) and passes the reference-style checks on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
OUT = os.path.join(ROOT, "build", "test_cpp_api")


def compile_test(msvd):
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    libdir = os.path.dirname(msvd.LIB_PATH)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", SRC, "-o", OUT, "-L", libdir, "-lmsvd_cuda",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{libdir}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return OUT


def test_cpp_api_compiles(msvd):
    compile_test(msvd)


@pytest.mark.gpu
def test_cpp_api_runs(msvd, cuda):
    exe = compile_test(msvd)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cpp api: OK" in r.stdout
