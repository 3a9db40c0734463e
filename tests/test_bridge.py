"""The device path behind the reference's own C++ types
(include/minsvd_bridge.hpp, paper_2602_16797_b200/bridge/minsvd_bridge.cpp):
compiled here against /root/reference/proj/include and the reference library
(oracle/Makefile `bridge`), run on the GPU (tests/cpp/test_bridge.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "test_bridge")
REF_INCLUDE = "/root/reference/proj/include"


def build(msvd):
    if os.path.isdir(REF_INCLUDE):
        from oracle import pyoracle

        pyoracle.build("ref")
        r = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "bridge"], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return EXE


def test_bridge_compiles_against_reference_headers(msvd):
    if not os.path.isdir(REF_INCLUDE):
        pytest.skip("reference headers absent (GPU box): the bridge is prebuilt")
    exe = build(msvd)
    assert os.path.exists(exe)
    # the adapter is a minsvd::LinearOperator: its vtable and the gpu_* entry
    # points are in the binary, next to the reference's own solver
    out = subprocess.run(["nm", "-C", exe], capture_output=True, text=True).stdout
    assert "minsvd::DeviceDenseOperatorAdapter::apply_block" in out
    assert "minsvd::gpu_lobpcg_solve" in out


@pytest.mark.gpu
def test_bridge_runs_on_device(msvd, cuda):
    exe = build(msvd)
    if not os.path.exists(exe):
        pytest.fail("oracle/_ref/test_bridge missing: build() compiles it where the reference headers exist")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bridge: OK" in r.stdout
