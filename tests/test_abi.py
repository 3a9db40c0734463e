"""The C-ABI library loads on a CPU-only host and exports every symbol
include/msvd.h declares; host-side logic (defaults, validation order,
row sharding, struct layout) runs without a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2602_16797_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "msvd.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(msvd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(msvd):
    declared = header_functions()
    assert len(declared) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", msvd.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (msvd_\w+)", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    lib = msvd.lib()
    for f in declared:
        assert hasattr(lib, f)
    assert set(msvd.EXPORTED) == set(declared)


def test_abi_struct_sizes_match_ctypes(msvd):
    sizes = (C.c_int64 * 6)()
    msvd.lib().msvd_abi_sizes(sizes, 6)
    assert list(sizes) == [C.sizeof(abi.Options), C.sizeof(abi.RecordRow), C.sizeof(abi.Truth),
                           C.sizeof(abi.Result), C.sizeof(abi.CtxDesc), C.sizeof(abi.LanczosResult)]


def test_defaults_match_solver_options(msvd):
    o = abi.Options()
    msvd.lib().msvd_options_default(C.byref(o))
    d = abi.default_options()
    for name, _ in abi.Options._fields_:
        assert getattr(o, name) == getattr(d, name), name
    py = msvd.SolverOptions().to_abi()
    for name, _ in abi.Options._fields_:
        assert getattr(o, name) == getattr(py, name), name
    assert msvd.lib().msvd_abi_version() == 1
    assert msvd.lib().msvd_default_tolerance(100) == pytest.approx(2 * 10 * 2.220446049250313e-16, rel=0)


@pytest.mark.parametrize("m,n,kw,exc", [
    (3, 5, {}, "DimensionError"),
    (40, 8, dict(block_size=0), "DimensionError"),
    (40, 8, dict(block_size=3), "DimensionError"),
    (40, 8, dict(tol=1.5), "NumericalError"),
    (40, 8, dict(tol=float("nan")), "NumericalError"),
    (40, 8, dict(check_every=0), "NumericalError"),
    (40, 8, dict(sketch_dim=30), "DimensionError"),
    (40, 8, dict(sketch_dim=4), "DimensionError"),
    (40, 8, dict(zeta=0), "DimensionError"),
    (40, 8, dict(sketch_dim=40, zeta=41), "DimensionError"),
    (40, 8, dict(block_size=2, max_iter=-5), None),
    (20, 8, dict(zeta=0), None),            # m <= 4n: sketch skipped, zeta unused
    (10**6, 1000, {}, None),
    (10**6, 4096, {}, None),                # wide A: column panels (the paper's 2e6 x 4e3 example)
    (2**22, 2**20 + 2, {}, "DimensionError"),  # this build: n <= 2^20
    (10**6, 1000, dict(block_size=9), "DimensionError"),  # this build: b <= 8
])
def test_validation_order_and_classes(msvd, m, n, kw, exc):
    """solver.cpp:306-315, prepare() :128-145, build_sparsestack :36-41."""
    opts = msvd.SolverOptions(**kw)
    if exc is None:
        msvd.validate_options(m, n, opts)
    else:
        with pytest.raises(getattr(msvd, exc)):
            msvd.validate_options(m, n, opts)


def test_error_messages_name_the_reference_checks(msvd):
    with pytest.raises(msvd.DimensionError, match="round_up_to_multiple"):
        msvd.validate_options(40, 8, msvd.SolverOptions(sketch_dim=30))
    with pytest.raises(msvd.NumericalError, match=r"tol must lie in \[0, 1\)"):
        msvd.validate_options(40, 8, msvd.SolverOptions(tol=1.0))
    assert msvd.lib().msvd_status_name(1) == b"DimensionError"
    assert msvd.lib().msvd_status_name(3) == b"NumericalError"


@pytest.mark.parametrize("m,p", [(10, 3), (1_000_000, 8), (8_000_000, 7), (5, 8), (0, 2)])
def test_shard_rows_partition(msvd, m, p):
    spans = [msvd.shard_rows(m, p, r) for r in range(p)]
    assert spans[0][0] == 0
    for (a0, ar), (b0, _) in zip(spans, spans[1:]):
        assert a0 + ar == b0
    assert spans[-1][0] + spans[-1][1] == m
    sizes = [r for _, r in spans]
    assert max(sizes) - min(sizes) <= 1


def test_no_gpu_calls_fail_loudly(msvd):
    """Without a device the context cannot be created, and the error says so
    (the product never falls back to a CPU path)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(msvd.Error):
        msvd.Context(0)


def test_product_does_not_import_the_oracle():
    """Only tests/, smoke() and bench.py may touch oracle/."""
    pkg = os.path.join(ROOT, "paper_2602_16797_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f), errors="replace").read()
                assert "pyoracle" not in text and "liboracle" not in text and "minsvd_ref" not in text, f
