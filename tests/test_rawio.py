"""Raw binary A interchange (the binary counterpart of the
reference's Matrix Market array files, io.cpp:174-184): exact round trips,
row-range reads for row-sharded loads, IoError on malformed files
(errors.hpp:21-24).  Host-only entry points: these run on CPU."""
import os

import numpy as np
import pytest


def test_raw_round_trip_bit_exact(msvd, tmp_path):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((257, 19))
    a[5, 7] = np.nextafter(0.0, 1.0)   # subnormal
    a[6, 2] = -0.0
    a[7, 1] = 1e308
    p = tmp_path / "a.raw"
    msvd.raw_write(p, a)
    assert os.path.getsize(p) == 32 + 8 * a.size
    assert msvd.raw_info(p) == (257, 19)
    back = msvd.raw_read(p)
    assert back.tobytes() == a.tobytes()
    # a row range is the matching slice (a rank's shard)
    assert msvd.raw_read(p, 100, 57).tobytes() == a[100:157].tobytes()
    assert msvd.raw_read(p, 257, 0).shape == (0, 19)


def test_raw_strided_write(msvd, tmp_path):
    rng = np.random.default_rng(4)
    big = rng.standard_normal((40, 12))
    view = big[:, :9]  # ld 12 > n 9: rows written without the padding
    p = tmp_path / "v.raw"
    msvd.raw_write(p, view)
    assert np.array_equal(msvd.raw_read(p), view)


def test_raw_errors(msvd, tmp_path):
    with pytest.raises(msvd.IoError, match="cannot open for reading"):
        msvd.raw_info(tmp_path / "missing.raw")
    bad = tmp_path / "bad.raw"
    bad.write_bytes(b"NOTMSVD!" + bytes(24))
    with pytest.raises(msvd.IoError, match="not an MSVDRAW1 file"):
        msvd.raw_info(bad)
    short = tmp_path / "short.raw"
    short.write_bytes(b"MSVD")
    with pytest.raises(msvd.IoError, match="truncated raw header"):
        msvd.raw_info(short)
    p = tmp_path / "t.raw"
    msvd.raw_write(p, np.ones((10, 4)))
    with open(p, "r+b") as f:
        f.truncate(32 + 8 * 39)
    with pytest.raises(msvd.IoError, match="truncated raw data"):
        msvd.raw_read(p)
    msvd.raw_write(p, np.ones((10, 4)))
    with pytest.raises(msvd.DimensionError):
        msvd.raw_read(p, 8, 5)
    with pytest.raises(msvd.IoError, match="cannot open for writing"):
        msvd.raw_write(tmp_path / "no_such_dir" / "x.raw", np.ones((2, 2)))


@pytest.mark.gpu
def test_raw_load_device_and_solve(msvd, cuda, port, tmp_path):
    """A file written from the host loads straight into HBM, in shards, and
    the solve on it equals the in-memory solve bit for bit."""
    import torch

    from paper_2602_16797_b200 import problems

    cfg = problems.CONFIGS["c1"]
    sig = cfg.spectrum()
    a, vmin = port.synth_dense(sig, cfg.m, problems.DATA_SEED)
    a_rm = np.ascontiguousarray(a)
    p = tmp_path / "c1.raw"
    msvd.raw_write(p, a_rm)
    dev = msvd.raw_load_device(p)
    assert torch.equal(dev.cpu(), torch.from_numpy(a_rm))
    half = msvd.raw_load_device(p, 4000, 3000)
    assert torch.equal(half.cpu(), torch.from_numpy(a_rm[4000:7000]))
    opts = msvd.SolverOptions(seed=7, sketch_dim=cfg.d, tol=cfg.tol, use_stagnation=False, record_timing=False)
    r1 = msvd.rlobpcg_single(msvd.DeviceDenseOperator(dev), opts)
    r2 = msvd.rlobpcg_single(msvd.DeviceDenseOperator(torch.from_numpy(a_rm).to(cuda)), opts)
    assert r1.record.to_csv() == r2.record.to_csv() and np.array_equal(r1.v, r2.v)
