"""Kernel-level parity of the CUDA hot path against the CPU oracle, through the C ABI.

Pins mirror the reference's own kernel tests:
SparseStack structure (test_sketch.cpp:27-98), sketch_apply vs S A
(test_sketch.cpp:126-147), Householder R (test_matrix_core.cpp:192-201),
SVD conventions (:203-301), precond_apply (test_precond.cpp:57-105).
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _rand(rng, m, n):
    return rng.standard_normal((m, n))


# ---------------------------------------------------------------- sketch (K1)
@pytest.mark.parametrize("d,m,zeta,seed", [(8, 3, 4, 11), (6, 5, 1, 3), (16, 7, 16, 5), (32, 9, 4, 1234),
                                           (4000, 100_000, 4, 7), (2000, 5_000, 4, 2**63 + 5)])
def test_sparsestack_bit_exact(msvd, cuda, port, d, m, zeta, seed):
    import torch

    pos = torch.empty(m * zeta, dtype=torch.int32, device=cuda)
    sgn = torch.empty(m * zeta, dtype=torch.int8, device=cuda)
    ctx = msvd.default_context()
    msvd.check(msvd.lib().msvd_build_sparsestack(ctx.handle, d, m, zeta, seed, _ptr(pos), _ptr(sgn)))
    p_ref, s_ref = port.build_sparsestack(d, m, zeta, seed)
    assert np.array_equal(pos.cpu().numpy().astype(np.uint32), p_ref)
    assert np.array_equal(sgn.cpu().numpy(), s_ref)


def test_sparsestack_validation(msvd, cuda):
    ctx = msvd.default_context()
    L = msvd.lib()
    for args in [(0, 5, 4), (8, 0, 4), (8, 5, 0), (8, 5, 9), (30, 5, 4)]:
        rc = L.msvd_build_sparsestack(ctx.handle, args[0], args[1], args[2], 1, None, None)
        assert rc == 1, args  # DimensionError


@pytest.mark.parametrize("m,n,d,zeta,ld_pad", [(10_000, 100, 200, 4, 0), (5_000, 37, 148, 4, 0),
                                               (3_000, 64, 64, 1, 0), (4_000, 50, 200, 4, 3),
                                               (20_000, 1000, 4000, 4, 0), (1_000, 1, 8, 2, 0)])
def test_sketch_bit_exact(msvd, cuda, port, m, n, d, zeta, ld_pad):
    """One rank: SA is bit-identical to sketch_apply(S, A) (sketch.cpp:75-95)."""
    import torch

    rng = np.random.default_rng(m + n)
    a = _rand(rng, m, n)
    a[rng.random((m, n)) < 0.01] = 0.0  # exact zeros are skipped by the reference
    dev = torch.zeros((m, n + ld_pad), dtype=torch.float64, device=cuda)
    dev[:, :n] = torch.from_numpy(a).to(cuda)
    op = msvd.DeviceDenseOperator(dev[:, :n] if ld_pad == 0 else dev.narrow(1, 0, n))
    sa = torch.empty((n, d), dtype=torch.float64, device=cuda)  # column-major d x n
    msvd.check(msvd.lib().msvd_sketch(op.handle, d, zeta, 99, _ptr(sa)))
    want = port.sketch_apply(a, d, zeta, 99)
    got = sa.cpu().numpy().T
    assert np.array_equal(got, want)


def test_sketch_rejects_nonfinite(msvd, cuda):
    import torch

    a = torch.randn(500, 20, dtype=torch.float64, device=cuda)
    a[17, 3] = float("nan")
    op = msvd.DeviceDenseOperator(a)
    sa = torch.empty((20, 80), dtype=torch.float64, device=cuda)
    with pytest.raises(msvd.NumericalError):
        msvd.check(msvd.lib().msvd_sketch(op.handle, 80, 4, 1, _ptr(sa)))


def test_sketch_overflow_is_not_a_nonfinite_a(msvd, cuda, port):
    """Finite entries whose sums overflow are not an error of A (the check is
    on A's elements, operator.cpp:33-35): SA carries the infinities, the same
    ones sketch_apply computes."""
    import torch

    rng = np.random.default_rng(5)
    a = rng.choice([-1.0, 1.0], size=(4000, 70)) * 1.5e308
    dev = torch.from_numpy(a).to(cuda)
    op = msvd.DeviceDenseOperator(dev)
    sa = torch.empty((70, 100), dtype=torch.float64, device=cuda)
    msvd.check(msvd.lib().msvd_sketch(op.handle, 100, 4, 3, _ptr(sa)))
    got = sa.cpu().numpy().T
    with np.errstate(over="ignore", invalid="ignore"):
        want = port.sketch_apply(a, 100, 4, 3)
    assert not np.all(np.isfinite(want))
    assert np.array_equal(got, want, equal_nan=True)


@pytest.mark.parametrize("env", [{}, {"MSVD_SKETCH_GATHER": "1"}])
def test_sketch_variants_bit_exact(msvd, cuda, port, env, monkeypatch):
    """The slice gather (entry batches, a ragged tail per list) and the
    one-launch gather: the same bits."""
    import torch

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(11)
    m, n, d = 30_000, 150, 600
    a = _rand(rng, m, n)
    dev = torch.from_numpy(a).to(cuda)
    op = msvd.DeviceDenseOperator(dev)
    sa = torch.empty((n, d), dtype=torch.float64, device=cuda)
    msvd.check(msvd.lib().msvd_sketch(op.handle, d, 4, 99, _ptr(sa)))
    assert np.array_equal(sa.cpu().numpy().T, port.sketch_apply(a, d, 4, 99))


# ------------------------------------------------------- A passes (K2 / K3)
@pytest.mark.parametrize("m,n,b", [(1, 1, 1), (7, 3, 1), (1000, 100, 1), (4097, 257, 3), (20_000, 1000, 2),
                                   (10_000, 2000, 5), (12_345, 500, 4), (3000, 2048, 8), (50, 1999, 6)])
def test_apply_and_adjoint(msvd, cuda, m, n, b):
    import torch

    g = torch.Generator(device=cuda).manual_seed(m * 31 + n)
    a = torch.randn(m, n, dtype=torch.float64, device=cuda, generator=g)
    x = torch.randn(n, b, dtype=torch.float64, device=cuda, generator=g)
    y = torch.randn(m, b, dtype=torch.float64, device=cuda, generator=g)
    op = msvd.DeviceDenseOperator(a)
    ax = op.apply_block(x)
    aty = op.apply_adjoint_block(y)
    ref_ax = a @ x
    ref_aty = a.t() @ y
    # fp64 dot products of length n / m: tolerance scaled by sqrt(len) u |a||x|
    tol_ax = 64 * np.sqrt(n) * 2.2e-16 * (a.abs() @ x.abs()).max().item()
    tol_aty = 64 * np.sqrt(m) * 2.2e-16 * (a.abs().t() @ y.abs()).max().item()
    assert (ax - ref_ax).abs().max().item() <= tol_ax
    assert (aty - ref_aty).abs().max().item() <= tol_aty


@pytest.mark.parametrize("m,n,b,kl", [(5000, 100, 1, 2), (20_000, 1000, 1, 2), (20_000, 1000, 2, 4), (9_999, 500, 4, 8),
                                      (4096, 2000, 5, 10), (3000, 64, 1, 0), (100, 7, 2, 0),
                                      # warp-pair one-pass kernel shapes (b * pairs per lane > 16)
                                      (8192, 2000, 1, 2), (10_001, 511, 3, 6), (7777, 999, 2, 0)])
def test_pass_primitives(msvd, cuda, m, n, b, kl):
    """msvd_gram_apply (K2), msvd_aw_tsqr (K3 + TSQR) and msvd_aw_gram (one pass)
    against torch fp64: solver.cpp:357-369/:421 and :412-416."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(m + 7 * n + b)
    a = torch.randn(m, n, dtype=torch.float64, device=cuda, generator=g)
    w = torch.randn(n, b, dtype=torch.float64, device=cuda, generator=g)
    lead = torch.randn(m, kl, dtype=torch.float64, device=cuda, generator=g) if kl else None
    op = msvd.DeviceDenseOperator(a)
    aw_ref = a @ w
    tol_aw = 64 * np.sqrt(n) * 2.2e-16 * (a.abs() @ w.abs()).max().item()
    # K3 + TSQR: AW and the R of [lead | AW] (R^T R is sign-free)
    aw, r = op.aw_tsqr(w, lead)
    assert (aw - aw_ref).abs().max().item() <= tol_aw
    t = torch.cat([lead, aw_ref], dim=1) if kl else aw_ref
    assert torch.allclose(torch.triu(r), r)
    gram = t.t() @ t
    assert (r.t() @ r - gram).abs().max().item() <= 1e-12 * gram.abs().max().item()
    # one pass: AW and A^T A W
    aw2, z = op.aw_gram(w)
    assert (aw2 - aw_ref).abs().max().item() <= tol_aw
    z_ref = a.t() @ aw_ref
    assert (z - z_ref).abs().max().item() <= 64 * np.sqrt(m) * 2.2e-16 * (a.abs().t() @ aw_ref.abs()).max().item()
    # K2: Y = T C, G = A^T Y[:, :b]
    k = kl + b
    cmat = torch.randn(k, 2 * b, dtype=torch.float64, device=cuda, generator=g)
    gg, y = op.gram_apply(t, cmat, b)
    y_ref = t @ cmat
    assert (y - y_ref).abs().max().item() <= 64 * np.sqrt(k) * 2.2e-16 * (t.abs() @ cmat.abs()).max().item()
    g_ref = a.t() @ y_ref[:, :b]
    assert (gg - g_ref).abs().max().item() <= 64 * np.sqrt(m) * 2.2e-16 * (a.abs().t() @ y_ref[:, :b].abs()).max().item()
    gd, none = op.gram_apply(aw_ref)  # direct: G = A^T T
    assert none is None
    assert (gd - z_ref).abs().max().item() <= 64 * np.sqrt(m) * 2.2e-16 * (a.abs().t() @ aw_ref.abs()).max().item()


@pytest.mark.parametrize("pad", [1, 2, 3])
def test_apply_unaligned_rows(msvd, cuda, pad):
    """Odd leading dimensions take the LDG producer path; results are the same."""
    import torch

    m, n, b = 3001, 301, 2
    base = torch.randn(m, n + pad, dtype=torch.float64, device=cuda)
    base[:, n:] = float("nan")  # padding must never be read into results
    a = base[:, :n]
    op = msvd.DeviceDenseOperator(a)
    x = torch.randn(n, b, dtype=torch.float64, device=cuda)
    y = torch.randn(m, b, dtype=torch.float64, device=cuda)
    assert torch.allclose(op.apply_block(x), a @ x, rtol=1e-12, atol=1e-11)
    assert torch.allclose(op.apply_adjoint_block(y), a.t() @ y, rtol=1e-12, atol=1e-10)


def test_adjoint_is_deterministic(msvd, cuda):
    import torch

    a = torch.randn(50_000, 300, dtype=torch.float64, device=cuda)
    y = torch.randn(50_000, 2, dtype=torch.float64, device=cuda)
    op = msvd.DeviceDenseOperator(a)
    r1 = op.apply_adjoint_block(y).clone()
    r2 = op.apply_adjoint_block(y)
    assert torch.equal(r1, r2)


def test_column_norms(msvd, cuda):
    import torch

    a = torch.randn(7777, 123, dtype=torch.float64, device=cuda)
    op = msvd.DeviceDenseOperator(a)
    assert torch.allclose(op.column_norms(), a.norm(dim=0), rtol=1e-13)


# ------------------------------------------------------------- TSQR (K4)
@pytest.mark.parametrize("m,k,scales", [(100, 3, None), (1_000_000, 3, (1e-8, 1.0, 0.3)), (20_000, 15, None),
                                        (5_000, 24, None), (33, 12, None), (200_000, 6, (1e-12, 1e-10, 1, 1, 1, 1))])
def test_tsqr_matches_householder_r(msvd, cuda, port, m, k, scales):
    """R^T R (and |R|) agree with householder_qr's R; columnwise accuracy keeps
    tiny columns exact to their own scale (svd.cpp:21-55)."""
    import torch

    rng = np.random.default_rng(k)
    t = rng.standard_normal((m, k))
    if scales:
        t *= np.asarray(scales)
    dt = torch.from_numpy(np.asfortranarray(t).T.copy()).to(cuda)  # column-major m x k
    r = torch.empty((k, k), dtype=torch.float64, device=cuda)
    msvd.check(msvd.lib().msvd_tsqr_r(msvd.default_context().handle, _ptr(dt), m, k, _ptr(r)))
    got = r.cpu().numpy().T  # column-major -> numpy (k x k)
    want = port.householder_r(t)
    assert np.allclose(np.triu(got), got)
    colscale = np.linalg.norm(t, axis=0)
    err = np.abs(np.abs(got) - np.abs(want)) / colscale[None, :]
    assert err.max() <= 1e-12


@pytest.mark.parametrize("k", [1, 2, 3, 6, 12, 15, 24])
def test_small_svd_conventions(msvd, cuda, port, k):
    import torch

    rng = np.random.default_rng(100 + k)
    bmat = np.triu(rng.standard_normal((k, k))) @ np.diag(np.logspace(0, -12, k))
    db = torch.from_numpy(np.asfortranarray(bmat).T.copy()).to(cuda)
    s = torch.empty(k, dtype=torch.float64, device=cuda)
    v = torch.empty((k, k), dtype=torch.float64, device=cuda)
    msvd.check(msvd.lib().msvd_small_svd(msvd.default_context().handle, _ptr(db), k, _ptr(s), _ptr(v)))
    s_ref, v_ref = port.dense_svd(bmat)
    s_got, v_got = s.cpu().numpy(), v.cpu().numpy().T
    assert np.all(np.diff(s_got) <= 0)
    assert np.allclose(s_got, s_ref, rtol=1e-12, atol=1e-15 * s_ref[0])
    # sign convention: the largest-magnitude entry of each column is positive
    for j in range(k):
        i = np.argmax(np.abs(v_got[:, j]))
        assert v_got[i, j] > 0
    assert np.allclose(v_got.T @ v_got, np.eye(k), atol=1e-13)
    # well-separated values -> identical vectors up to roundoff
    assert np.allclose(v_got, v_ref, atol=1e-8)


# ------------------------------------------------- preconditioner (K5, K7)
@pytest.mark.parametrize("rows,n", [(200, 100), (4000, 1000), (400, 200), (12, 5)])
def test_precond_build_and_apply(msvd, cuda, port, rows, n):
    import torch

    rng = np.random.default_rng(rows)
    sa = rng.standard_normal((rows, n)) @ np.diag(np.logspace(0, -6, n))
    dsa = torch.from_numpy(np.asfortranarray(sa).T.copy()).to(cuda)
    vt = torch.empty((n, n), dtype=torch.float64, device=cuda)
    sig = torch.empty(n, dtype=torch.float64, device=cuda)
    smax, nf = C.c_double(), C.c_int64()
    ctx = msvd.default_context()
    msvd.check(msvd.lib().msvd_precond_build(ctx.handle, _ptr(dsa), rows, n, _ptr(vt), _ptr(sig),
                                             C.byref(smax), C.byref(nf)))
    vt_ref, sig_ref, smax_ref, nf_ref = port.build_preconditioner(sa)
    got_sig = sig.cpu().numpy()
    assert np.allclose(got_sig, sig_ref, rtol=1e-10)
    assert abs(smax.value - smax_ref) <= 1e-13 * smax_ref
    assert nf.value == nf_ref
    got_v = vt.cpu().numpy().T
    assert np.allclose(got_v.T @ got_v, np.eye(n), atol=1e-12)
    assert np.allclose(got_v, vt_ref, atol=1e-7)  # distinct sigmas -> same signed vectors
    # apply: V diag(s^-2) V^T r vs the explicit product (test_precond.cpp:57-76)
    r = rng.standard_normal((n, 3))
    dr = torch.from_numpy(r.T.copy()).to(cuda)
    w = torch.empty((3, n), dtype=torch.float64, device=cuda)
    msvd.check(msvd.lib().msvd_precond_apply(ctx.handle, _ptr(vt), _ptr(sig), n, _ptr(dr), 3, _ptr(w)))
    explicit = (got_v / got_sig[None, :] ** 2) @ got_v.T @ r
    assert np.allclose(w.cpu().numpy().T, explicit, rtol=1e-9, atol=1e-9 * np.abs(explicit).max())
    want = port.precond_apply(got_v, got_sig, r)
    assert np.allclose(w.cpu().numpy().T, want, rtol=1e-9, atol=1e-9 * np.abs(want).max())


@pytest.mark.parametrize("algo", ["eigj", "gesvdj", "gesvd", "polar", "gesvdp"])
def test_precond_floor_and_zero(msvd, cuda, algo, monkeypatch):
    """The floor (precond.cpp:26-34).  An exactly rank-deficient sketch is
    floored by the Jacobi / QR-iteration SVDs and by the default polar SVD
    with its tail refinement; the raw polar SVD resolves tiny values only to
    ~u sigma_1, so there the check is that every value sits at or above the
    floor."""
    import torch

    monkeypatch.setenv("MSVD_SVD", algo)

    rng = np.random.default_rng(9)
    sa = rng.standard_normal((10, 4))
    sa[:, 3] = sa[:, 0]  # exact duplicate column (test_precond.cpp:94-105)
    ctx = msvd.default_context()
    dsa = torch.from_numpy(sa.T.copy()).to(cuda)
    vt = torch.empty((4, 4), dtype=torch.float64, device=cuda)
    sig = torch.empty(4, dtype=torch.float64, device=cuda)
    smax, nf = C.c_double(), C.c_int64()
    msvd.check(msvd.lib().msvd_precond_build(ctx.handle, _ptr(dsa), 10, 4, _ptr(vt), _ptr(sig), C.byref(smax),
                                             C.byref(nf)))
    if algo != "gesvdp":  # raw polar SVD: tiny values only to ~u sigma_1
        assert nf.value >= 1
    assert sig.min().item() >= 2.0 * 2.220446049250313e-16 * smax.value * (1 - 1e-12)
    zero = torch.zeros((3, 6), dtype=torch.float64, device=cuda)
    rc = msvd.lib().msvd_precond_build(ctx.handle, _ptr(zero), 6, 3, _ptr(vt), _ptr(sig), C.byref(smax),
                                       C.byref(nf))
    assert rc == 3  # NumericalError: sketched matrix is exactly zero
    rc = msvd.lib().msvd_precond_build(ctx.handle, _ptr(zero), 2, 3, _ptr(vt), _ptr(sig), C.byref(smax),
                                       C.byref(nf))
    assert rc == 1  # DimensionError: fewer rows than columns
