"""Device CSR operator (msvd_csr_attach; operator.hpp:58-74 CsrOperator)
against the CPU oracle.

Bit-exact: the CSR sketch (sketch.cpp:97-118) and the column norms
(operator.cpp:98-104).  Within the north-star gates: products, full solves
(|dsigma| <= 1e-10 sigma_max, subspace angle <= 1e-8, iterations +-1), the
Lanczos baseline over a CSR operator.  Validation errors carry the
reference's class and message (csr.cpp:9-31).
"""
import json
import os
import threading

import numpy as np
import pytest

from paper_2602_16797_b200 import abi, problems

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
SIGMA_TOL = 1e-10
ANGLE_TOL = 1e-8


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs])


def subspace_sin(v_ref, v_got):
    v_ref = np.asarray(v_ref).reshape(v_ref.shape[0], -1)
    v_got = np.asarray(v_got).reshape(v_got.shape[0], -1)
    return np.linalg.norm(v_ref - v_got @ (v_got.T @ v_ref), 2)


def device_csr(msvd, cuda, a, index_bytes=8, **kw):
    import torch

    rp, ci, v, m, n = a
    return msvd.DeviceCsrOperator(torch.as_tensor(rp, device=cuda),
                                  torch.as_tensor(ci, device=cuda).to(torch.int64 if index_bytes == 8 else torch.int32),
                                  torch.as_tensor(v, device=cuda), n, **kw)


def golden_csr(name):
    case = GOLDEN["csr"][name]
    rp, ci, v = problems.random_csr(case["m"], case["n"], case["density"], case["seed"])
    return case, (rp, ci, v, case["m"], case["n"])


@pytest.mark.parametrize("name", sorted(GOLDEN["csr"]))
@pytest.mark.parametrize("index_bytes", [8, 4])
def test_csr_golden_solve(msvd, cuda, name, index_bytes):
    """The reference's CsrOperator solves (tol-only), from the committed
    goldens; int64 and int32 column indices give the same answer."""
    case, a = golden_csr(name)
    op = device_csr(msvd, cuda, a, index_bytes)
    opts = msvd.SolverOptions(seed=GOLDEN["solver_seed"], sketch_dim=case["d"], tol=case["tol"],
                              block_size=case["b"], use_stagnation=False, record_timing=False)
    res = msvd.rlobpcg_block(op, opts)
    smax = float.fromhex(case["sigma_max_estimate"])
    assert abs(res.sigma_max_estimate - smax) <= 1e-12 * smax
    sig = unhex(case["sigma"])
    assert np.all(np.abs(res.sigma - sig) <= SIGMA_TOL * smax), (res.sigma, sig)
    vref = unhex(case["v"]).reshape(case["n"], case["b"], order="F")
    assert subspace_sin(vref, res.v) <= ANGLE_TOL
    assert abs(res.iterations() - case["iterations"]) <= 1
    assert res.status == case["status"]


@pytest.mark.parametrize("name", sorted(GOLDEN["csr"]))
def test_csr_sketch_and_norms_bit_exact(msvd, cuda, name):
    import torch

    case, a = golden_csr(name)
    op = device_csr(msvd, cuda, a)
    n, d = case["n"], case["d"]
    sa = torch.empty((n, d), dtype=torch.float64, device=cuda)  # column-major d x n
    msvd.check(msvd.lib().msvd_sketch(op.handle, d, 4, GOLDEN["solver_seed"], sa.data_ptr()))
    sa = sa.cpu().numpy().T
    import hashlib

    assert hashlib.sha256(np.asfortranarray(sa).tobytes(order="F")).hexdigest() == case["sketch_sha256"]
    norms = op.column_norms().cpu().numpy()
    assert np.array_equal(norms, unhex(case["column_norms"]))


def test_csr_products_match_oracle(msvd, cuda, port):
    """csr.cpp:33-57 at 1e-15-level (different summation order), b = 1..8."""
    rp, ci, v = problems.random_csr(20_000, 300, 0.05, 21)
    a = (rp, ci, v, 20_000, 300)
    op = device_csr(msvd, cuda, a)
    rng = np.random.default_rng(1)
    for b in (1, 3, 8):
        x = rng.standard_normal((300, b))
        y = rng.standard_normal((20_000, b))
        got_y = op.apply_block(x).cpu().numpy()
        got_x = op.apply_adjoint_block(y).cpu().numpy()
        for c in range(b):
            ry, rx, _ = port.csr_products(a, x[:, c], y[:, c])
            assert np.max(np.abs(got_y[:, c] - ry)) <= 1e-13 * np.max(np.abs(ry))
            assert np.max(np.abs(got_x[:, c] - rx)) <= 1e-13 * np.max(np.abs(rx))
    # the adjoint is a deterministic gather: same bits on a repeat
    y = rng.standard_normal((20_000, 2))
    assert np.array_equal(op.apply_adjoint_block(y).cpu().numpy(), op.apply_adjoint_block(y).cpu().numpy())
    # to_dense round trip
    dense = op.to_dense().cpu().numpy()
    assert np.array_equal(dense @ x[:, :1], dense @ x[:, :1])
    assert np.max(np.abs(dense @ x[:, 0] - port.csr_products(a, x[:, 0])[0])) <= 1e-13


def test_csr_solver_variants_match_oracle(msvd, cuda, port):
    """Preconditioner kinds, block mode, the sketch-skip path (m <= 4n) and
    the primitives over a CSR operator."""
    import torch

    rp, ci, v = problems.random_csr(12_000, 100, 0.06, 31)
    a = (rp, ci, v, 12_000, 100)
    op = device_csr(msvd, cuda, a)
    for kind, b in ((abi.PRECOND_RANDOMIZED, 1), (abi.PRECOND_RANDOMIZED, 2), (abi.PRECOND_NONE, 1),
                    (abi.PRECOND_DIAGONAL, 1)):
        opts = msvd.SolverOptions(seed=9, sketch_dim=400, tol=1e-10, block_size=b, use_stagnation=False,
                                  record_timing=False, max_iter=60)
        res = msvd.lobpcg_solve(op, kind, opts)
        ref = port.lobpcg_solve_csr(a, opts.to_abi(kind))
        smax = ref["sigma_max_estimate"]
        assert np.all(np.abs(res.sigma - ref["sigma"]) <= SIGMA_TOL * smax), (kind, b)
        assert abs(res.iterations() - ref["iterations"]) <= 1, (kind, b)
        if ref["status"] == "converged":
            assert subspace_sin(ref["v"], res.v) <= ANGLE_TOL, (kind, b)
    sq = (rp[:301], ci[:rp[300]], v[:rp[300]], 300, 100)  # m = 300 <= 4n: sketch skipped
    ops = device_csr(msvd, cuda, sq)
    opts = msvd.SolverOptions(seed=2, tol=1e-12, use_stagnation=False, record_timing=False)
    res = msvd.rlobpcg_single(ops, opts)
    ref = port.lobpcg_solve_csr(sq, opts.to_abi())
    assert res.sketch_skipped and ref["sketch_skipped"]
    assert abs(res.sigma[0] - ref["sigma"][0]) <= SIGMA_TOL * ref["sigma_max_estimate"]
    assert abs(res.iterations() - ref["iterations"]) <= 1
    # primitives: K2 gram apply and the A*W + TSQR pass
    t = torch.randn(12_000, 3, dtype=torch.float64, device="cuda:0")
    g, _ = op.gram_apply(t[:, :1])
    ref_g = port.csr_products(a, None, t[:, 0].cpu().numpy())[1]
    assert np.max(np.abs(g[:, 0].cpu().numpy() - ref_g)) <= 1e-13 * np.max(np.abs(ref_g))
    w = torch.randn(100, 1, dtype=torch.float64, device="cuda:0")
    aw, r = op.aw_tsqr(w, lead=t[:, :2])
    blk = torch.cat([t[:, :2], aw], dim=1).cpu().numpy()
    rr = np.linalg.qr(blk, mode="r")
    assert np.allclose(np.abs(np.diag(r.cpu().numpy())), np.abs(np.diag(rr)), rtol=1e-12)


def test_csr_lanczos(msvd, cuda, port):
    """baselines.cpp:51-166 over the CSR operator (the golden Krylov runs)."""
    for name in sorted(GOLDEN["csr"]):
        case, a = golden_csr(name)
        op = device_csr(msvd, cuda, a)
        lz = case["lanczos"]
        res = msvd.lanczos_gk(op, lz["iters"], np.ones(case["n"]), record_timing=False)
        theta = unhex(lz["theta"])
        scale = float.fromhex(case["sigma_max_estimate"])
        assert res.steps == lz["steps"] and res.status == lz["status"]
        assert np.max(np.abs(np.array([r.theta for r in res.record.rows]) - theta)) <= SIGMA_TOL * scale


def test_csr_validation_errors(msvd, cuda):
    """csr.cpp:9-31 classes and messages."""
    rp = np.array([0, 2, 3, 5], dtype=np.int64)
    ci = np.array([0, 2, 1, 0, 3], dtype=np.int64)
    v = np.array([1.0, 2.0, 3.0, 4.0, 5.0])
    cases = [
        ((np.array([1, 2, 3, 5]), ci, v), msvd.DimensionError, "endpoints"),
        ((np.array([0, 2, 1, 5]), ci, v), msvd.DimensionError, "nondecreasing at row 1"),
        ((rp, np.array([0, 2, 1, 0, 4]), v), msvd.DimensionError, "out of range in row 2"),
        ((rp, np.array([2, 0, 1, 0, 3]), v), msvd.DimensionError, "strictly increasing in row 0"),
        ((rp, ci, np.array([1.0, np.inf, 3.0, 4.0, 5.0])), msvd.NumericalError, "non-finite"),
    ]
    for (r, c, vv), exc, msg in cases:
        with pytest.raises(exc) as e:
            device_csr(msvd, cuda, (r, c, vv, 3, 4))
        assert msg in str(e.value), (msg, e.value)
    ok = device_csr(msvd, cuda, (rp, ci, v, 3, 4))
    assert ok.nnz() == 5


def test_csr_fake_group_two_ranks(msvd, cuda, port):
    """Row-sharded CSR solve (2 ranks on one GPU): each rank attaches its own
    rows (local offsets); the sketch keys stay global."""
    import torch

    case, a = golden_csr("csr_s")
    rp, ci, v, m, n = a
    opts = msvd.SolverOptions(seed=GOLDEN["solver_seed"], sketch_dim=case["d"], tol=case["tol"],
                              use_stagnation=False, record_timing=False)
    one = msvd.rlobpcg_single(device_csr(msvd, cuda, a), opts)
    nr = 2
    grp = msvd.FakeGroup(nr)
    out = [None] * nr
    errs = []

    def run(r):
        try:
            torch.cuda.set_device(0)
            ctx = grp.context(r)
            r0, rows = msvd.shard_rows(m, nr, r)
            lrp = rp[r0:r0 + rows + 1] - rp[r0]
            sub = (lrp, ci[rp[r0]:rp[r0 + rows]], v[rp[r0]:rp[r0 + rows]], rows, n)
            op = device_csr(msvd, cuda, sub, ctx=ctx, row0=r0, m_global=m)
            out[r] = msvd.rlobpcg_single(op, opts)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(nr)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errs, errs
    for r in range(nr):
        assert out[r].record.to_csv() == out[0].record.to_csv()
        assert abs(out[r].iterations() - one.iterations()) <= 1
        assert abs(out[r].sigma[0] - one.sigma[0]) <= SIGMA_TOL * one.sigma_max_estimate
        assert subspace_sin(one.v, out[r].v) <= ANGLE_TOL
    grp.close()
