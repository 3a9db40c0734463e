"""The Cholesky-QR preconditioner route (csrc/precond_chol.cu) against the
SVD route (csrc/svd.cu, MSVD_PRECOND=svd) on the same bytes.

Without flooring (precond.cpp:26-34), Vt diag(sigma~^-2) Vt^T = (SA^T SA)^-1
= R^-1 R^-T exactly, so both routes apply the same preconditioner; sigma~_1
and the start block V0 (precond.cpp:50-57) come from block iterations
instead of the full SVD.  Gates: the same answer to the north-star
tolerances, sigma~_1 to 1e-13, iterations within one.  Where the floor
fires (C3's exact nullspace) the route must refuse and the SVD route runs."""
import numpy as np
import pytest

from _parity import subspace_sin
from paper_2602_16797_b200 import problems

@pytest.mark.gpu
@pytest.mark.parametrize("name,shape", [("c2", dict(m=60_000, n=1000)), ("c4", dict(m=60_000, n=500)),
                                        ("c5", dict(m=60_000, n=1000)), ("c1", dict(m=10_000, n=100))])
def test_cholesky_route_matches_svd_route(msvd, cuda, name, shape, monkeypatch):
    cfg = problems.CONFIGS[name].scaled(**shape)
    a_dev, _ = problems.make_problem_gpu(cfg.m, cfg.n, cfg.spectrum(), device=cuda)
    opts = msvd.SolverOptions(seed=problems.SOLVER_SEED, sketch_dim=cfg.d, tol=cfg.tol, block_size=cfg.b,
                              use_stagnation=False, record_timing=False)
    op = msvd.DeviceDenseOperator(a_dev)
    op.ctx.kernel_paths(reset=True)
    fast = msvd.rlobpcg_block(op, opts)
    taken = "chol_precond" in op.ctx.kernel_paths()
    # b = 1 and well-separated blocks take the route; C5's clustered tail
    # (sigma_{n-1} / sigma_{n-2} = 0.99) would need too many block-inverse
    # rounds for V0, so the route refuses early and the SVD route runs
    assert taken or name == "c5"
    monkeypatch.setenv("MSVD_PRECOND", "svd")
    slow = msvd.rlobpcg_block(op, opts)
    assert "chol_precond" not in op.ctx.kernel_paths()
    smax = slow.sigma_max_estimate
    print(f"[{name}] chol route: {fast.iterations()} it, {fast.timings_ms['svd']:.2f} ms set-up factorization; "
          f"svd route: {slow.iterations()} it, {slow.timings_ms['svd']:.2f} ms")
    assert abs(fast.sigma_max_estimate - smax) <= 1e-13 * smax
    assert np.all(np.abs(fast.sigma - slow.sigma) <= 1e-10 * smax)
    assert subspace_sin(slow.v[:, 0], fast.v[:, 0]) <= 1e-8
    assert abs(fast.iterations() - slow.iterations()) <= 1
    assert fast.status == slow.status or abs(fast.iterations() - slow.iterations()) == 1


@pytest.mark.gpu
def test_cholesky_route_refuses_floored_sketch(msvd, cuda):
    """C3's five exact zeros: sigma~ reaches the floor, so the SVD route runs
    (floor_count 5, as the reference)."""
    cfg = problems.CONFIGS["c3"].scaled(m=20_000, n=300)
    a_dev, _ = problems.make_problem_gpu(cfg.m, cfg.n, cfg.spectrum(), device=cuda)
    opts = msvd.SolverOptions(seed=problems.SOLVER_SEED, sketch_dim=cfg.d, tol=cfg.tol, block_size=cfg.b,
                              use_stagnation=False, record_timing=False)
    op = msvd.DeviceDenseOperator(a_dev)
    op.ctx.kernel_paths(reset=True)
    res = msvd.rlobpcg_block(op, opts, want_precond=False)
    assert "chol_precond" not in op.ctx.kernel_paths()
    assert res.precond.floor_count == 5 and res.precond.floored


def test_preconditioner_apply_equals_inverse_gram(port):
    """What the route relies on: with no floor, the reference's
    Vt diag(sigma~^-2) Vt^T r equals (SA^T SA)^-1 r (oracle, fp64)."""
    cfg = problems.CONFIGS["c2"].scaled(m=4_000, n=120)
    a, _ = port.synth_dense(cfg.spectrum(), cfg.m, problems.DATA_SEED)
    sa = port.sketch_apply(a, cfg.d, 4, problems.SOLVER_SEED)
    vt, sig, smax, nfloor = port.build_preconditioner(sa)
    assert nfloor == 0
    r = np.random.default_rng(3).standard_normal(cfg.n)
    w_ref = port.precond_apply(vt, sig, r)[:, 0]
    # R^-1 R^-T r with the R of a Householder QR of SA (kappa(R) u accurate;
    # solving with SA^T SA itself would lose kappa^2 u = 1e-4 here)
    rr = np.linalg.qr(sa, mode="r")
    w_qr = np.linalg.solve(rr, np.linalg.solve(rr.T, r))
    assert np.linalg.norm(w_ref - w_qr) <= 1e-8 * np.linalg.norm(w_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("name,shape", [("c4", dict(m=60_000, n=500)), ("c5", dict(m=60_000, n=1000)),
                                        ("c3", dict(m=20_000, n=300))])
def test_trial_block_cholqr_matches_tsqr(msvd, cuda, name, shape, monkeypatch):
    """The R factor of the trial block [AV AX AW] from Cholesky QR2
    (csrc/trial_qr.cu, b >= 2 on one rank) against the Householder TSQR
    (MSVD_TRIAL_QR=householder): the same Rayleigh-Ritz answers.  Where the
    block is too ill-conditioned (C3's exact nullspace, C5's 1e-7) the device
    flag sends those iterations down the TSQR path on its own."""
    cfg = problems.CONFIGS[name].scaled(**shape)
    a_dev, _ = problems.make_problem_gpu(cfg.m, cfg.n, cfg.spectrum(), device=cuda)
    opts = msvd.SolverOptions(seed=problems.SOLVER_SEED, sketch_dim=cfg.d, tol=cfg.tol, block_size=cfg.b,
                              use_stagnation=False, record_timing=False)
    op = msvd.DeviceDenseOperator(a_dev)
    monkeypatch.setenv("MSVD_TRIAL_QR", "cholqr")  # default only for b >= 3 (api.cu use_cholqr_req)
    fast = msvd.rlobpcg_block(op, opts)
    monkeypatch.setenv("MSVD_TRIAL_QR", "householder")
    ref = msvd.rlobpcg_block(op, opts)
    smax = ref.sigma_max_estimate
    print(f"[{name}] cholqr2 {fast.iterations()} it {fast.timings_ms['loop']:.2f} ms loop; "
          f"householder {ref.iterations()} it {ref.timings_ms['loop']:.2f} ms loop")
    assert np.all(np.abs(fast.sigma - ref.sigma) <= 1e-10 * smax)
    # C3: the five zero singular values make single vectors of the nullspace
    # arbitrary; only the 5-D subspace is defined
    gate = [0] if name == "c5" else ([] if name == "c3" else list(range(cfg.b)))
    for j in gate:
        assert subspace_sin(ref.v[:, j], fast.v[:, j]) <= 1e-8
    if name != "c5":
        assert subspace_sin(ref.v, fast.v) <= 1e-8
    assert abs(fast.iterations() - ref.iterations()) <= 1
