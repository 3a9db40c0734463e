"""Device Golub-Kahan-Lanczos baseline (msvd_lanczos_gk) against the CPU oracle.

baselines.cpp:51-166 as the compare client runs it (cli.cpp:356-362): start
vector = sketch_and_solve_init of the randomized run's preconditioner.  Gates:
every record row's Ritz value within 1e-10 sigma_max of the oracle's, the
same step count and exit status, and the final Ritz vector within a 1e-8
subspace angle where the smallest Ritz value has separated (the reference's
own tolerances, BASELINE.json north_star).
"""
import json
import os
import threading

import numpy as np
import pytest

from paper_2602_16797_b200 import problems

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
SIGMA_TOL = 1e-10
ANGLE_TOL = 1e-8


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs])


def sin_angle(a, b):
    a = a / np.linalg.norm(a)
    b = b / np.linalg.norm(b)
    return np.linalg.norm(a - b * (b @ a))


def to_device(a_colmajor, cuda):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a_colmajor)).to(cuda)


def golden_problem(port, name):
    case = GOLDEN["lanczos"][name]
    sig = problems.spectrum(case["recipe"], case["n"])
    a, vmin = port.synth_dense(sig, case["m"], problems.DATA_SEED)
    return case, sig, a, vmin


def assert_lanczos_parity(res, ref, scale, vec=True):
    assert res.steps == ref["steps"]
    assert res.status == ref["status"]
    assert len(res.record.rows) == len(ref["record"])
    for g, r in zip(res.record.rows, ref["record"]):
        assert (g.iter, g.matvecs_a, g.matvecs_at) == (r["iter"], r["matvecs_a"], r["matvecs_at"])
        assert abs(g.theta - r["theta"]) <= SIGMA_TOL * scale, (g.iter, g.theta, r["theta"])
    assert abs(res.sigma_min - ref["sigma_min"]) <= SIGMA_TOL * scale
    if vec:
        assert sin_angle(ref["v"], res.v) <= ANGLE_TOL


@pytest.mark.parametrize("name", sorted(GOLDEN["lanczos"]))
def test_lanczos_golden_parity(msvd, cuda, port, name):
    """The committed reference runs (c1 full: n steps to an invariant
    subspace; c2 recipe 20000 x 200, 60 steps)."""
    case, sig, a, vmin = golden_problem(port, name)
    v0 = unhex(case["v0"])
    op = msvd.DeviceDenseOperator(to_device(a, cuda))
    res = msvd.lanczos_gk(op, case["iters"], v0, msvd.GroundTruth(sig[-1], vmin), record_timing=False)
    ref = dict(steps=case["steps"], status=case["status"], sigma_min=float.fromhex(case["sigma_min"]),
               v=unhex(case["v"]),
               record=[dict(iter=r[0], matvecs_a=r[1], matvecs_at=r[2], theta=float.fromhex(r[3]))
                       for r in case["record"]])
    assert_lanczos_parity(res, ref, scale=sig[0])
    # truth columns: relerr of the final row
    last = res.record.rows[-1]
    assert abs(last.relerr - float.fromhex(case["record"][-1][5])) <= SIGMA_TOL * sig[0] / sig[-1]


def test_lanczos_compare_flow_reduced_c2(msvd, cuda, port):
    """compare's chain on the device: rlobpcg's preconditioner seeds the
    Krylov run (cli.cpp:356-360); 120 steps on the c2 recipe at 1e5 x 400."""
    cfg = problems.CONFIGS["c2"].scaled(m=100_000, n=400)
    sig = cfg.spectrum()
    a_dev, vmin = problems.make_problem_gpu(cfg.m, cfg.n, sig, device=cuda)
    op = msvd.DeviceDenseOperator(a_dev)
    opts = msvd.SolverOptions(seed=problems.SOLVER_SEED, sketch_dim=cfg.d, tol=cfg.tol, use_stagnation=False,
                              record_timing=False)
    pre = msvd.lobpcg_solve(op, msvd.PrecondKind.randomized, opts, want_precond=True)
    v0 = msvd.sketch_and_solve_init(pre.precond, 1)[:, 0]
    res = msvd.lanczos_gk(op, 120, v0, msvd.GroundTruth(sig[-1], vmin), record_timing=False)
    a_host = a_dev.cpu().numpy()
    ref = port.lanczos_gk(a_host, 120, v0, truth=(sig[-1], vmin))
    assert_lanczos_parity(res, ref, scale=sig[0])


def test_lanczos_bases_and_recurrence(msvd, cuda, port):
    """Both bases orthonormal, and A V_j = U_j B_j (the bidiagonal section)."""
    rng = np.random.default_rng(2)
    m, n, iters = 3000, 64, 40
    q = np.linalg.qr(rng.standard_normal((m, n)))[0]
    a = q @ np.diag(np.logspace(0, -4, n)) @ np.linalg.qr(rng.standard_normal((n, n)))[0].T
    op = msvd.DeviceDenseOperator(to_device(a, cuda))
    v0 = rng.standard_normal(n)
    res = msvd.lanczos_gk(op, iters, v0, record_timing=False, want_bases=True)
    vb, ub = res.v_basis, res.u_basis
    assert vb.shape == (n, iters) and ub.shape == (m, iters)
    assert np.linalg.norm(vb.T @ vb - np.eye(iters)) <= 1e-12
    assert np.linalg.norm(ub.T @ ub - np.eye(iters)) <= 1e-12
    b = ub.T @ (a @ vb)  # upper bidiagonal up to roundoff
    assert np.linalg.norm(np.tril(b, -1)) <= 1e-12 and np.linalg.norm(np.triu(b, 2)) <= 1e-12
    ref = port.lanczos_gk(a, iters, v0)
    assert abs(res.sigma_min - ref["sigma_min"]) <= SIGMA_TOL


def test_lanczos_invariant_start_and_errors(msvd, cuda):
    """baselines.cpp:75-80 (exact null start) and :53-61 (errors)."""
    rng = np.random.default_rng(4)
    a = rng.standard_normal((500, 12))
    a[:, 5] = 0.0
    op = msvd.DeviceDenseOperator(to_device(a, cuda))
    e = np.zeros(12)
    e[5] = 1.0
    r = msvd.lanczos_gk(op, 6, e)
    assert r.status == msvd.LanczosStatus.invariant_subspace and r.steps == 0 and r.sigma_min == 0.0
    assert np.array_equal(r.v, e) and not r.record.rows
    with pytest.raises(msvd.DimensionError):
        msvd.lanczos_gk(op, 0, np.ones(12))
    with pytest.raises(msvd.DimensionError):
        msvd.lanczos_gk(op, 13, np.ones(12))
    with pytest.raises(msvd.NumericalError):
        msvd.lanczos_gk(op, 3, np.zeros(12))
    with pytest.raises(msvd.DimensionError):
        msvd.lanczos_gk(op, 3, np.ones(11))


def test_lanczos_fake_group_two_ranks(msvd, cuda, port):
    """Row-sharded run (2 ranks on one GPU, host-mediated reductions): the
    same record as one rank to the parity gates."""
    import torch

    case, sig, a, vmin = golden_problem(port, "lz_c2s")
    dev = to_device(a, cuda)
    v0 = unhex(case["v0"])
    one = msvd.lanczos_gk(msvd.DeviceDenseOperator(dev), case["iters"], v0, record_timing=False)
    nr = 2
    grp = msvd.FakeGroup(nr)
    out = [None] * nr
    errs = []

    def run(r):
        try:
            torch.cuda.set_device(0)
            ctx = grp.context(r)
            r0, rows = msvd.shard_rows(case["m"], nr, r)
            op = msvd.DeviceDenseOperator(dev[r0:r0 + rows], ctx=ctx, row0=r0, m_global=case["m"])
            out[r] = msvd.lanczos_gk(op, case["iters"], v0, record_timing=False)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(nr)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errs, errs
    ref = dict(steps=one.steps, status=one.status, sigma_min=one.sigma_min, v=one.v,
               record=[dict(iter=x.iter, matvecs_a=x.matvecs_a, matvecs_at=x.matvecs_at, theta=x.theta)
                       for x in one.record.rows])
    for r in range(nr):
        assert_lanczos_parity(out[r], ref, scale=sig[0])
    grp.close()
