"""The CPU oracle is pinned before it is trusted (CPU-only tests).

1. The C restatement (oracle/minsvd_oracle.c, "port") is BIT-IDENTICAL to the
   reference itself (oracle/_ref, minsvd compiled from its own sources) on
   every routine of the hot path, when the reference library is available.
2. The port reproduces the committed golden vectors (tests/golden/golden.json,
   generated from the reference by tests/golden/make_golden.py) exactly.
3. The reference's own property pins for the sketch and the stopping rule
   (test_sketch.cpp:27-147, test_solver.cpp:84-145) hold for the port.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2602_16797_b200 import abi, problems

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs])


def sha(a):
    return hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).hexdigest()


def matrix(port, case):
    sig = problems.spectrum(case["recipe"], case["n"])
    if np.all(sig > 0):
        a, vmin = port.synth_dense(sig, case["m"], GOLDEN["data_seed"])
    else:
        a, vmin = port.assemble_svd(sig, case["m"], GOLDEN["data_seed"])
    return sig, a, vmin


# ------------------------------------------------------------- rng.hpp
@pytest.mark.parametrize("kind", ["u64", "below", "unit", "gauss"])
@pytest.mark.parametrize("seed,key", [(0, None), (7, 3), (2**64 - 1, 2**63), (123456789, None)])
def test_splitmix_bit_exact(port, ref, kind, seed, key):
    a = port.splitmix_draws(seed, key=key, kind=kind, count=257, bound=1000)
    b = ref.splitmix_draws(seed, key=key, kind=kind, count=257, bound=1000)
    assert np.array_equal(a, b)


def test_splitmix_golden(port):
    g = GOLDEN["splitmix"]
    assert [int(x) for x in port.splitmix_draws(7, key=3, kind="u64", count=8)] == g["u64_keyed_7_3"]
    assert [int(x) for x in port.splitmix_draws(42, kind="below", count=8, bound=1000)] == g["below_1000_seed42"]
    assert np.array_equal(port.splitmix_draws(5, kind="gauss", count=8), unhex(g["gauss_seed5"]))


# ------------------------------------------------------------- sketch.cpp
@pytest.mark.parametrize("d,m,zeta,seed", [(8, 3, 4, 11), (6, 5, 1, 3), (16, 7, 16, 5), (4000, 5000, 4, 7),
                                           (12, 6, 3, 77), (2, 1000, 2, 2**63)])
def test_sparsestack_bit_exact(port, ref, d, m, zeta, seed):
    p1, s1 = port.build_sparsestack(d, m, zeta, seed)
    p2, s2 = ref.build_sparsestack(d, m, zeta, seed)
    assert np.array_equal(p1, p2) and np.array_equal(s1, s2)


def test_sparsestack_structure(port):
    """test_sketch.cpp:27-98: one entry per block, |value| = zeta^-1/2,
    determinism, prefix (order-free) property."""
    d, m, zeta = 32, 9, 4
    pos, sgn = port.build_sparsestack(d, m, zeta, 1234)
    assert np.all(pos < d // zeta) and set(np.unique(sgn)) <= {-1, 1}
    wide_p, wide_s = port.build_sparsestack(d, 20, zeta, 1234)
    assert np.array_equal(wide_p[: m * zeta], pos) and np.array_equal(wide_s[: m * zeta], sgn)
    other, _ = port.build_sparsestack(d, m, zeta, 1235)
    assert not np.array_equal(other, pos)
    g = GOLDEN["sketch"]["stack"]
    p, s = port.build_sparsestack(g["d"], g["m"], g["zeta"], g["seed"])
    assert hashlib.sha256(p.tobytes()).hexdigest() == g["positions_sha256"]
    assert hashlib.sha256(s.tobytes()).hexdigest() == g["signs_sha256"]


def test_sketch_matches_dense_product(port):
    """test_sketch.cpp:126-147: sketch_apply equals S A within 1e-15 max."""
    d, m, zeta = 20, 50, 4
    rng = np.random.default_rng(9)
    a = rng.standard_normal((m, 4))
    pos, sgn = port.build_sparsestack(d, m, zeta, 8)
    s = np.zeros((d, m))
    for j in range(m):
        for k in range(zeta):
            s[k * (d // zeta) + pos[j * zeta + k], j] = sgn[j * zeta + k] / np.sqrt(zeta)
    want = s @ a
    got = port.sketch_apply(a, d, zeta, 8)
    assert np.max(np.abs(got - want)) <= 1e-15 * np.max(np.abs(want))


def test_sketch_bit_exact_and_golden(port, ref):
    g = GOLDEN["sketch"]["c1_sa"]
    sig, a, _ = matrix(port, GOLDEN["cases"]["c1"])
    sa = port.sketch_apply(a, g["d"], g["zeta"], g["seed"])
    assert sha(sa) == g["sha256"]
    assert np.array_equal(sa, ref.sketch_apply(a, g["d"], g["zeta"], g["seed"]))


def test_sketch_row_sharded_sum(port):
    """The sharded sketch (global row keys) sums to the full sketch."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((1001, 17))
    full = port.sketch_apply(a, 68, 4, 5)
    parts = sum(port.sketch_apply(a[r0:r1], 68, 4, 5, row0=r0) for r0, r1 in [(0, 333), (333, 700), (700, 1001)])
    assert np.allclose(parts, full, rtol=0, atol=1e-13 * np.abs(full).max())


# ---------------------------------------------------------- svd.cpp, precond.cpp
@pytest.mark.parametrize("m,k", [(100, 3), (2000, 15), (50, 50), (400, 24)])
def test_householder_and_svd_bit_exact(port, ref, m, k):
    rng = np.random.default_rng(m + k)
    a = rng.standard_normal((m, k)) @ np.diag(np.logspace(0, -10, k))
    assert np.array_equal(port.householder_r(a), ref.householder_r(a))
    s1, v1 = port.dense_svd(a)
    s2, v2 = ref.dense_svd(a)
    assert np.array_equal(s1, s2) and np.array_equal(v1, v2)


def test_preconditioner_bit_exact(port, ref):
    rng = np.random.default_rng(4)
    sa = rng.standard_normal((80, 20)) @ np.diag(np.logspace(0, -5, 20))
    sa[:, 19] = sa[:, 0]  # rank deficient -> floored
    p1 = port.build_preconditioner(sa)
    p2 = ref.build_preconditioner(sa)
    for x, y in zip(p1, p2):
        assert np.array_equal(x, y)
    assert p1[3] >= 1
    r = rng.standard_normal((20, 3))
    assert np.array_equal(port.precond_apply(p1[0], p1[1], r), ref.precond_apply(p2[0], p2[1], r))


def test_cgs2_bit_exact(port, ref):
    rng = np.random.default_rng(5)
    basis = np.linalg.qr(rng.standard_normal((60, 4)))[0]
    w = rng.standard_normal((60, 3))
    w[:, 1] = basis[:, 0]  # degenerate column -> seeded Gaussian replacement
    w1, r1 = port.cgs2(w, basis, 19)
    w2, r2 = ref.cgs2(w, basis, 19)
    assert r1 == r2 == 1
    assert np.array_equal(w1, w2)


# ---------------------------------------------------------- stopping rule
def test_stopping_logic_synthetic_histories(port, ref):
    """test_solver.cpp:84-145"""
    for o in (port, ref):
        resid = [1e-8 * 0.5 ** j for j in range(12)]
        theta = [1.0 + 0.25 ** j for j in range(12)]
        d = o.check_convergence(resid, theta, 10, 1.0, 1e-10, 1.1, True)
        assert d["tol_ok"] and not d["resid_stalled"] and not d["stop"]
        flat_r, flat_t = [1e-20] * 12, [1.0] * 12
        d10 = o.check_convergence(flat_r, flat_t, 10, 1.0, 1e-10, 1.1, True)
        assert d10["tol_ok"] and d10["resid_stalled"] and d10["progress_stalled"] and d10["stop"]
        d5 = o.check_convergence(flat_r, flat_t, 5, 1.0, 1e-10, 1.1, True)
        assert d5["resid_stalled"] and not d5["progress_stalled"] and not d5["stop"]
        assert not o.check_convergence(flat_r, flat_t, 0, 1.0, 1e-10, 1.1, True)["stop"]
        assert not o.check_convergence([1e-3] * 12, [1.0] * 12, 10, 1.0, 1e-10, 1.1, True)["stop"]
        assert o.check_convergence(flat_r, [0.0] * 12, 10, 1.0, 1e-10, 1.1, True)["stop"]
        assert o.check_convergence([1e-3, 1e-20], [1.0, 1.0], 0, 1.0, 1e-10, 1.1, False)["stop"]
        with pytest.raises(Exception):
            o.check_convergence([1.0, 0.5], [1.0, 1.0], 5, 1.0, 1e-10, 1.1, True)


# ------------------------------------------------------------ full solves
@pytest.mark.parametrize("name", sorted(GOLDEN["cases"]))
def test_port_reproduces_golden(port, name):
    case = GOLDEN["cases"][name]
    sig, a, vmin = matrix(port, case)
    assert sha(a) == case["a_sha256"], "input regeneration drifted"
    opts = abi.default_options(seed=GOLDEN["solver_seed"], sketch_dim=case["d"], tol=case["tol"],
                               block_size=case["b"], use_stagnation=int(case["use_stagnation"]), record_timing=0)
    r = port.lobpcg_solve(a, opts, truth=(sig[-1], vmin))
    assert r["iterations"] == case["iterations"] and r["status"] == case["status"]
    assert np.array_equal(r["sigma"], unhex(case["sigma"]))
    assert np.array_equal(r["v"].ravel(order="F"), unhex(case["v"]))
    assert float(r["sigma_max_estimate"]).hex() == case["sigma_max_estimate"]
    rec = [[x["iter"], x["matvecs_a"], x["matvecs_at"], float(x["theta"]).hex(), float(x["resid"]).hex(),
            float(x["relerr"]).hex(), float(x["sin_angle"]).hex()] for x in r["record"]]
    assert rec == case["record"]


def test_port_equals_reference_solver_variants(port, ref):
    """Options the goldens do not cover: block kinds, verification, iterates,
    sketch skip, explicit d > m."""
    rng = np.random.default_rng(11)
    q = np.linalg.qr(rng.standard_normal((300, 30)))[0]
    a = q @ np.diag(np.logspace(0, -6, 30)) @ np.linalg.qr(rng.standard_normal((30, 30)))[0].T
    variants = [
        dict(seed=5, max_iter=40, record_timing=0),
        dict(seed=5, max_iter=37, tol=0.0, record_timing=0, verify_cached_products=1),
        dict(seed=5, block_size=3, max_iter=30, record_timing=0, store_iterates=1),
        dict(seed=2, sketch_dim=512, record_timing=0),
        dict(seed=3, precond_kind=abi.PRECOND_NONE, max_iter=50, record_timing=0),
        dict(seed=3, precond_kind=abi.PRECOND_DIAGONAL, max_iter=50, record_timing=0),
    ]
    for kw in variants:
        r1 = port.lobpcg_solve(a, abi.default_options(**kw), want_precond=True, want_iterates=True)
        r2 = ref.lobpcg_solve(a, abi.default_options(**kw), want_precond=True, want_iterates=True)
        for key in ("sigma", "v", "vtilde", "sigma_tilde"):
            assert np.array_equal(r1[key], r2[key]), (kw, key)
        for key in ("iterations", "status", "record", "verify_count", "max_cache_drift", "degenerate_replacements",
                    "floor_count", "sketch_dim", "sketch_skipped"):
            assert r1[key] == r2[key], (kw, key)
        assert len(r1["trail_t"]) == len(r2["trail_t"])
        for (i1, t1), (i2, t2) in zip(r1["trail_t"], r2["trail_t"]):
            assert i1 == i2 and np.array_equal(t1, t2)
    skip = port.lobpcg_solve(a[:100], abi.default_options(seed=2))
    assert skip["sketch_skipped"] and skip["sketch_dim"] == 0


def test_port_validation_errors(port, ref):
    """test_solver.cpp:446-477 error classes (msvd_status codes)."""
    from oracle.pyoracle import OracleError

    rng = np.random.default_rng(17)
    a = rng.standard_normal((40, 8))
    bad = [(np.zeros((3, 5)), {}, abi.MSVD_ERR_DIMENSION), (a, dict(block_size=3), abi.MSVD_ERR_DIMENSION),
           (a, dict(tol=1.5), abi.MSVD_ERR_NUMERICAL), (a, dict(check_every=0), abi.MSVD_ERR_NUMERICAL),
           (a, dict(sketch_dim=30), abi.MSVD_ERR_DIMENSION), (a, dict(sketch_dim=4), abi.MSVD_ERR_DIMENSION)]
    for o in (port, ref):
        for mat, kw, code in bad:
            with pytest.raises(OracleError) as e:
                o.lobpcg_solve(mat, abi.default_options(**kw))
            assert e.value.code == code, (kw, e.value)
        nan = a.copy()
        nan[3, 2] = np.nan
        with pytest.raises(OracleError) as e:
            o.lobpcg_solve(nan, abi.default_options())
        assert e.value.code == abi.MSVD_ERR_NUMERICAL


# ------------------------------------------------- lanczos_gk (baselines)
def lanczos_rows(r):
    return [[x["iter"], x["matvecs_a"], x["matvecs_at"], float(x["theta"]).hex(), float(x["resid"]).hex(),
             float(x["relerr"]).hex(), float(x["sin_angle"]).hex()] for x in r["record"]]


@pytest.mark.parametrize("name", sorted(GOLDEN["lanczos"]))
def test_port_reproduces_lanczos_golden(port, name):
    case = GOLDEN["lanczos"][name]
    sig, a, vmin = matrix(port, case)
    assert sha(a) == case["a_sha256"], "input regeneration drifted"
    r = port.lanczos_gk(a, case["iters"], unhex(case["v0"]), truth=(sig[-1], vmin))
    assert r["steps"] == case["steps"] and r["status"] == case["status"]
    assert float(r["sigma_min"]).hex() == case["sigma_min"]
    assert np.array_equal(r["v"], unhex(case["v"]))
    assert lanczos_rows(r) == case["record"]


def test_lanczos_port_equals_reference(port, ref):
    """Step counts, early exits and both bases, bit for bit."""
    rng = np.random.default_rng(5)
    q = np.linalg.qr(rng.standard_normal((200, 24)))[0]
    a = q @ np.diag(np.logspace(0, -5, 24)) @ np.linalg.qr(rng.standard_normal((24, 24)))[0].T
    v0 = rng.standard_normal(24)
    for iters in (1, 2, 7, 24):
        r1 = port.lanczos_gk(a, iters, v0, want_bases=True)
        r2 = ref.lanczos_gk(a, iters, v0, want_bases=True)
        for key in ("steps", "status", "record"):
            assert r1[key] == r2[key], (iters, key)
        for key in ("v", "v_basis", "u_basis"):
            assert np.array_equal(r1[key], r2[key]), (iters, key)
        assert r1["sigma_min"] == r2["sigma_min"]
    # exact null start: A v0 = 0 -> invariant subspace before any step
    z = a.copy()
    z[:, 3] = 0.0
    e = np.zeros(24)
    e[3] = 1.0
    for o in (port, ref):
        r = o.lanczos_gk(z, 5, e)
        assert r["status"] == "invariant_subspace" and r["steps"] == 0 and r["sigma_min"] == 0.0
        assert np.array_equal(r["v"], e)


def test_lanczos_validation_errors(port, ref):
    """baselines.cpp:53-61 error classes."""
    from oracle.pyoracle import OracleError

    rng = np.random.default_rng(3)
    a = rng.standard_normal((30, 6))
    cases = [(a, 0, np.ones(6), abi.MSVD_ERR_DIMENSION), (a, 7, np.ones(6), abi.MSVD_ERR_DIMENSION),
             (a, 3, np.zeros(6), abi.MSVD_ERR_NUMERICAL), (a[:4], 2, np.ones(6), abi.MSVD_ERR_DIMENSION)]
    for o in (port, ref):
        for mat, iters, v0, code in cases:
            with pytest.raises(OracleError) as e:
                o.lanczos_gk(mat, iters, v0)
            assert e.value.code == code, (iters, e.value)


# ------------------------------------------- CSR operator (csr.cpp, sketch.cpp:97-118)
def csr_case(case):
    rp, ci, v = problems.random_csr(case["m"], case["n"], case["density"], case["seed"])
    assert hashlib.sha256(rp.tobytes() + ci.tobytes() + v.tobytes()).hexdigest() == case["csr_sha256"]
    return (rp, ci, v, case["m"], case["n"])


@pytest.mark.parametrize("name", sorted(GOLDEN["csr"]))
def test_port_reproduces_csr_golden(port, name):
    case = GOLDEN["csr"][name]
    a = csr_case(case)
    opts = abi.default_options(seed=GOLDEN["solver_seed"], sketch_dim=case["d"], tol=case["tol"],
                               block_size=case["b"], use_stagnation=0, record_timing=0)
    r = port.lobpcg_solve_csr(a, opts)
    assert r["iterations"] == case["iterations"] and r["status"] == case["status"]
    assert np.array_equal(r["sigma"], unhex(case["sigma"]))
    assert np.array_equal(r["v"].ravel(order="F"), unhex(case["v"]))
    assert [[x["iter"], x["matvecs_a"], x["matvecs_at"], float(x["theta"]).hex(), float(x["resid"]).hex()]
            for x in r["record"]] == case["record"]
    _, _, norms = port.csr_products(a, norms=True)
    assert np.array_equal(norms, unhex(case["column_norms"]))
    sa = port.sketch_csr(a, case["d"], 4, GOLDEN["solver_seed"])
    assert sha(sa) == case["sketch_sha256"]
    lz = port.lanczos_gk_csr(a, case["lanczos"]["iters"], np.ones(case["n"]))
    assert float(lz["sigma_min"]).hex() == case["lanczos"]["sigma_min"]
    assert [float(x["theta"]).hex() for x in lz["record"]] == case["lanczos"]["theta"]


def test_csr_port_equals_reference(port, ref):
    """Products, sketch (sketch.cpp:97-118), every preconditioner kind, the
    sketch-skip path (m <= 4n densifies, solver.cpp:132-134)."""
    rp, ci, v = problems.random_csr(900, 40, 0.15, 5)
    a = (rp, ci, v, 900, 40)
    rng = np.random.default_rng(8)
    x, y = rng.standard_normal(40), rng.standard_normal(900)
    y[::7] = 0.0  # the adjoint skips zero y_i (csr.cpp:51)
    for u, w in zip(port.csr_products(a, x, y, True), ref.csr_products(a, x, y, True)):
        assert np.array_equal(u, w)
    assert np.array_equal(port.sketch_csr(a, 160, 4, 3), ref.sketch_csr(a, 160, 4, 3))
    assert np.array_equal(port.sketch_csr(a, 120, 2, 3), ref.sketch_csr(a, 120, 2, 3))
    for kw in (dict(seed=4, max_iter=30, record_timing=0), dict(seed=4, block_size=2, max_iter=25, record_timing=0),
               dict(seed=4, precond_kind=abi.PRECOND_NONE, max_iter=20, record_timing=0),
               dict(seed=4, precond_kind=abi.PRECOND_DIAGONAL, max_iter=20, record_timing=0)):
        r1 = port.lobpcg_solve_csr(a, abi.default_options(**kw), want_precond=True)
        r2 = ref.lobpcg_solve_csr(a, abi.default_options(**kw), want_precond=True)
        for key in ("sigma", "v", "vtilde", "sigma_tilde"):
            assert np.array_equal(r1[key], r2[key]), (kw, key)
        assert r1["record"] == r2["record"] and r1["iterations"] == r2["iterations"]
    sq = (rp[:151], ci[:rp[150]], v[:rp[150]], 150, 40)  # m = 150 <= 4n: sketch skipped
    r1 = port.lobpcg_solve_csr(sq, abi.default_options(seed=1, max_iter=15, record_timing=0))
    r2 = ref.lobpcg_solve_csr(sq, abi.default_options(seed=1, max_iter=15, record_timing=0))
    assert r1["sketch_skipped"] and r1["record"] == r2["record"] and np.array_equal(r1["v"], r2["v"])


def test_csr_validation_errors(port, ref):
    """csr.cpp:9-31: the same exception class and message, in the same order."""
    from oracle.pyoracle import OracleError

    rp = np.array([0, 2, 3, 5], dtype=np.int64)
    ci = np.array([0, 2, 1, 0, 3], dtype=np.int64)
    v = np.array([1.0, 2.0, 3.0, 4.0, 5.0])
    cases = [
        ((np.array([1, 2, 3, 5]), ci, v), abi.MSVD_ERR_DIMENSION, "endpoints"),
        ((np.array([0, 2, 1, 5]), ci, v), abi.MSVD_ERR_DIMENSION, "nondecreasing at row 1"),
        ((rp, np.array([0, 2, 1, 0, 4]), v), abi.MSVD_ERR_DIMENSION, "out of range in row 2"),
        ((rp, np.array([2, 0, 1, 0, 3]), v), abi.MSVD_ERR_DIMENSION, "strictly increasing in row 0"),
        ((rp, ci, np.array([1.0, np.inf, 3.0, 4.0, 5.0])), abi.MSVD_ERR_NUMERICAL, "non-finite"),
    ]
    for o in (port, ref):
        for (r, c, vv), code, msg in cases:
            with pytest.raises(OracleError) as e:
                o.csr_products((r, c, vv, 3, 4), x=np.ones(4))
            assert e.value.code == code and msg in str(e.value), (o.kind, msg, e.value)
