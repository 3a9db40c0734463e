"""Race and ordering stress for the hand-rolled synchronization.

compute-sanitizer is closed on this GPU pool (profiles/round2_compute_sanitizer_closed.txt),
so the TMA/mbarrier stage rings, the per-pair named barriers, the split-role kernel's mbarriers and tickets and the
fixed-order reductions are stressed here instead: every pass variant runs many
times on inputs large enough that each CTA's stage ring wraps hundreds of times
(the mbarrier parity must never run ahead -- the ABA bug fixed in round 1), at
several stage geometries, and must give the SAME BITS every time and agree
with a torch fp64 reference.  A race or a missed barrier shows up as a
run-to-run difference or a wrong value.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPEATS = 12


def _ptr(t):
    import ctypes as C

    return C.c_void_p(t.data_ptr())


@pytest.mark.parametrize("b,n,env", [
    (1, 1000, {}),                                  # apply_self (one-pass, TMA) at C2's n
    (1, 1000, {"MSVD_ROWS_STAGE_KB": "16"}),
    (2, 1000, {}),                                  # split-role one-pass (dot / acc warps)
    (2, 1000, {"MSVD_SPLIT_STAGE_KB": "16"}),
    (4, 500, {}),
    (4, 500, {"MSVD_SPLIT_GROUPS": "4"}),           # four groups (16 warps)
    (4, 500, {"MSVD_SPLIT_STAGE_KB": "16", "MSVD_SPLIT_DEPTH": "2"}),
    (3, 501, {}), (2, 700, {}), (4, 300, {}),
    (1, 2000, {}),                                  # b = 1, wide rows: the warp-pair kernel
])
def test_one_pass_pass_repeatable(msvd, cuda, b, n, env, monkeypatch):
    """msvd_aw_gram: AW = A W and Z = A^T A W from one sweep."""
    import torch

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    m = 300_000 if n <= 600 else 150_000
    ldp = n + (n & 1)  # even leading dimension: the TMA row stream
    g = torch.Generator(device=cuda).manual_seed(n + b)
    full = torch.randn(m, ldp, dtype=torch.float64, device=cuda, generator=g)
    a = full[:, :n]
    w = torch.randn(n, b, dtype=torch.float64, device=cuda, generator=g)
    op = msvd.DeviceDenseOperator(a)
    op.ctx.kernel_paths(reset=True)
    aw0, z0 = op.aw_gram(w)
    paths = op.ctx.kernel_paths()
    for _ in range(REPEATS):
        aw, z = op.aw_gram(w)
        assert torch.equal(aw, aw0) and torch.equal(z, z0), paths
    aw_ref = a @ w
    z_ref = a.t() @ aw_ref
    assert torch.allclose(aw0, aw_ref, rtol=0, atol=1e-10 * aw_ref.abs().max().item())
    assert torch.allclose(z0, z_ref, rtol=0, atol=1e-10 * z_ref.abs().max().item())
    print(f"[b={b} n={n} {env}] paths {sorted(paths)}: {REPEATS + 1} identical runs")


@pytest.mark.parametrize("b,n,env", [
    (1, 1000, {}),                                  # warp-pair EX (b = 1)
    (2, 1000, {}), (3, 501, {}), (4, 500, {}),      # split-role EX
    (2, 130, {}), (4, 120, {}),                     # narrow rows: one column pair per lane
    (4, 500, {"MSVD_SPLIT_STAGE_KB": "16"}),
])
def test_check_refresh_pass_repeatable(msvd, cuda, b, n, env, monkeypatch):
    """msvd_aw_gram_ex: AW = A W, Z = A^T A W and ZE = A^T E from one sweep."""
    import torch

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    m = 200_003 if n <= 600 else 100_001
    ldp = n + (n & 1)  # even leading dimension: the TMA row stream
    g = torch.Generator(device=cuda).manual_seed(7 * n + b)
    full = torch.randn(m, ldp, dtype=torch.float64, device=cuda, generator=g)
    a = full[:, :n]
    w = torch.randn(n, b, dtype=torch.float64, device=cuda, generator=g)
    e = torch.randn(m, b, dtype=torch.float64, device=cuda, generator=g)
    op = msvd.DeviceDenseOperator(a)
    op.ctx.kernel_paths(reset=True)
    aw0, z0, ze0 = op.aw_gram_ex(w, e)
    paths = op.ctx.kernel_paths()
    for _ in range(REPEATS):
        aw, z, ze = op.aw_gram_ex(w, e)
        assert torch.equal(aw, aw0) and torch.equal(z, z0) and torch.equal(ze, ze0), paths
    aw_ref = a @ w
    z_ref = a.t() @ aw_ref
    ze_ref = a.t() @ e
    assert torch.allclose(aw0, aw_ref, rtol=0, atol=1e-10 * aw_ref.abs().max().item())
    assert torch.allclose(z0, z_ref, rtol=0, atol=1e-10 * z_ref.abs().max().item())
    assert torch.allclose(ze0, ze_ref, rtol=0, atol=1e-10 * ze_ref.abs().max().item())
    # the same A W and A^T A W bits as the plain one-pass pass of the same kernel family
    print(f"[check refresh b={b} n={n} {env}] paths {sorted(paths)}: {REPEATS + 1} identical runs")


@pytest.mark.parametrize("m", [1, 7, 150, 1001, 5000])
@pytest.mark.parametrize("b,n", [(4, 500), (2, 1000), (3, 333), (2, 64)])
def test_one_pass_passes_few_rows(msvd, cuda, b, n, m):
    """Fewer rows than CTAs, partial stages, partial row groups: the one-pass pass and
    the check-refresh pass against fp64 torch products."""
    import torch

    ldp = n + (n & 1)
    g = torch.Generator(device=cuda).manual_seed(m + 13 * n + b)
    a = torch.randn(m, ldp, dtype=torch.float64, device=cuda, generator=g)[:, :n]
    w = torch.randn(n, b, dtype=torch.float64, device=cuda, generator=g)
    e = torch.randn(m, b, dtype=torch.float64, device=cuda, generator=g)
    op = msvd.DeviceDenseOperator(a)
    aw, z = op.aw_gram(w)
    try:
        aw2, z2, ze = op.aw_gram_ex(w, e)
    except msvd.Error as ex:  # a one-row view has ld = n: odd n has no TMA row stream, no such pass
        assert m == 1 and n % 2 == 1 and "unsupported shape" in str(ex)
        aw2, z2, ze = aw, z, a.t() @ e
    aw_ref = a @ w
    scale = max(aw_ref.abs().max().item(), 1e-300)
    assert torch.allclose(aw, aw_ref, rtol=0, atol=1e-12 * scale)
    assert torch.allclose(aw2, aw_ref, rtol=0, atol=1e-12 * scale)
    z_ref = a.t() @ aw_ref
    zs = max(z_ref.abs().max().item(), 1e-300)
    assert torch.allclose(z, z_ref, rtol=0, atol=1e-11 * zs)
    assert torch.allclose(z2, z_ref, rtol=0, atol=1e-11 * zs)
    ze_ref = a.t() @ e
    assert torch.allclose(ze, ze_ref, rtol=0, atol=1e-11 * max(ze_ref.abs().max().item(), 1e-300))


@pytest.mark.parametrize("b,n,env", [(1, 1000, {}), (1, 999, {}), (5, 2000, {}), (8, 700, {}),
                                     (1, 1000, {"MSVD_STAGE_KB": "8"})])
def test_apply_and_gram_repeatable(msvd, cuda, b, n, env, monkeypatch):
    """The plain A W pass (producer-warp rows kernel, ticket kernel) and the
    K2 gram pass, odd and even leading dimensions."""
    import torch

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    m = 120_000
    g = torch.Generator(device=cuda).manual_seed(3 * n + b)
    a = torch.randn(m, n, dtype=torch.float64, device=cuda, generator=g)
    w = torch.randn(n, b, dtype=torch.float64, device=cuda, generator=g)
    y = torch.randn(m, b, dtype=torch.float64, device=cuda, generator=g)
    op = msvd.DeviceDenseOperator(a)
    y0 = op.apply_block(w).clone()
    x0 = op.apply_adjoint_block(y).clone()
    for _ in range(REPEATS):
        assert torch.equal(op.apply_block(w), y0)
        assert torch.equal(op.apply_adjoint_block(y), x0)
    assert torch.allclose(y0, a @ w, rtol=0, atol=1e-10 * (a @ w).abs().max().item())
    xr = a.t() @ y
    assert torch.allclose(x0, xr, rtol=0, atol=1e-10 * xr.abs().max().item())


@pytest.mark.parametrize("name,shape", [("c2", dict(m=60_000, n=1000)), ("c5", dict(m=60_000, n=1000)),
                                        ("c4", dict(m=60_000, n=500))])
def test_whole_solve_repeatable(msvd, cuda, name, shape):
    """Complete solves (the one-pass loop with the check refresh -- the
    pair-EX and split-EX passes --, the trial-block QR, the preconditioner
    route): the same record and vectors, bit for bit, on every repeat."""
    from paper_2602_16797_b200 import problems

    cfg = problems.CONFIGS[name].scaled(**shape)
    a, _ = problems.make_problem_gpu(cfg.m, cfg.n, cfg.spectrum(), device=cuda)
    opts = msvd.SolverOptions(seed=problems.SOLVER_SEED, sketch_dim=cfg.d, tol=cfg.tol, block_size=cfg.b,
                              use_stagnation=False, record_timing=False, max_iter=40)
    op = msvd.DeviceDenseOperator(a)
    r0 = msvd.rlobpcg_block(op, opts)
    for _ in range(3):
        r = msvd.rlobpcg_block(op, opts)
        assert r.record.to_csv() == r0.record.to_csv()
        assert np.array_equal(r.v, r0.v) and np.array_equal(r.sigma, r0.sigma)
