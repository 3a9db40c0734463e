#!/usr/bin/env python
"""Small device solves for compute-sanitizer (memcheck / racecheck / synccheck),
one tool per gpurun call (profiling guide):

    gpurun -- compute-sanitizer --tool racecheck python scripts/sanitize_target.py

Covers the hand-rolled synchronization: the TMA/mbarrier stage rings of the
one-pass passes (b = 1 self-fed + fused TSQR, the warp-pair b = 1 check
refresh), the split-role pass and the trial-block Cholesky QR2 (b = 4),
the ticket pass and the K2 gram pass (b = 5), the Cholesky-QR preconditioner
route and the SVD route, the sketch gather.  Shapes are C1 (BASELINE
configs[0], full size) and scaled C4 / C3 recipes; each solve is checked
against the construction's truth so a silent corruption also fails.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2602_16797_b200 import minsvd as msvd
    from paper_2602_16797_b200 import problems

    dev = torch.device("cuda", 0)
    cases = [("c1", 10_000, 100, {}), ("c2", 12_000, 600, {}), ("c4", 6_000, 500, {}), ("c3", 4_000, 120, {}),
             ("c2", 6_000, 200, {"MSVD_PRECOND": "svd"})]
    for name, m, n, env in cases:
        for k, v in env.items():
            os.environ[k] = v
        cfg = problems.CONFIGS[name].scaled(m=m, n=n)
        sig = cfg.spectrum()
        a, vt = problems.make_problem_gpu(cfg.m, cfg.n, sig, device=dev, tail=cfg.b)
        opts = msvd.SolverOptions(seed=problems.SOLVER_SEED, sketch_dim=cfg.d, tol=cfg.tol, block_size=cfg.b,
                                  use_stagnation=False, record_timing=False)
        op = msvd.DeviceDenseOperator(a)
        op.ctx.kernel_paths(reset=True)
        res = msvd.rlobpcg_block(op, opts)
        paths = sorted(op.ctx.kernel_paths())
        smax = res.sigma_max_estimate
        err = float(np.max(np.abs(res.sigma - sig[::-1][:cfg.b]))) / smax
        print(f"{name} m={m} n={n} b={cfg.b} env={env}: {res.iterations()} it, |dsigma|/smax {err:.2e}, paths {paths}",
              flush=True)
        assert err <= 1e-6, err
        for k in env:
            del os.environ[k]
    torch.cuda.synchronize()
    print("sanitize target: OK")


if __name__ == "__main__":
    main()
