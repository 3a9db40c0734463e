"""Row-sharded RLOBPCG protocol on CPU with torch.distributed (gloo, world 2).

The multi-GPU path shards A by contiguous rows and exchanges
exactly: an allreduce of the partial sketches (keyed by GLOBAL row index), an
allgather of per-rank TSQR R factors (merged in rank order), and an allreduce
of the n x b Gram product each iteration.  This test runs that protocol with
the oracle's building blocks on each rank and checks the result against the
unsharded oracle solve -- the same structure the CUDA host loop follows
(paper_2602_16797_b200/csrc/api.cu, solve()).
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def sharded_solve(a_loc, row0, m, cfg, comm, port):
    """solver.cpp:301-477 with the three collectives of the sharded path."""
    import torch

    n, b, d, tol = cfg["n"], cfg["b"], cfg["d"], cfg["tol"]
    eps = np.finfo(np.float64).eps

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x))
        comm.all_reduce(t)
        return t.numpy().reshape(x.shape)

    def tsqr(t):
        r_loc = port.householder_r(t) if t.shape[0] >= t.shape[1] else np.vstack(
            [t, np.zeros((t.shape[1] - t.shape[0], t.shape[1]))])
        parts = [torch.zeros(r_loc.shape, dtype=torch.float64) for _ in range(comm.get_world_size())]
        comm.all_gather(parts, torch.from_numpy(np.ascontiguousarray(r_loc)))
        return port.householder_r(np.vstack([p.numpy() for p in parts]))

    sa = allreduce(port.sketch_apply(a_loc, d, 4, cfg["seed"], row0=row0))
    vt, sig, smax, _ = port.build_preconditioner(sa)
    w = vt[:, n - b:]
    aw = a_loc @ w
    s, c = port.dense_svd(tsqr(aw))
    v, av, theta = w @ c, aw @ c, s
    g = allreduce(a_loc.T @ av)
    r = g - v * theta ** 2
    x = np.zeros((n, 0))
    ax = np.zeros((a_loc.shape[0], 0))
    it = 0
    for i in range(cfg["max_iter"]):
        w = port.precond_apply(vt, sig, r)
        w, _ = port.cgs2(w, np.hstack([v, x]), cfg["seed"])
        t = np.hstack([v, x, w])
        at = np.hstack([av, ax, a_loc @ w])
        k = t.shape[1]
        s, cf = port.dense_svd(tsqr(at))
        c = cf[:, k - b:]
        theta = s[k - b:]
        v_n, av_n = t @ c, at @ c
        g = allreduce(a_loc.T @ av_n)
        r = g - v_n * theta ** 2
        resid = np.max(np.linalg.norm(r, axis=0))
        it = i + 1
        if i % 5 == 0 and resid <= smax * smax * tol:
            v, av = v_n, av_n
            break
        lead = k - b
        q = np.linalg.qr(cf[:b, :lead].T)[0]
        mix = cf[:, :lead] @ q
        x, ax = t @ mix, at @ mix
        v, av = v_n, av_n
    order = np.arange(b)[::-1]
    return theta[order], v[:, order], it, eps


def _worker(rank, world, port_no, q):
    import torch.distributed as dist

    import sys
    sys.path.insert(0, ROOT)
    from oracle import pyoracle
    from paper_2602_16797_b200 import problems

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        port = pyoracle.load("port")
        cfg = dict(n=100, b=1, d=200, tol=1e-12, seed=7, max_iter=200)
        sig = problems.spectrum("c1", 100)
        a, _ = port.synth_dense(sig, 10_000, problems.DATA_SEED)
        m = a.shape[0]
        r0 = (m * rank) // world
        r1 = (m * (rank + 1)) // world
        res = sharded_solve(np.ascontiguousarray(a[r0:r1]), r0, m, cfg, dist, port)
        q.put((rank, res[0], res[1], res[2]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_protocol_matches_oracle(port):
    import torch.multiprocessing as mp

    from paper_2602_16797_b200 import abi, problems

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port_no = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    sig = problems.spectrum("c1", 100)
    a, _ = port.synth_dense(sig, 10_000, problems.DATA_SEED)
    ref = port.lobpcg_solve(a, abi.default_options(seed=7, sketch_dim=200, tol=1e-12, use_stagnation=0))
    smax = ref["sigma_max_estimate"]
    for rank, sigma, v, iters in out:
        # every rank holds identical replicated state
        assert np.array_equal(sigma, out[0][1]) and np.array_equal(v, out[0][2])
        assert abs(iters - ref["iterations"]) <= 1
        assert abs(sigma[0] - ref["sigma"][0]) <= 1e-10 * smax
        vr = ref["v"][:, 0]
        assert np.linalg.norm(vr - v[:, 0] * (v[:, 0] @ vr)) <= 1e-8


# ---------------------------------------------------------------- bench launcher
def test_bench_spawns_ranks_itself():
    """`bench.py --gpus 2` outside torchrun launches two ranks (gloo selftest:
    no GPU needed) and rank 0 prints one line for the whole job."""
    import json
    import subprocess
    import sys

    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--selftest", "--steps", "2",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ranks_reported"] == 2 and d["steps"] == 2 and d["warmup"] == 3
    for key in ("metric", "value", "unit", "ms_per_step", "higher_is_better", "scaling", "config"):
        assert key in d


def test_bench_refuses_missing_gpus():
    """Never a silent downgrade: --gpus 2 without two visible GPUs fails."""
    import subprocess
    import sys

    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode != 0 and "needs 2 GPUs" in (out.stderr + out.stdout)


# ------------------------------------------------- shard-by-shard generator
def _gen_worker(rank, world, port_no, m, n, q):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_2602_16797_b200 import problems

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r0, r1 = (m * rank) // world, (m * (rank + 1)) // world
        a, _ = problems.make_problem_shard(m, n, problems.spectrum("c5", n), r0, r1 - r0,
                                           lambda t: dist.all_reduce(t), device="cpu", block_rows=450)
        q.put((rank, r0, a.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shard_generator_independent_of_rank_count(world):
    """BASELINE configs[4]: U generated and orthonormalised shard by shard
    (two-level TSQR across ranks); the global A is the same for every rank
    count, and U diag(sigma) V^T has the requested spectrum."""
    import torch.multiprocessing as mp

    from paper_2602_16797_b200 import problems

    m, n = 3100, 24  # 6 generator blocks that straddle the rank boundaries
    sig = problems.spectrum("c5", n)
    whole, v = problems.make_problem_shard(m, n, sig, 0, m, None, device="cpu", block_rows=450)
    whole = whole.numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = free_port()
    procs = [ctx.Process(target=_gen_worker, args=(r, world, port_no, m, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    glued = np.vstack([p[2] for p in parts])
    assert glued.shape == (m, n)
    assert np.max(np.abs(glued - whole)) <= 1e-13 * np.max(np.abs(whole))
    s = np.linalg.svd(whole, compute_uv=False)
    assert np.max(np.abs(s - sig)) <= 1e-13
    assert np.linalg.norm(whole @ v[:, -1]) <= 1e-13 + sig[-1] * 1.0001
