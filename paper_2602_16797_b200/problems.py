"""The five BASELINE.json configurations and an on-device input generator.

A = U diag(sigma) V^T in fp64, row-major on the device.  U is the sign-fixed
(R_jj > 0) Householder Q of an m x n i.i.d. N(0,1) matrix and V the same for
n x n, as in matgen.cpp:126-139 / :141-176; the Gaussians come from torch's
seeded CUDA generator and the QR from cuSOLVER (via torch), so generation
takes seconds instead of the hours a CPU Householder would need at m = 1e6.
The parity tests hand the SAME bytes to the CPU oracle ("one
buffer for both solvers").  Generation is harness, not the measured path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DATA_SEED = 20260216   # S in SURVEY 8d
SOLVER_SEED = 7        # SolverOptions::seed for every config


def geometric(first, last, count):
    """matgen.cpp:30-39 geometric_fill: first..last inclusive, geometric."""
    if count == 1:
        return np.array([first], dtype=np.float64)
    i = np.arange(count, dtype=np.float64)
    return first * np.power(last / first, i / float(count - 1))


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    b: int
    d_factor: int      # d = d_factor * n
    tol: float
    note: str = ""

    @property
    def d(self):
        return self.d_factor * self.n

    def spectrum(self, n=None):
        return spectrum(self.name, self.n if n is None else n)

    def scaled(self, m=None, n=None):
        """Same recipe at a smaller shape (parity-test sizes)."""
        return Config(self.name, m or self.m, n or self.n, self.b, self.d_factor, self.tol, self.note)


CONFIGS = {
    "c1": Config("c1", 10_000, 100, 1, 2, 1e-12, "CPU-oracle size"),
    "c2": Config("c2", 1_000_000, 1_000, 1, 4, 1e-12, "headline"),
    "c3": Config("c3", 1_000_000, 2_000, 5, 2, 1e-12, "5-dim exact nullspace"),
    "c4": Config("c4", 500_000, 500, 4, 4, 1e-10, "small gap, ill-conditioned"),
    "c5": Config("c5", 8_000_000, 1_000, 2, 4, 1e-12, "multi-GPU scaling; tol unspecified -> 1e-12"),
    # the paper's illustrative example (section 1.2): m = 2e6, n = 4e3, 64 GB;
    # n > 2048 streams in column panels
    "paper_easy": Config("paper_easy", 2_000_000, 4_000, 1, 4, 1e-12, "paper section 1.2, easy"),
    "paper_hard": Config("paper_hard", 2_000_000, 4_000, 1, 4, 1e-12, "paper section 1.2, hard"),
}


def spectrum(name, n):
    """Descending singular values per BASELINE.json configs[0..4]."""
    if name == "c1":
        return np.concatenate([geometric(1.0, 1e-6, n - 1), [1e-8]])
    if name == "c2":
        return np.concatenate([geometric(1.0, 1e-4, n - 1), [1e-6]])
    if name == "c3":
        return np.concatenate([geometric(1.0, 1e-3, n - 5), np.zeros(5)])
    if name == "c4":
        return np.concatenate([geometric(1.0, 1e-3, n - 4), [1.3e-4, 1.2e-4, 1.1e-4, 1.0e-4]])
    if name == "c5":
        return np.concatenate([geometric(1.0, 1e-5, n - 1), [1e-7]])
    # the paper's own 2e6 x 4e3 examples (section 1.2), with Haar U, V
    if name == "paper_easy":  # sigma_1..n-1 geometric 1 -> 0.1, sigma_n = 1e-7
        return np.concatenate([geometric(1.0, 0.1, n - 1), [1e-7]])
    if name == "paper_hard":  # geometric 1 -> 1e-10: relative gap ~0.05 at the minimum
        return geometric(1.0, 1e-10, n)
    raise KeyError(name)


def _haar_gpu(torch, rows, cols, gen, device, block_rows=None):
    """Sign-fixed Q of a seeded Gaussian rows x cols, on the device.  Tall
    inputs larger than `block_rows` are orthonormalised as a two-level TSQR
    (local QR per block, QR of the stacked R factors), so peak memory stays
    near one copy of Q."""
    if block_rows is None or rows <= block_rows:
        g = torch.randn(rows, cols, dtype=torch.float64, device=device, generator=gen)
        q, r = torch.linalg.qr(g)
        del g
        s = torch.sign(torch.diagonal(r))
        s[s == 0] = 1.0
        q *= s
        return q.contiguous()  # cuSOLVER's Q is column-major; A is row-major
    nb = (rows + block_rows - 1) // block_rows
    q = torch.empty(rows, cols, dtype=torch.float64, device=device)
    rs = []
    for i in range(nb):
        r0, r1 = i * block_rows, min(rows, (i + 1) * block_rows)
        g = torch.randn(r1 - r0, cols, dtype=torch.float64, device=device, generator=gen)
        qi, ri = torch.linalg.qr(g)
        q[r0:r1] = qi
        rs.append(ri)
        del g, qi
    q2, r2 = torch.linalg.qr(torch.cat(rs, 0))
    s = torch.sign(torch.diagonal(r2))
    s[s == 0] = 1.0
    q2 *= s
    for i in range(nb):
        r0, r1 = i * block_rows, min(rows, (i + 1) * block_rows)
        q[r0:r1] = q[r0:r1] @ q2[i * cols:(i + 1) * cols]
    return q


def make_problem_gpu(m, n, sigma, seed=DATA_SEED, device="cuda:0", block_rows=2_000_000, ld=None, tail=None):
    """Row-major A (m x n, leading dimension ld >= n) on the device plus the
    true v_min (numpy) -- or, with `tail`, the last `tail` columns of V (the
    right singular vectors of the smallest sigma).  A = U diag(sigma) V^T is
    formed block by block in U's own storage."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    v = _haar_gpu(torch, n, n, gen, device)
    u = _haar_gpu(torch, m, n, gen, device, block_rows=block_rows)
    sig = torch.as_tensor(np.asarray(sigma, dtype=np.float64), device=device)
    vt_scaled = sig[:, None] * v.t()  # diag(sigma) V^T
    step = max(1, min(m, 1 << 18))
    ldv = n if ld is None else ld
    if ldv != n:
        a = torch.zeros(m, ldv, dtype=torch.float64, device=device)
        for r0 in range(0, m, step):
            r1 = min(m, r0 + step)
            a[r0:r1, :n] = u[r0:r1] @ vt_scaled
        del u
        out = a[:, :n]
    else:
        for r0 in range(0, m, step):
            r1 = min(m, r0 + step)
            u[r0:r1] = u[r0:r1] @ vt_scaled
        out = u
    if tail:
        return out, v[:, n - tail:].cpu().numpy().copy()
    vmin = v[:, n - 1].cpu().numpy().copy()
    return out, vmin


def _block_seed(seed, i):
    """Per-block generator seed (a SplitMix64 step, rng.hpp:18-19 style)."""
    z = (seed + 0x9E3779B97F4A7C15 * (i + 1)) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return (z ^ (z >> 31)) & 0x7FFFFFFFFFFFFFFF


def make_problem_shard(m, n, sigma, r0, rows, allreduce=None, seed=DATA_SEED, device="cuda:0",
                       block_rows=500_000):
    """Rows [r0, r0 + rows) of A = U diag(sigma) V^T, generated and
    orthonormalised shard by shard on the device (BASELINE configs[4]).

    U is the sign-fixed Q of an m x n Gaussian whose nb = m // block_rows
    fixed row blocks (boundaries i m / nb) draw from their own seeded generators, orthonormalised as a
    two-level TSQR: each block's local QR, then the QR of the stacked R
    factors (the same matgen.cpp:126-139 recipe, R_jj > 0).  Every rank
    factors only the blocks its rows touch; the R factors meet through
    `allreduce` (a sum over ranks of the [blocks * n, n] stack, each block's
    R contributed by the rank holding its first row; None on one rank).  The
    global A is therefore the same for every rank count.  Returns (A_local
    row-major, V) with V the n x n right factor."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    v = _haar_gpu(torch, n, n, gen, device)
    nb = max(1, m // block_rows)  # blocks [i m / nb, (i + 1) m / nb): each >= block_rows rows
    bound = [i * m // nb for i in range(nb + 1)]
    touch = [i for i in range(nb) if bound[i] < r0 + rows and bound[i + 1] > r0]
    first, last = (touch[0], touch[-1]) if touch else (0, -1)
    rstack = torch.zeros(nb * n, n, dtype=torch.float64, device=device)
    a = torch.empty(rows, n, dtype=torch.float64, device=device)  # holds the local Q rows first
    for i in range(first, last + 1):
        b0, b1 = bound[i], bound[i + 1]
        g = torch.Generator(device=device)
        g.manual_seed(_block_seed(int(seed), i))
        x = torch.randn(b1 - b0, n, dtype=torch.float64, device=device, generator=g)
        q, r = torch.linalg.qr(x)
        del x
        lo, hi = max(b0, r0), min(b1, r0 + rows)
        a[lo - r0:hi - r0] = q[lo - b0:hi - b0]
        del q
        if r0 <= b0 < r0 + rows:  # this rank holds the block's first row
            rstack[i * n:(i + 1) * n] = r
    if allreduce is not None:
        allreduce(rstack)
    q2, r2 = torch.linalg.qr(rstack)
    del rstack
    s = torch.sign(torch.diagonal(r2))
    s[s == 0] = 1.0
    q2 *= s
    sig = torch.as_tensor(np.asarray(sigma, dtype=np.float64), device=device)
    m2 = sig[:, None] * v.t()  # diag(sigma) V^T
    for i in range(first, last + 1):
        lo, hi = max(bound[i], r0), min(bound[i + 1], r0 + rows)
        m3 = q2[i * n:(i + 1) * n] @ m2  # U rows = Q_i Q2_i, so A rows = Q_i (Q2_i diag(sigma) V^T)
        step = 1 << 18
        for c0 in range(lo - r0, hi - r0, step):
            c1 = min(hi - r0, c0 + step)
            a[c0:c1] = a[c0:c1] @ m3
    return a, v.cpu().numpy()


def random_csr(m, n, density, seed, decay=1e-4):
    """A seeded sparse test operator for the CSR path (no BASELINE config is
    sparse): each row holds ~density*n distinct columns drawn uniformly,
    N(0,1) values, column j scaled by decay**(j/(n-1)) so the spectrum spans
    several decades.  Returns (row_offsets int64, col_indices int64, values
    float64) with sorted, unique columns per row (csr.hpp:10-25).
    numpy's PCG64 stream is stable across versions, so the bytes are
    reproducible from (m, n, density, seed)."""
    rng = np.random.default_rng(seed)
    k = max(1, int(round(density * n)))
    scale = decay ** (np.arange(n) / max(n - 1, 1))
    cols = np.argsort(rng.random((m, n)), axis=1)[:, :k] if n <= 256 else None
    if cols is None:  # large n: sample with replacement, then dedupe per row
        raw = rng.integers(0, n, size=(m, k))
        raw.sort(axis=1)
        keep = np.ones_like(raw, dtype=bool)
        keep[:, 1:] = raw[:, 1:] != raw[:, :-1]
        counts = keep.sum(axis=1)
        ci = raw[keep]
    else:
        cols.sort(axis=1)
        counts = np.full(m, k)
        ci = cols.ravel()
    rp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    v = rng.standard_normal(ci.size) * scale[ci]
    return rp, ci.astype(np.int64), v
