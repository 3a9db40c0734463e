"""ORACLE / TEST INFRASTRUCTURE ONLY -- the checker, never the thing measured.

ctypes front-end over the two CPU oracles:

* ``port`` -- oracle/_build/liboracle.so, the plain-C restatement
  (oracle/minsvd_oracle.c).  Self-contained: built on demand with gcc.
* ``ref``  -- oracle/_ref/libminsvd_ref.so, the UNMODIFIED reference library
  compiled from /root/reference/proj/src by oracle/Makefile.  Only present where
  it was built (this container; the built .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.  Inputs are numpy arrays; matrices are handed to
the C side column-major (minsvd::DenseMatrix), so a row-major device A is
transposed once here.
"""
import ctypes as C
import os
import subprocess
import sys
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
from paper_2602_16797_b200 import abi  # noqa: E402  (plain ctypes structs only)

PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libminsvd_ref.so")
REF_SRC = "/root/reference/proj/src"

_lock = threading.Lock()
_cache = {}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(kind="port", quiet=True):
    """Compile the requested oracle with oracle/Makefile (no-op when fresh)."""
    target = {"port": "port", "ref": "ref"}[kind]
    if kind == "ref" and not os.path.isdir(REF_SRC) and not os.path.exists(REF_SO):
        raise FileNotFoundError("reference sources absent and oracle/_ref not prebuilt")
    if kind == "ref" and not os.path.isdir(REF_SRC):
        return REF_SO
    out = subprocess.run(["make", "-C", HERE, target, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{out.stdout}\n{out.stderr}")
    return PORT_SO if kind == "port" else REF_SO


def available(kind):
    if kind == "port":
        return True
    return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)


def load(kind="port"):
    with _lock:
        if kind in _cache:
            return _cache[kind]
        path = build(kind)
        lib = C.CDLL(path)
        o = Oracle(lib, kind)
        _cache[kind] = o
        return o


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _colmajor(a):
    """Column-major float64 copy of a 2-D array (numpy Fortran order)."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


class Oracle:
    def __init__(self, lib, kind):
        self.lib = lib
        self.kind = kind
        pre = "orc_" if kind == "port" else "ref_"
        self.pre = pre
        self._err = getattr(lib, pre + "last_error")
        self._err.restype = C.c_char_p
        g = lambda name: getattr(lib, pre + name)  # noqa: E731
        self._solve = g("lobpcg_solve")
        self._solve.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.POINTER(abi.Options),
                                C.POINTER(abi.Truth), C.POINTER(abi.Result)]
        self._synth = g("synth_dense")
        self._synth.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_uint64,
                                C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self._haar = g("haar_orthonormal")
        self._haar.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.POINTER(C.c_double)]
        self._draws = g("splitmix_draws")
        self._draws.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int64,
                                C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_uint64]
        self._draws.restype = None
        self._stack = g("build_sparsestack")
        self._stack.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_uint64, C.POINTER(C.c_uint32),
                                C.POINTER(C.c_int8)]
        if kind == "port":
            self._sketch = lib.orc_sketch_rows
            self._sketch.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.POINTER(C.c_double), C.c_int64,
                                     C.c_int64, C.c_int64, C.POINTER(C.c_double)]
            self._orth = lib.orc_orth_coefficients
            self._orth.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.POINTER(C.c_double)]
        else:
            self._sketch = lib.ref_sketch_apply
            self._sketch.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.POINTER(C.c_double), C.c_int64,
                                     C.c_int64, C.POINTER(C.c_double)]
        self._hr = g("householder_r")
        self._hr.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.POINTER(C.c_double)]
        self._svd = g("dense_svd")
        self._svd.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.POINTER(C.c_double),
                              C.POINTER(C.c_double)]
        self._pc = g("build_preconditioner")
        self._pc.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.POINTER(C.c_double),
                             C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        self._pa = g("precond_apply")
        self._pa.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64,
                             C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double)]
        self._cc = g("check_convergence")
        self._cc.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64, C.c_int,
                             C.c_double, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_int)]
        self._lz = g("lanczos_gk")
        self._lz.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_int, C.POINTER(C.c_double),
                             C.POINTER(abi.Truth), C.c_int, C.POINTER(abi.LanczosResult)]
        I64 = C.POINTER(C.c_int64)
        csr_args = [C.c_int64, C.c_int64, I64, I64, C.POINTER(C.c_double), C.c_int64]
        self._solve_csr = g("lobpcg_solve_csr")
        self._solve_csr.argtypes = csr_args + [C.POINTER(abi.Options), C.POINTER(abi.Truth), C.POINTER(abi.Result)]
        self._lz_csr = g("lanczos_gk_csr")
        self._lz_csr.argtypes = csr_args + [C.c_int, C.POINTER(C.c_double), C.POINTER(abi.Truth), C.c_int,
                                            C.POINTER(abi.LanczosResult)]
        self._csr_prod = g("csr_products")
        self._csr_prod.argtypes = csr_args + [C.POINTER(C.c_double)] * 5
        self._sk_csr = g("sketch_csr")
        if kind == "port":
            self._sk_csr.argtypes = [C.c_int64, C.c_int, C.c_uint64] + csr_args + [C.c_int64, C.POINTER(C.c_double)]
        else:
            self._sk_csr.argtypes = [C.c_int64, C.c_int, C.c_uint64] + csr_args + [C.POINTER(C.c_double)]
        self._cgs2 = g("cgs2")
        self._cgs2.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.POINTER(C.c_double),
                               C.c_int64, C.c_uint64, C.POINTER(C.c_int64)]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err().decode(errors="replace"))

    # -- generators ---------------------------------------------------------
    def synth_dense(self, sigma, m, seed):
        """matgen.cpp:141-176 synth(explicit_list): returns (A column-major
        numpy (m, n) Fortran array, v_min)."""
        sigma = _f64(sigma)
        n = sigma.size
        a = np.empty((m, n), dtype=np.float64, order="F")
        vmin = np.empty(n)
        self._check(self._synth(_p(sigma), n, m, seed, _p(a), _p(vmin)))
        return a, vmin

    def assemble_svd(self, sigma, m, seed):
        """U diag(sigma) V^T with synth's factors but no spectrum validation
        (zeros allowed); port only."""
        sigma = _f64(sigma)
        n = sigma.size
        a = np.empty((m, n), dtype=np.float64, order="F")
        vmin = np.empty(n)
        f = self.lib.orc_assemble_svd
        f.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_uint64, C.POINTER(C.c_double),
                      C.POINTER(C.c_double)]
        self._check(f(_p(sigma), n, m, seed, _p(a), _p(vmin)))
        return a, vmin

    def synth_fast(self, sigma, m, seed):
        """Harness-only generator (port only; minsvd_oracle.c orc_synth_fast):
        A = U diag(sigma) V^T with U = X R^-1 from a Cholesky QR of a seeded
        Gaussian X and V = haar_orthonormal(n, n); bit-reproducible and
        thread-count independent.  Returns (A column-major, V n x n)."""
        sigma = _f64(sigma)
        n = sigma.size
        a = np.empty((m, n), dtype=np.float64, order="F")
        v = np.empty((n, n), dtype=np.float64, order="F")
        f = self.lib.orc_synth_fast
        f.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_uint64, C.POINTER(C.c_double),
                      C.POINTER(C.c_double)]
        self._check(f(_p(sigma), n, m, seed, _p(a), _p(v)))
        return a, v

    def haar_orthonormal(self, m, n, seed):
        q = np.empty((m, n), order="F")
        self._check(self._haar(m, n, seed, _p(q)))
        return q

    def splitmix_draws(self, seed, key=None, kind="u64", count=16, bound=1):
        kinds = {"u64": 0, "below": 1, "unit": 2, "gauss": 3}[kind]
        f = np.zeros(count)
        u = np.zeros(count, dtype=np.uint64)
        self._draws(seed, key or 0, int(key is not None), kinds, count, _p(f), _p(u, C.c_uint64), bound)
        return u if kinds < 2 else f

    # -- kernels ------------------------------------------------------------
    def build_sparsestack(self, d, m, zeta, seed):
        pos = np.empty(m * zeta, dtype=np.uint32)
        sgn = np.empty(m * zeta, dtype=np.int8)
        self._check(self._stack(d, m, zeta, seed, _p(pos, C.c_uint32), _p(sgn, C.c_int8)))
        return pos, sgn

    def sketch_apply(self, a, d, zeta, seed, row0=0):
        a = _colmajor(a)
        m, n = a.shape
        sa = np.empty((d, n), order="F")
        if self.kind == "port":
            self._check(self._sketch(d, zeta, seed, _p(a), m, n, row0, _p(sa)))
        else:
            if row0:
                raise ValueError("row-sharded sketch is a port-only helper")
            self._check(self._sketch(d, zeta, seed, _p(a), m, n, _p(sa)))
        return sa

    def householder_r(self, a):
        a = _colmajor(a)
        m, k = a.shape
        r = np.empty((k, k), order="F")
        self._check(self._hr(_p(a), m, k, _p(r)))
        return r

    def dense_svd(self, a):
        a = _colmajor(a)
        rows, n = a.shape
        s = np.empty(n)
        v = np.empty((n, n), order="F")
        self._check(self._svd(_p(a), rows, n, _p(s), _p(v)))
        return s, v

    def build_preconditioner(self, sa):
        sa = _colmajor(sa)
        rows, n = sa.shape
        vt = np.empty((n, n), order="F")
        sig = np.empty(n)
        smax = C.c_double()
        nf = C.c_int64()
        self._check(self._pc(_p(sa), rows, n, _p(vt), _p(sig), C.byref(smax), C.byref(nf)))
        return vt, sig, smax.value, nf.value

    def precond_apply(self, vt, sig, r):
        vt = _colmajor(vt)
        n = vt.shape[0]
        r = _colmajor(r.reshape(n, -1))
        w = np.empty_like(r, order="F")
        self._check(self._pa(_p(vt), _p(_f64(sig)), n, _p(r), r.shape[1], _p(w)))
        return w

    def check_convergence(self, resid, theta, i, sigma1, tol, factor=1.1, use_stagnation=True):
        resid, theta = _f64(resid), _f64(theta)
        flags = (C.c_int * 4)()
        self._check(self._cc(_p(resid), _p(theta), resid.size, i, sigma1, tol, factor,
                             int(use_stagnation), flags))
        return dict(tol_ok=bool(flags[0]), resid_stalled=bool(flags[1]),
                    progress_stalled=bool(flags[2]), stop=bool(flags[3]))

    def cgs2(self, w, basis, seed):
        w = _colmajor(w).copy(order="F")
        n, c = w.shape
        basis = _colmajor(basis) if basis is not None and basis.size else np.zeros((n, 0), order="F")
        rep = C.c_int64()
        self._check(self._cgs2(_p(w), n, c, _p(basis), basis.shape[1], seed, C.byref(rep)))
        return w, rep.value

    # -- full solve ---------------------------------------------------------
    def lobpcg_solve(self, a, opts=None, truth=None, want_precond=False, want_iterates=False, **kw):
        """solver.cpp:301-477 on a dense A; returns a dict shaped like SolveResult."""
        a = _colmajor(a)
        m, n = a.shape
        o = opts if opts is not None else abi.default_options()
        for k, v in kw.items():
            setattr(o, k, int(v) if isinstance(v, bool) else v)
        b = int(o.block_size)
        max_iter = o.max_iter if o.max_iter >= 0 else (200 if b == 1 else 100)
        cap = max_iter + 2
        sigma = np.zeros(max(b, 1))
        v = np.zeros((n, max(b, 1)), order="F")
        rows = (abi.RecordRow * cap)()
        res = abi.Result()
        res.sigma = _p(sigma)
        res.v = _p(v)
        res.rows = rows
        res.rows_capacity = cap
        vt = sig = None
        if want_precond:
            vt = np.zeros((n, n), order="F")
            sig = np.zeros(n)
            res.vtilde = _p(vt)
            res.sigma_tilde = _p(sig)
        trail = {"t": [], "v": []}

        def sink(_u, kind, it, data, r, c):
            arr = np.ctypeslib.as_array(data, shape=(int(c), int(r))).T.copy(order="F")
            trail["t" if kind == 0 else "v"].append((int(it), arr))

        cb = abi.ITERATE_FN(sink) if want_iterates else abi.ITERATE_FN()
        res.iterate_cb = cb
        tr = None
        if truth is not None:
            vmin = _f64(truth[1])
            tr = abi.Truth(float(truth[0]), _p(vmin))
        self._check(self._solve(_p(a), m, n, C.byref(o), C.byref(tr) if tr else None, C.byref(res)))
        return _result_dict(res, rows, sigma, v, vt, sig, trail, has_truth=truth is not None)

    # -- CSR operator (csr.cpp, operator.hpp:58-74) ---------------------------
    def _csr(self, a):
        """a = (row_offsets, col_indices, values, m, n) -> ctypes argument list."""
        rp, ci, v, m, n = a
        rp = np.ascontiguousarray(rp, dtype=np.int64)
        ci = np.ascontiguousarray(ci, dtype=np.int64)
        v = _f64(v)
        keep = (rp, ci, v)
        return keep, [int(m), int(n), _p(rp, C.c_int64), _p(ci, C.c_int64), _p(v), int(v.size)]

    def csr_products(self, a, x=None, y=None, norms=False):
        keep, args = self._csr(a)
        m, n = a[3], a[4]
        yo = np.zeros(m) if x is not None else None
        xo = np.zeros(n) if y is not None else None
        no = np.zeros(n) if norms else None
        xi = _f64(x) if x is not None else None
        yi = _f64(y) if y is not None else None
        nul = C.POINTER(C.c_double)()
        self._check(self._csr_prod(*args, _p(xi) if xi is not None else nul, _p(yo) if yo is not None else nul,
                                   _p(yi) if yi is not None else nul, _p(xo) if xo is not None else nul,
                                   _p(no) if no is not None else nul))
        del keep
        return yo, xo, no

    def sketch_csr(self, a, d, zeta, seed, row0=0):
        keep, args = self._csr(a)
        sa = np.empty((d, a[4]), order="F")
        if self.kind == "port":
            self._check(self._sk_csr(d, zeta, seed, *args, row0, _p(sa)))
        else:
            if row0:
                raise ValueError("row-sharded sketch is a port-only helper")
            self._check(self._sk_csr(d, zeta, seed, *args, _p(sa)))
        del keep
        return sa

    def lobpcg_solve_csr(self, a, opts=None, truth=None, want_precond=False, **kw):
        """solver.cpp:301-477 on a CsrOperator."""
        keep, args = self._csr(a)
        n = a[4]
        o = opts if opts is not None else abi.default_options()
        for k, v in kw.items():
            setattr(o, k, int(v) if isinstance(v, bool) else v)
        b = int(o.block_size)
        max_iter = o.max_iter if o.max_iter >= 0 else (200 if b == 1 else 100)
        cap = max_iter + 2
        sigma = np.zeros(max(b, 1))
        v = np.zeros((n, max(b, 1)), order="F")
        rows = (abi.RecordRow * cap)()
        res = abi.Result()
        res.sigma = _p(sigma)
        res.v = _p(v)
        res.rows = rows
        res.rows_capacity = cap
        vt = sig = None
        if want_precond:
            vt = np.zeros((n, n), order="F")
            sig = np.zeros(n)
            res.vtilde = _p(vt)
            res.sigma_tilde = _p(sig)
        res.iterate_cb = abi.ITERATE_FN()
        tr = None
        if truth is not None:
            vmin = _f64(truth[1])
            tr = abi.Truth(float(truth[0]), _p(vmin))
        self._check(self._solve_csr(*args, C.byref(o), C.byref(tr) if tr else None, C.byref(res)))
        del keep
        return _result_dict(res, rows, sigma, v, vt, sig, {"t": [], "v": []}, has_truth=truth is not None)

    def lanczos_gk_csr(self, a, iters, v0, truth=None, record_timing=False, want_bases=False):
        keep, args = self._csr(a)
        m, n = a[3], a[4]
        v0 = _f64(v0)
        res, rows, v, vb, ub = _lanczos_buffers(m, n, iters, want_bases)
        tr = None
        if truth is not None:
            vmin = _f64(truth[1])
            tr = abi.Truth(float(truth[0]), _p(vmin))
        self._check(self._lz_csr(*args, int(iters), _p(v0), C.byref(tr) if tr else None, int(record_timing),
                                 C.byref(res)))
        del keep
        return lanczos_dict(res, rows, v, vb, ub)

    # -- Krylov baseline ----------------------------------------------------
    def lanczos_gk(self, a, iters, v0, truth=None, record_timing=False, want_bases=False):
        """baselines.cpp:51-166 on a dense A; returns a dict shaped like
        LanczosResult."""
        a = _colmajor(a)
        m, n = a.shape
        v0 = _f64(v0)
        res, rows, v, vb, ub = _lanczos_buffers(m, n, iters, want_bases)
        tr = None
        if truth is not None:
            vmin = _f64(truth[1])
            tr = abi.Truth(float(truth[0]), _p(vmin))
        self._check(self._lz(_p(a), m, n, int(iters), _p(v0), C.byref(tr) if tr else None, int(record_timing),
                             C.byref(res)))
        return lanczos_dict(res, rows, v, vb, ub)


def _lanczos_buffers(m, n, iters, want_bases):
    cap = max(int(iters), 1)
    rows = (abi.RecordRow * cap)()
    v = np.zeros(n)
    res = abi.LanczosResult()
    res.v = _p(v)
    res.rows = rows
    res.rows_capacity = cap
    vb = ub = None
    if want_bases:
        vb = np.zeros((n, cap), order="F")
        ub = np.zeros((m, cap), order="F")
        res.v_basis = _p(vb)
        res.u_basis = _p(ub)
    return res, rows, v, vb, ub


def lanczos_dict(res, rows, v, vb, ub):
    cnt = res.rows_count
    rec = [dict(iter=r.iter, matvecs_a=r.matvecs_a, matvecs_at=r.matvecs_at, wall_ms=r.wall_ms,
                theta=r.theta, resid=r.resid, relerr=r.relerr, sin_angle=r.sin_angle)
           for r in rows[:min(cnt, res.rows_capacity)]]
    steps = res.steps
    return dict(sigma_min=res.sigma_min, v=v.copy(), record=rec, steps=steps,
                status="completed" if res.status == abi.LANCZOS_COMPLETED else "invariant_subspace",
                v_basis=None if vb is None else vb[:, :steps].copy(order="F"),
                u_basis=None if ub is None else ub[:, :steps].copy(order="F"))


def _result_dict(res, rows, sigma, v, vt, sig, trail, has_truth):
    cnt = res.rows_count
    rec = [dict(iter=r.iter, matvecs_a=r.matvecs_a, matvecs_at=r.matvecs_at, wall_ms=r.wall_ms,
                theta=r.theta, resid=r.resid, relerr=r.relerr, sin_angle=r.sin_angle)
           for r in rows[:min(cnt, res.rows_capacity)]]
    return dict(sigma=sigma.copy(), v=np.array(v), status=("converged" if res.status == 0 else
                                                         "max_iter_reached"),
                iterations=res.iterations, record=rec, has_truth=has_truth,
                sigma_max_estimate=res.sigma_max_estimate, floored=bool(res.floored),
                floor_count=res.floor_count, sketch_skipped=bool(res.sketch_skipped),
                sketch_dim=res.sketch_dim, zeta=res.zeta, verify_count=res.verify_count,
                max_cache_drift=res.max_cache_drift,
                degenerate_replacements=res.degenerate_replacements,
                vtilde=vt, sigma_tilde=sig, trail_t=trail["t"], trail_v=trail["v"])
