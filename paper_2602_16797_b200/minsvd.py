"""Python mirror of the reference's solve API over libmsvd_cuda.so.

Same names, argument meaning and error behaviour as minsvd's C++ API
(/root/reference/proj/include/minsvd/solver.hpp:25-190, operator.hpp:15-56,
errors.hpp:9-38), so tests read like the reference's own:

    opts = SolverOptions(seed=7, block_size=4, tol=1e-10, use_stagnation=False)
    res = rlobpcg_block(DeviceDenseOperator(A_cuda), opts, truth)
    res.sigma, res.v, res.record.to_csv(), res.iterations()

Device memory is plumbing from torch; every computation runs in the CUDA
library.  There is no CPU path: importing works anywhere, but any call that
needs the GPU raises when the extension or the device is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmsvd_cuda.so")
CSRC = os.path.join(HERE, "csrc")


# --------------------------------------------------------------- errors.hpp
class Error(RuntimeError):
    """minsvd::Error"""


class DimensionError(Error):
    """minsvd::DimensionError"""


class IoError(Error):
    """minsvd::IoError"""


class NumericalError(Error):
    """minsvd::NumericalError"""


class ConvergenceError(Error):
    """minsvd::ConvergenceError"""


_STATUS_EXC = {
    abi.MSVD_ERR_DIMENSION: DimensionError,
    abi.MSVD_ERR_IO: IoError,
    abi.MSVD_ERR_NUMERICAL: NumericalError,
    abi.MSVD_ERR_CONVERGENCE: ConvergenceError,
}


# ----------------------------------------------------------------- library
_lib = None


def build(force=False, quiet=True):
    """Compile libmsvd_cuda.so in-tree (nvcc, sm_100a)."""
    args = ["make", "-C", CSRC, "-j8"]
    if force:
        subprocess.run(["make", "-C", CSRC, "clean"], check=True, capture_output=quiet)
    out = subprocess.run(args, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"libmsvd_cuda build failed:\n{out.stdout[-4000:]}\n{out.stderr[-4000:]}")
    return LIB_PATH


def _declare(lib):
    P = C.POINTER
    d = C.c_double
    i64 = C.c_int64
    i32 = C.c_int32
    vp = C.c_void_p
    sig = {
        "msvd_abi_version": (i32, []),
        "msvd_last_error": (C.c_char_p, []),
        "msvd_status_name": (C.c_char_p, [i32]),
        "msvd_options_default": (None, [P(abi.Options)]),
        "msvd_default_tolerance": (d, [i64]),
        "msvd_validate_options": (i32, [i64, i64, P(abi.Options), P(abi.Truth)]),
        "msvd_shard_rows": (None, [i64, i32, i32, P(i64), P(i64)]),
        "msvd_get_nccl_unique_id": (i32, [P(C.c_uint8)]),
        "msvd_fake_group_create": (i32, [i32, P(vp)]),
        "msvd_fake_group_destroy": (i32, [vp]),
        "msvd_ctx_create": (i32, [P(abi.CtxDesc), P(vp)]),
        "msvd_ctx_destroy": (i32, [vp]),
        "msvd_ctx_synchronize": (i32, [vp]),
        "msvd_matrix_attach": (i32, [vp, vp, i64, i64, i64, i64, i64, P(vp)]),
        "msvd_matrix_detach": (i32, [vp]),
        "msvd_csr_attach": (i32, [vp, vp, vp, i32, vp, i64, i64, i64, i64, i64, P(vp)]),
        "msvd_apply": (i32, [vp, vp, i64, vp]),
        "msvd_apply_adjoint": (i32, [vp, vp, i64, vp]),
        "msvd_column_norms": (i32, [vp, vp]),
        "msvd_build_sparsestack": (i32, [vp, i64, i64, i32, C.c_uint64, vp, vp]),
        "msvd_sketch": (i32, [vp, i64, i32, C.c_uint64, vp]),
        "msvd_precond_build": (i32, [vp, vp, i64, i64, vp, vp, P(d), P(i64)]),
        "msvd_precond_apply": (i32, [vp, vp, vp, i64, vp, i64, vp]),
        "msvd_tsqr_r": (i32, [vp, vp, i64, i64, vp]),
        "msvd_gram_apply": (i32, [vp, vp, i64, vp, i64, i64, vp, vp]),
        "msvd_aw_tsqr": (i32, [vp, vp, i64, vp, i64, vp, vp]),
        "msvd_aw_gram": (i32, [vp, vp, i64, vp, vp]),
        "msvd_aw_gram_ex": (i32, [vp, vp, i64, vp, vp, vp, vp]),
        "msvd_small_svd": (i32, [vp, vp, i64, vp, vp]),
        "msvd_check_convergence": (i32, [vp, P(d), P(d), i64, i32, d, d, d, i32, P(i32)]),
        "msvd_raw_write": (i32, [C.c_char_p, vp, i64, i64, i64]),
        "msvd_raw_info": (i32, [C.c_char_p, P(i64), P(i64)]),
        "msvd_raw_read_rows": (i32, [C.c_char_p, i64, i64, vp, i64]),
        "msvd_raw_load_device": (i32, [vp, C.c_char_p, i64, i64, vp, i64]),
        "msvd_lanczos_gk": (i32, [vp, i32, vp, P(abi.Truth), i32, P(abi.LanczosResult)]),
        "msvd_lobpcg_solve": (i32, [vp, P(abi.Options), P(abi.Truth), P(abi.Result)]),
        "msvd_rlobpcg_single": (i32, [vp, P(abi.Options), P(abi.Truth), P(abi.Result)]),
        "msvd_rlobpcg_block": (i32, [vp, P(abi.Options), P(abi.Truth), P(abi.Result)]),
        "msvd_solve_host": (i32, [vp, vp, i64, i64, i64, i64, i64, P(abi.Options), P(abi.Truth),
                                  P(abi.Result)]),
        "msvd_launch_count": (i64, [vp]),
        "msvd_abi_sizes": (None, [P(i64), i32]),
        "msvd_ctx_profile": (i32, [vp, i32]),
        "msvd_ctx_kernel_paths": (i64, [vp, i32]),
        "msvd_ctx_profile_read": (i32, [vp, P(d), P(i64), i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


EXPORTED = (
    "msvd_abi_version msvd_last_error msvd_status_name msvd_options_default msvd_default_tolerance "
    "msvd_validate_options msvd_shard_rows msvd_get_nccl_unique_id msvd_fake_group_create "
    "msvd_fake_group_destroy msvd_ctx_create msvd_ctx_destroy msvd_ctx_synchronize msvd_matrix_attach "
    "msvd_matrix_detach msvd_csr_attach msvd_apply msvd_apply_adjoint msvd_column_norms msvd_build_sparsestack msvd_sketch "
    "msvd_precond_build msvd_precond_apply msvd_tsqr_r msvd_gram_apply msvd_aw_tsqr msvd_aw_gram msvd_aw_gram_ex msvd_small_svd "
    "msvd_raw_write msvd_raw_info msvd_raw_read_rows msvd_raw_load_device msvd_lanczos_gk msvd_lobpcg_solve msvd_rlobpcg_single "
    "msvd_rlobpcg_block msvd_solve_host msvd_launch_count msvd_abi_sizes msvd_ctx_profile msvd_ctx_profile_read "
    "msvd_ctx_kernel_paths msvd_check_convergence"
).split()


def lib():
    """Load the CUDA extension; fails loudly if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2602_16797_b200.minsvd.build() "
                              "(the solver has no CPU fallback)")
        _lib = _declare(C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL))
        if _lib.msvd_abi_version() != 1:
            raise ImportError("libmsvd_cuda ABI version mismatch")
    return _lib


def check(rc):
    if rc != 0:
        msg = lib().msvd_last_error().decode(errors="replace")
        raise _STATUS_EXC.get(rc, Error)(msg)


def default_tolerance(n):
    """solver.hpp:83-85"""
    return 2.0 * np.sqrt(float(n)) * np.finfo(np.float64).eps


# --------------------------------------------------------- solver.hpp types
@dataclass
class SolverOptions:
    """solver.hpp:25-78, same fields and defaults."""

    tol: float = -1.0
    max_iter: int = -1
    check_every: int = 5
    stagnation_factor: float = 1.1
    block_size: int = 1
    seed: int = 0
    sketch_dim: int = -1
    zeta: int = 4
    use_stagnation: bool = True
    record_timing: bool = True
    verify_cached_products: bool = False
    store_iterates: bool = False

    def to_abi(self, kind=abi.PRECOND_RANDOMIZED):
        return abi.Options(tol=float(self.tol), max_iter=int(self.max_iter), check_every=int(self.check_every),
                           stagnation_factor=float(self.stagnation_factor), block_size=int(self.block_size),
                           seed=int(self.seed) & 0xFFFFFFFFFFFFFFFF, sketch_dim=int(self.sketch_dim),
                           zeta=int(self.zeta), use_stagnation=int(bool(self.use_stagnation)),
                           record_timing=int(bool(self.record_timing)),
                           verify_cached_products=int(bool(self.verify_cached_products)),
                           store_iterates=int(bool(self.store_iterates)), precond_kind=int(kind))


class PrecondKind:
    """solver.hpp:14"""

    none = abi.PRECOND_NONE
    diagonal = abi.PRECOND_DIAGONAL
    randomized = abi.PRECOND_RANDOMIZED


@dataclass
class GroundTruth:
    sigma_min: float
    v_min: np.ndarray


@dataclass
class RecordRow:
    iter: int
    matvecs_a: int
    matvecs_at: int
    wall_ms: float
    theta: float
    resid: float
    relerr: float = -1.0
    sin_angle: float = -1.0


def format_double(x):
    """io.cpp:11-15 (%.17g)"""
    return "%.17g" % x


@dataclass
class ConvergenceRecord:
    rows: List[RecordRow] = field(default_factory=list)
    has_truth: bool = False

    def to_csv(self):
        """solver.cpp:149-171"""
        out = ["iter,matvecs_A,matvecs_At,wall_ms,theta,resid_norm,singval_relerr,sin_angle\n"]
        for r in self.rows:
            line = f"{r.iter},{r.matvecs_a},{r.matvecs_at},{format_double(r.wall_ms)},"
            line += f"{format_double(r.theta)},{format_double(r.resid)},"
            line += (f"{format_double(r.relerr)},{format_double(r.sin_angle)}" if self.has_truth else ",")
            out.append(line + "\n")
        return "".join(out)


@dataclass
class Preconditioner:
    vtilde: Optional[np.ndarray]
    sigma_tilde: Optional[np.ndarray]
    sigma_max_estimate: float
    floored: bool
    floor_count: int


@dataclass
class SolveResult:
    """solver.hpp:118-137"""

    v: np.ndarray
    sigma: np.ndarray
    status: str
    record: ConvergenceRecord
    precond: Preconditioner
    sigma_max_estimate: float
    sketch_skipped: bool
    sketch_dim: int
    zeta: int
    verify_count: int
    max_cache_drift: float
    degenerate_replacements: int
    trail_t: list = field(default_factory=list)
    trail_v: list = field(default_factory=list)
    timings_ms: dict = field(default_factory=dict)

    def iterations(self):
        return len(self.record.rows) - 1


# ----------------------------------------------------------------- context
class Context:
    """A CUDA device + stream + communicator (msvd_ctx)."""

    def __init__(self, device=0, comm_kind=0, nranks=1, rank=0, nccl_id=None, fake_group=None, stream=None):
        desc = abi.CtxDesc()
        desc.device = device
        desc.comm_kind = comm_kind
        desc.nranks = nranks
        desc.rank = rank
        if nccl_id is not None:
            for i, byte in enumerate(bytes(nccl_id)[:128]):
                desc.nccl_id[i] = byte
        desc.fake_group = fake_group
        desc.stream = stream
        h = C.c_void_p()
        check(lib().msvd_ctx_create(C.byref(desc), C.byref(h)))
        self.handle = h
        self.device = device
        self.nranks = nranks
        self.rank = rank

    def synchronize(self):
        check(lib().msvd_ctx_synchronize(self.handle))

    def launch_count(self):
        return lib().msvd_launch_count(self.handle)

    PATHS = ("rows", "self", "pair", "pair_ex", "team_ex", "ticket", "gram", "tsqr", "chol_precond", "team", "split", "split_ex")

    def kernel_paths(self, reset=True):
        """Names of the A-pass kernel variants launched since the last reset
        (msvd_ctx_kernel_paths)."""
        mask = lib().msvd_ctx_kernel_paths(self.handle, int(bool(reset)))
        return {name for i, name in enumerate(self.PATHS) if mask >> i & 1}

    PROFILE_SLOTS = ("apply", "gram", "tsqr", "rr", "sketch", "svd", "precond", "cgs2", "reduce", "control")

    def profile(self, enable=True):
        """Per-kernel-class CUDA-event timing on this context's stream.
        enable: True / 2 every class, 1 the A-pass classes only (apply, gram),
        False / 0 off."""
        check(lib().msvd_ctx_profile(self.handle, 2 if enable is True else int(enable)))

    def profile_read(self):
        n = len(self.PROFILE_SLOTS)
        ms = (C.c_double * n)()
        cnt = (C.c_int64 * n)()
        check(lib().msvd_ctx_profile_read(self.handle, ms, cnt, n))
        return {k: (ms[i], cnt[i]) for i, k in enumerate(self.PROFILE_SLOTS)}

    def close(self):
        if self.handle:
            lib().msvd_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = {}


def torch_stream_handle(device=0):
    """The current torch stream of `device` as a cudaStream_t for the
    library, so library kernels are ordered with the torch work that
    produced their inputs (torch's default stream 0 -> cudaStreamLegacy)."""
    import torch

    h = torch.cuda.current_stream(device).cuda_stream
    return h if h else 1  # cudaStreamLegacy


def default_context(device=0):
    """Context on `device` bound to torch's current stream there."""
    if device not in _default_ctx:
        _default_ctx[device] = Context(device, stream=torch_stream_handle(device))
    return _default_ctx[device]


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    check(lib().msvd_get_nccl_unique_id(buf))
    return bytes(buf)


class FakeGroup:
    """In-process group of `nranks` contexts on one GPU (test communicator)."""

    def __init__(self, nranks):
        h = C.c_void_p()
        check(lib().msvd_fake_group_create(nranks, C.byref(h)))
        self.handle = h
        self.nranks = nranks

    def context(self, rank, device=0, stream=None):
        return Context(device, comm_kind=2, nranks=self.nranks, rank=rank, fake_group=self.handle, stream=stream)

    def close(self):
        if self.handle:
            lib().msvd_fake_group_destroy(self.handle)
            self.handle = None


def shard_rows(m, nranks, rank):
    """Contiguous row block owned by `rank`."""
    r0, rows = C.c_int64(), C.c_int64()
    lib().msvd_shard_rows(m, nranks, rank, C.byref(r0), C.byref(rows))
    return r0.value, rows.value


# --------------------------------------------------------------- operator
def _torch():
    import torch

    return torch


class DeviceDenseOperator:
    """operator.hpp:41-56 DenseOperator over device memory (row-major A).

    `a` is a CUDA float64 torch tensor holding this rank's rows (m_local x n,
    row stride `ld`); row0/m_global place them in the global matrix.
    Products are deterministic for a fixed device and rank count.
    """

    def __init__(self, a, ctx: Optional[Context] = None, row0=0, m_global=None):
        torch = _torch()
        if not (isinstance(a, torch.Tensor) and a.is_cuda and a.dtype == torch.float64 and a.dim() == 2):
            raise DimensionError("DeviceDenseOperator needs a 2-D float64 CUDA tensor")
        if a.stride(1) != 1:
            raise DimensionError("DeviceDenseOperator needs row-major storage (unit column stride)")
        self.a = a
        self.device = a.device
        self.ctx = ctx or default_context(a.device.index or 0)
        self.m_local, self.n = a.shape
        self.ld = a.stride(0) if self.m_local > 1 else self.n
        self.row0 = row0
        self.m_global = self.m_local if m_global is None else m_global
        h = C.c_void_p()
        check(lib().msvd_matrix_attach(self.ctx.handle, C.c_void_p(a.data_ptr()), self.m_local, self.n,
                                       max(self.ld, self.n), row0, self.m_global, C.byref(h)))
        self.handle = h

    def rows(self):
        return self.m_global

    def cols(self):
        return self.n

    def nnz(self):
        return self.m_global * self.n

    def _cm(self, x, rows):
        """column-major (rows x b) device copy of x"""
        torch = _torch()
        x = torch.as_tensor(x, dtype=torch.float64, device=self.device)
        if x.dim() == 1:
            x = x.reshape(-1, 1)
        if x.shape[0] != rows:
            raise DimensionError("apply_block: dimension mismatch")
        return x.t().contiguous(), x.shape[1]

    def apply_block(self, x):
        """operator.cpp:7-12: Y = A X (local rows)."""
        torch = _torch()
        xt, b = self._cm(x, self.n)
        y = torch.empty((b, self.m_local), dtype=torch.float64, device=self.device)
        check(lib().msvd_apply(self.handle, C.c_void_p(xt.data_ptr()), b, C.c_void_p(y.data_ptr())))
        return y.t()

    def apply_adjoint_block(self, y):
        """operator.cpp:14-19: X = A^T Y (summed over ranks)."""
        torch = _torch()
        yt, b = self._cm(y, self.m_local)
        x = torch.empty((b, self.n), dtype=torch.float64, device=self.device)
        check(lib().msvd_apply_adjoint(self.handle, C.c_void_p(yt.data_ptr()), b, C.c_void_p(x.data_ptr())))
        return x.t()

    def gram_apply(self, t, c=None, b=None):
        """K2 (solver.cpp:357-369, :421): Y = T C, G = A^T Y[:, :b]; c=None: G = A^T T."""
        torch = _torch()
        tt, k = self._cm(t, self.m_local)
        if c is None:
            b = k
            q = k
            ct = None
        else:
            c = torch.as_tensor(c, dtype=torch.float64, device=self.device)
            q = c.shape[1]
            b = q if b is None else b
            ct = c.t().contiguous()  # column-major k x q
        g = torch.empty((b, self.n), dtype=torch.float64, device=self.device)
        y = torch.empty((q, self.m_local), dtype=torch.float64, device=self.device) if ct is not None else None
        check(lib().msvd_gram_apply(self.handle, C.c_void_p(tt.data_ptr()), k,
                                    C.c_void_p(ct.data_ptr()) if ct is not None else None, q, b,
                                    C.c_void_p(g.data_ptr()), C.c_void_p(y.data_ptr()) if y is not None else None))
        return g.t(), (y.t() if y is not None else None)

    def aw_tsqr(self, w, lead=None):
        """K3 (solver.cpp:412-416): AW = A W and the R factor of [lead | AW]."""
        torch = _torch()
        wt, b = self._cm(w, self.n)
        if lead is not None:
            lt, kl = self._cm(lead, self.m_local)
        else:
            lt, kl = None, 0
        k = kl + b
        aw = torch.empty((b, self.m_local), dtype=torch.float64, device=self.device)
        r = torch.empty((k, k), dtype=torch.float64, device=self.device)
        check(lib().msvd_aw_tsqr(self.handle, C.c_void_p(wt.data_ptr()), b,
                                 C.c_void_p(lt.data_ptr()) if lt is not None else None, kl,
                                 C.c_void_p(aw.data_ptr()), C.c_void_p(r.data_ptr())))
        return aw.t(), r.t()

    def aw_gram(self, w):
        """One pass: AW = A W and Z = A^T A W."""
        torch = _torch()
        wt, b = self._cm(w, self.n)
        aw = torch.empty((b, self.m_local), dtype=torch.float64, device=self.device)
        z = torch.empty((b, self.n), dtype=torch.float64, device=self.device)
        check(lib().msvd_aw_gram(self.handle, C.c_void_p(wt.data_ptr()), b, C.c_void_p(aw.data_ptr()),
                                 C.c_void_p(z.data_ptr())))
        return aw.t(), z.t()

    def aw_gram_ex(self, w, e):
        """One pass (the check refresh): AW = A W, Z = A^T A W and ZE = A^T E."""
        torch = _torch()
        wt, b = self._cm(w, self.n)
        et, be = self._cm(e, self.m_local)
        if be != b:
            raise DimensionError("aw_gram_ex: E must have as many columns as W")
        aw = torch.empty((b, self.m_local), dtype=torch.float64, device=self.device)
        z = torch.empty((b, self.n), dtype=torch.float64, device=self.device)
        ze = torch.empty((b, self.n), dtype=torch.float64, device=self.device)
        check(lib().msvd_aw_gram_ex(self.handle, C.c_void_p(wt.data_ptr()), b, C.c_void_p(et.data_ptr()),
                                    C.c_void_p(aw.data_ptr()), C.c_void_p(z.data_ptr()), C.c_void_p(ze.data_ptr())))
        return aw.t(), z.t(), ze.t()

    def apply(self, x):
        return self.apply_block(x)[:, 0]

    def apply_adjoint(self, y):
        return self.apply_adjoint_block(y)[:, 0]

    def column_norms(self):
        torch = _torch()
        out = torch.empty(self.n, dtype=torch.float64, device=self.device)
        check(lib().msvd_column_norms(self.handle, C.c_void_p(out.data_ptr())))
        return out

    def to_dense(self):
        return self.a[:, : self.n]

    def close(self):
        if getattr(self, "handle", None):
            lib().msvd_matrix_detach(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceCsrOperator(DeviceDenseOperator):
    """operator.hpp:58-74 CsrOperator over device memory (csr.hpp:10-25).

    `row_offsets` (int64, m_local + 1), `col_indices` (int32 or int64, sorted
    and unique within each row) and `values` (float64) are CUDA tensors holding
    this rank's rows; row0/m_global place them in the global matrix.  The
    structure is validated like CsrMatrix::validate (csr.cpp:9-31) when the
    operator is built, and its transpose is formed once on the device.
    """

    def __init__(self, row_offsets, col_indices, values, n, ctx: Optional[Context] = None, row0=0, m_global=None):
        torch = _torch()
        for t, name in ((row_offsets, "row_offsets"), (col_indices, "col_indices"), (values, "values")):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dim() == 1 and t.is_contiguous()):
                raise DimensionError(f"DeviceCsrOperator: {name} must be a contiguous 1-D CUDA tensor")
        if row_offsets.dtype != torch.int64 or values.dtype != torch.float64:
            raise DimensionError("DeviceCsrOperator: row_offsets int64 and values float64 required")
        if col_indices.dtype not in (torch.int32, torch.int64):
            raise DimensionError("DeviceCsrOperator: col_indices must be int32 or int64")
        if col_indices.numel() != values.numel():
            raise DimensionError("CsrMatrix: col_indices and values length mismatch")
        self.rp, self.ci, self.vals = row_offsets, col_indices, values
        self.device = values.device
        self.ctx = ctx or default_context(self.device.index or 0)
        self.m_local = row_offsets.numel() - 1
        self.n = int(n)
        self.row0 = row0
        self.m_global = self.m_local if m_global is None else m_global
        self.nnz_local = values.numel()
        h = C.c_void_p()
        check(lib().msvd_csr_attach(self.ctx.handle, C.c_void_p(row_offsets.data_ptr()),
                                    C.c_void_p(col_indices.data_ptr()), col_indices.element_size(),
                                    C.c_void_p(values.data_ptr()), self.m_local, self.n, self.nnz_local, row0,
                                    self.m_global, C.byref(h)))
        self.handle = h

    @classmethod
    def from_scipy(cls, a, device="cuda:0", index_dtype=None, **kw):
        """Upload a scipy.sparse CSR matrix (indices sorted) to the device."""
        torch = _torch()
        a = a.tocsr()
        a.sort_indices()
        idx = index_dtype or torch.int64
        rp = torch.as_tensor(np.asarray(a.indptr, dtype=np.int64), device=device)
        ci = torch.as_tensor(np.asarray(a.indices), device=device).to(idx)
        v = torch.as_tensor(np.asarray(a.data, dtype=np.float64), device=device)
        return cls(rp, ci, v, a.shape[1], **kw)

    def nnz(self):
        return self.nnz_local

    def to_dense(self):
        torch = _torch()
        out = torch.zeros((self.m_local, self.n), dtype=torch.float64, device=self.device)
        rows = torch.repeat_interleave(torch.arange(self.m_local, device=self.device), self.rp[1:] - self.rp[:-1])
        out[rows, self.ci.long()] = self.vals
        return out


# ------------------------------------------------------------------ solve
class _ResultBuffers:
    def __init__(self, n, b, max_iter, want_precond, store):
        cap = max_iter + 2
        self.sigma = np.zeros(b)
        self.v = np.zeros((b, n))  # row j = column j (column-major n x b)
        self.rows = (abi.RecordRow * cap)()
        self.res = abi.Result()
        self.res.sigma = self.sigma.ctypes.data_as(C.POINTER(C.c_double))
        self.res.v = self.v.ctypes.data_as(C.POINTER(C.c_double))
        self.res.rows = self.rows
        self.res.rows_capacity = cap
        self.vt = self.sg = None
        if want_precond:
            self.vt = np.zeros((n, n))  # [j, i] = V(i, j) (column-major)
            self.sg = np.zeros(n)
            self.res.vtilde = self.vt.ctypes.data_as(C.POINTER(C.c_double))
            self.res.sigma_tilde = self.sg.ctypes.data_as(C.POINTER(C.c_double))
        self.trail = {"t": [], "v": []}

        def sink(_u, kind, it, data, r, c):
            arr = np.ctypeslib.as_array(data, shape=(int(c), int(r))).T.copy()
            self.trail["t" if kind == 0 else "v"].append(arr)

        self._cb = abi.ITERATE_FN(sink) if store else abi.ITERATE_FN()
        self.res.iterate_cb = self._cb

    def result(self, has_truth):
        r = self.res
        rows = [RecordRow(x.iter, x.matvecs_a, x.matvecs_at, x.wall_ms, x.theta, x.resid, x.relerr, x.sin_angle)
                for x in self.rows[: min(r.rows_count, r.rows_capacity)]]
        pre = Preconditioner(self.vt.T.copy() if self.vt is not None else None,
                             self.sg.copy() if self.sg is not None else None, r.sigma_max_estimate,
                             bool(r.floored), r.floor_count)
        return SolveResult(v=self.v.T.copy(), sigma=self.sigma.copy(),
                           status="converged" if r.status == 0 else "max_iter_reached",
                           record=ConvergenceRecord(rows, has_truth), precond=pre,
                           sigma_max_estimate=r.sigma_max_estimate, sketch_skipped=bool(r.sketch_skipped),
                           sketch_dim=r.sketch_dim, zeta=r.zeta, verify_count=r.verify_count,
                           max_cache_drift=r.max_cache_drift, degenerate_replacements=r.degenerate_replacements,
                           trail_t=self.trail["t"], trail_v=self.trail["v"],
                           timings_ms=dict(sketch=r.t_sketch_ms, svd=r.t_svd_ms, init=r.t_init_ms,
                                           loop=r.t_loop_ms, total=r.t_total_ms))


def _truth(truth, n):
    if truth is None:
        return None, None
    v = np.ascontiguousarray(truth.v_min, dtype=np.float64)
    if v.size != n:
        raise DimensionError("solver: ground-truth vector length mismatch")
    t = abi.Truth(float(truth.sigma_min), v.ctypes.data_as(C.POINTER(C.c_double)))
    return t, v


def _run(fn, a, kind, opts, truth, want_precond):
    if not isinstance(a, DeviceDenseOperator):
        raise DimensionError("msvd: the GPU solver accepts a DeviceDenseOperator or DeviceCsrOperator only "
                             "(no CPU fallback)")
    opts = opts or SolverOptions()
    o = opts.to_abi(kind)
    if fn == "msvd_rlobpcg_single":
        o.block_size = 1
    b = max(int(o.block_size), 1)
    max_iter = o.max_iter if o.max_iter >= 0 else (200 if b == 1 else 100)
    t, keep = _truth(truth, a.n)
    bufs = _ResultBuffers(a.n, b, max(max_iter, 0), want_precond, bool(o.store_iterates))
    check(getattr(lib(), fn)(a.handle, C.byref(o), C.byref(t) if t is not None else None, C.byref(bufs.res)))
    del keep
    return bufs.result(truth is not None)


def lobpcg_solve(a, kind=PrecondKind.randomized, opts=None, truth=None, want_precond=False):
    """solver.hpp:172-173"""
    return _run("msvd_lobpcg_solve", a, kind, opts, truth, want_precond)


def rlobpcg_single(a, opts=None, truth=None, want_precond=False):
    """solver.hpp:176-177 (block size forced to 1)"""
    return _run("msvd_rlobpcg_single", a, abi.PRECOND_RANDOMIZED, opts, truth, want_precond)


def rlobpcg_block(a, opts=None, truth=None, want_precond=False):
    """solver.hpp:180-181"""
    return _run("msvd_rlobpcg_block", a, abi.PRECOND_RANDOMIZED, opts, truth, want_precond)


# ------------------------------------------- raw binary A interchange
def raw_write(path, a):
    """Write a 2-D float64 array (row-major rows) as an MSVDRAW1 file."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise DimensionError("raw_write: need a 2-D array")
    check(lib().msvd_raw_write(os.fsencode(path), a.ctypes.data_as(C.c_void_p), a.shape[0], a.shape[1],
                               a.shape[1]))


def raw_info(path):
    """(m, n) of an MSVDRAW1 file."""
    m, n = C.c_int64(), C.c_int64()
    check(lib().msvd_raw_info(os.fsencode(path), C.byref(m), C.byref(n)))
    return m.value, n.value


def raw_read(path, row0=0, rows=None):
    """Rows [row0, row0 + rows) as a host float64 array."""
    m, n = raw_info(path)
    rows = m - row0 if rows is None else rows
    out = np.empty((max(rows, 0), n), dtype=np.float64)
    check(lib().msvd_raw_read_rows(os.fsencode(path), row0, rows, out.ctypes.data_as(C.c_void_p), n))
    return out


def raw_load_device(path, row0=0, rows=None, ctx: Optional["Context"] = None, device=0):
    """Rows [row0, row0 + rows) straight into a row-major CUDA float64 tensor
    (a rank's shard of a row-sharded run)."""
    torch = _torch()
    m, n = raw_info(path)
    rows = m - row0 if rows is None else rows
    ctx = ctx or default_context(device)
    out = torch.empty((max(rows, 0), n), dtype=torch.float64, device=f"cuda:{ctx.device}")
    check(lib().msvd_raw_load_device(ctx.handle, os.fsencode(path), row0, rows, C.c_void_p(out.data_ptr()), n))
    return out


# ------------------------------------------------ baselines.hpp:12-42
def lobpcg_generic(a, kind=PrecondKind.randomized, opts=None, truth=None, want_precond=False):
    """baselines.hpp:12-14: LOBPCG with a selectable preconditioner kind."""
    return lobpcg_solve(a, kind, opts, truth, want_precond)


def sketch_and_solve_init(precond, b):
    """precond.cpp:50-57: the last b columns of V-tilde."""
    vt = precond.vtilde
    if vt is None:
        raise DimensionError("sketch_and_solve_init: preconditioner factors were not requested")
    n = vt.shape[0]
    if b < 1 or b > n:
        raise DimensionError("sketch_and_solve_init: block size out of range")
    return vt[:, n - b:].copy()


class LanczosStatus:
    completed = "completed"
    invariant_subspace = "invariant_subspace"


@dataclass
class LanczosResult:
    """baselines.hpp:25-33"""

    sigma_min: float
    v: np.ndarray
    record: ConvergenceRecord
    status: str
    steps: int
    v_basis: Optional[np.ndarray] = None
    u_basis: Optional[np.ndarray] = None


def lanczos_gk(a, iters, v0, truth=None, record_timing=True, want_bases=False):
    """baselines.cpp:51-166 on the device (msvd_lanczos_gk)."""
    if not isinstance(a, DeviceDenseOperator):
        raise DimensionError("msvd: lanczos_gk accepts a DeviceDenseOperator only (no CPU fallback)")
    v0 = np.ascontiguousarray(np.asarray(v0, dtype=np.float64).reshape(-1))
    if v0.size != a.n:
        raise DimensionError("lanczos_gk: starting vector length mismatch")
    t, keep = _truth(truth, a.n) if truth is not None else (None, None)
    if truth is not None and keep.size != a.n:
        raise DimensionError("lanczos_gk: ground-truth vector length mismatch")
    cap = max(int(iters), 1)
    rows = (abi.RecordRow * cap)()
    v = np.zeros(a.n)
    r = abi.LanczosResult()
    r.v = v.ctypes.data_as(C.POINTER(C.c_double))
    r.rows = rows
    r.rows_capacity = cap
    vb = ub = None
    if want_bases:
        vb = np.zeros((a.n, cap), order="F")
        ub = np.zeros((a.m_local, cap), order="F")
        r.v_basis = vb.ctypes.data_as(C.POINTER(C.c_double))
        r.u_basis = ub.ctypes.data_as(C.POINTER(C.c_double))
    check(lib().msvd_lanczos_gk(a.handle, int(iters), v0.ctypes.data_as(C.c_void_p),
                                C.byref(t) if t is not None else None, int(bool(record_timing)), C.byref(r)))
    del keep
    recs = [RecordRow(x.iter, x.matvecs_a, x.matvecs_at, x.wall_ms, x.theta, x.resid, x.relerr, x.sin_angle)
            for x in rows[:min(r.rows_count, cap)]]
    steps = r.steps
    return LanczosResult(sigma_min=r.sigma_min, v=v, record=ConvergenceRecord(recs, truth is not None),
                         status=(LanczosStatus.completed if r.status == abi.LANCZOS_COMPLETED
                                 else LanczosStatus.invariant_subspace), steps=steps,
                         v_basis=None if vb is None else vb[:, :steps].copy(order="F"),
                         u_basis=None if ub is None else ub[:, :steps].copy(order="F"))


def solve_host(a_host, opts=None, truth=None, ctx=None, row0=0, m_global=None, kind=abi.PRECOND_RANDOMIZED,
               want_precond=False):
    """End-to-end entry (msvd_solve_host): A in host memory (row-major numpy,
    ideally pinned), copied to the device inside the call."""
    a_host = np.asarray(a_host)
    if a_host.dtype != np.float64 or a_host.ndim != 2 or a_host.strides[1] != 8:
        raise DimensionError("solve_host needs a row-major float64 2-D array")
    ctx = ctx or default_context(0)
    m, n = a_host.shape
    ld = a_host.strides[0] // 8 if m > 1 else n
    opts = opts or SolverOptions()
    o = opts.to_abi(kind)
    b = max(int(o.block_size), 1)
    max_iter = o.max_iter if o.max_iter >= 0 else (200 if b == 1 else 100)
    t, keep = _truth(truth, n)
    bufs = _ResultBuffers(n, b, max(max_iter, 0), want_precond, bool(o.store_iterates))
    check(lib().msvd_solve_host(ctx.handle, C.c_void_p(a_host.ctypes.data), m, n, ld, row0,
                                m if m_global is None else m_global, C.byref(o),
                                C.byref(t) if t is not None else None, C.byref(bufs.res)))
    del keep
    return bufs.result(truth is not None)


@dataclass
class StopDecision:
    """solver.hpp:145-155"""

    tol_ok: bool = False
    resid_stalled: bool = False
    progress_stalled: bool = False
    stop: bool = False


def check_convergence(resid_hist, theta_hist, i, sigma1_estimate, tol, factor=1.1, use_stagnation=True, ctx=None):
    """solver.cpp:177-211, evaluated by the device solver's stop rule (the
    control kernel's code) on a host history (msvd_check_convergence)."""
    ctx = ctx or default_context(0)
    rh = np.ascontiguousarray(resid_hist, dtype=np.float64)
    th = np.ascontiguousarray(theta_hist, dtype=np.float64)
    n = min(rh.size, th.size)
    flags = (C.c_int32 * 4)()
    check(lib().msvd_check_convergence(ctx.handle, rh.ctypes.data_as(C.POINTER(C.c_double)),
                                       th.ctypes.data_as(C.POINTER(C.c_double)), n, int(i), float(sigma1_estimate),
                                       float(tol), float(factor), int(bool(use_stagnation)), flags))
    return StopDecision(*(bool(x) for x in flags))


def validate_options(m, n, opts: SolverOptions, kind=abi.PRECOND_RANDOMIZED):
    """Host-only check of the reference's option/shape validation order."""
    o = opts.to_abi(kind)
    check(lib().msvd_validate_options(m, n, C.byref(o), None))
