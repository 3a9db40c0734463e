"""ctypes mirrors of the plain C structs in include/msvd.h.

These are the ABI types of the drop-in boundary (libmsvd_cuda.so).  The field
order, widths and padding must match msvd.h exactly; tests/test_abi.py checks
the sizes against the compiled library.
"""
import ctypes as C

MSVD_OK = 0
MSVD_ERR_DIMENSION = 1
MSVD_ERR_IO = 2
MSVD_ERR_NUMERICAL = 3
MSVD_ERR_CONVERGENCE = 4
MSVD_ERR_CUDA = 5
MSVD_ERR_COMM = 6
MSVD_ERR_INVALID = 7

PRECOND_NONE = 0
PRECOND_DIAGONAL = 1
PRECOND_RANDOMIZED = 2


class Options(C.Structure):
    """solver.hpp:25-78 SolverOptions (msvd_options)."""

    _fields_ = [
        ("tol", C.c_double),
        ("max_iter", C.c_int32),
        ("check_every", C.c_int32),
        ("stagnation_factor", C.c_double),
        ("block_size", C.c_int64),
        ("seed", C.c_uint64),
        ("sketch_dim", C.c_int64),
        ("zeta", C.c_int32),
        ("use_stagnation", C.c_int32),
        ("record_timing", C.c_int32),
        ("verify_cached_products", C.c_int32),
        ("store_iterates", C.c_int32),
        ("precond_kind", C.c_int32),
    ]


class RecordRow(C.Structure):
    """solver.hpp:93-102 RecordRow (msvd_record_row)."""

    _fields_ = [
        ("iter", C.c_int32),
        ("pad_", C.c_int32),
        ("matvecs_a", C.c_int64),
        ("matvecs_at", C.c_int64),
        ("wall_ms", C.c_double),
        ("theta", C.c_double),
        ("resid", C.c_double),
        ("relerr", C.c_double),
        ("sin_angle", C.c_double),
    ]


class Truth(C.Structure):
    _fields_ = [("sigma_min", C.c_double), ("v_min", C.POINTER(C.c_double))]


ITERATE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                         C.c_int64, C.c_int64)


class Result(C.Structure):
    """solver.hpp:118-137 SolveResult (msvd_result); arrays are caller-owned."""

    _fields_ = [
        ("sigma", C.POINTER(C.c_double)),
        ("v", C.POINTER(C.c_double)),
        ("rows", C.POINTER(RecordRow)),
        ("rows_capacity", C.c_int32),
        ("rows_count", C.c_int32),
        ("status", C.c_int32),
        ("iterations", C.c_int32),
        ("vtilde", C.POINTER(C.c_double)),
        ("sigma_tilde", C.POINTER(C.c_double)),
        ("sigma_max_estimate", C.c_double),
        ("floored", C.c_int32),
        ("sketch_skipped", C.c_int32),
        ("floor_count", C.c_int64),
        ("sketch_dim", C.c_int64),
        ("zeta", C.c_int32),
        ("pad_", C.c_int32),
        ("verify_count", C.c_int64),
        ("max_cache_drift", C.c_double),
        ("degenerate_replacements", C.c_int64),
        ("iterate_cb", ITERATE_FN),
        ("iterate_user", C.c_void_p),
        ("t_sketch_ms", C.c_double),
        ("t_svd_ms", C.c_double),
        ("t_init_ms", C.c_double),
        ("t_loop_ms", C.c_double),
        ("t_total_ms", C.c_double),
    ]


LANCZOS_COMPLETED = 0
LANCZOS_INVARIANT_SUBSPACE = 1


class LanczosResult(C.Structure):
    """baselines.hpp:25-33 LanczosResult (msvd_lanczos_result); arrays are
    caller-owned."""

    _fields_ = [
        ("sigma_min", C.c_double),
        ("v", C.POINTER(C.c_double)),
        ("rows", C.POINTER(RecordRow)),
        ("rows_capacity", C.c_int32),
        ("rows_count", C.c_int32),
        ("status", C.c_int32),
        ("steps", C.c_int32),
        ("v_basis", C.POINTER(C.c_double)),
        ("u_basis", C.POINTER(C.c_double)),
    ]


class CtxDesc(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("comm_kind", C.c_int32),
        ("nranks", C.c_int32),
        ("rank", C.c_int32),
        ("nccl_id", C.c_uint8 * 128),
        ("fake_group", C.c_void_p),
        ("stream", C.c_void_p),
    ]


def default_options(**kw):
    """msvd_options_default() restated for hosts without the library loaded
    (the compiled default is checked against this in tests/test_abi.py)."""
    o = Options(tol=-1.0, max_iter=-1, check_every=5, stagnation_factor=1.1, block_size=1,
                seed=0, sketch_dim=-1, zeta=4, use_stagnation=1, record_timing=1,
                verify_cached_products=0, store_iterates=0, precond_kind=PRECOND_RANDOMIZED)
    for k, v in kw.items():
        if not hasattr(o, k):
            raise AttributeError(k)
        setattr(o, k, int(v) if isinstance(v, bool) else v)
    return o
