/*
 * msvd.h -- C ABI of libmsvd_cuda.so, the B200-native RLOBPCG hot path.
 *
 * This is the drop-in boundary for the reference's C++ solve API
 * (minsvd, /root/reference/proj/include/minsvd/solver.hpp).  Every function
 * returns an msvd_status, never throws across the boundary, and records a
 * thread-local message readable with msvd_last_error().  Status codes map 1:1
 * onto the reference's exception classes (errors.hpp:9-38); the C++ wrapper
 * include/minsvd_gpu.hpp rethrows them as those classes.
 *
 * Layout conventions
 *   A            device, ROW-major, m_local x n, leading dimension ld >= n
 *                (ld even enables the 16-byte TMA bulk path; every kernel
 *                requires 8*ld*rows chunks to be 16-byte aligned).
 *   n x b blocks column-major (leading dimension n), like minsvd::DenseMatrix.
 *   m x b blocks column-major (leading dimension m_local).
 *
 * Reference interface each entry point replaces is cited beside it.
 */
#ifndef MSVD_H_
#define MSVD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSVD_ABI_VERSION 1

/* errors.hpp:9-38 -> status codes */
typedef enum msvd_status {
    MSVD_OK = 0,
    MSVD_ERR_DIMENSION = 1,   /* minsvd::DimensionError   */
    MSVD_ERR_IO = 2,          /* minsvd::IoError          */
    MSVD_ERR_NUMERICAL = 3,   /* minsvd::NumericalError   */
    MSVD_ERR_CONVERGENCE = 4, /* minsvd::ConvergenceError */
    MSVD_ERR_CUDA = 5,        /* device failure  -> minsvd::Error */
    MSVD_ERR_COMM = 6,        /* NCCL / comm failure -> minsvd::Error */
    MSVD_ERR_INVALID = 7      /* bad handle / null pointer -> minsvd::Error */
} msvd_status;

/* solver.hpp:14 PrecondKind */
typedef enum msvd_precond_kind {
    MSVD_PRECOND_NONE = 0,
    MSVD_PRECOND_DIAGONAL = 1,
    MSVD_PRECOND_RANDOMIZED = 2
} msvd_precond_kind;

/* solver.hpp:25-78 SolverOptions, field by field (same defaults). */
typedef struct msvd_options {
    double tol;                 /* <0: default_tolerance(n) = 2 sqrt(n) eps   */
    int32_t max_iter;           /* <0: 200 if block_size==1 else 100          */
    int32_t check_every;        /* 5                                          */
    double stagnation_factor;   /* 1.1                                        */
    int64_t block_size;         /* 1                                          */
    uint64_t seed;              /* 0                                          */
    int64_t sketch_dim;         /* -1: round_up(4n, zeta), skip if m <= 4n     */
    int32_t zeta;               /* 4                                          */
    int32_t use_stagnation;     /* 1                                          */
    int32_t record_timing;      /* 1                                          */
    int32_t verify_cached_products; /* 0                                      */
    int32_t store_iterates;     /* 0                                          */
    int32_t precond_kind;       /* msvd_precond_kind, lobpcg_solve's `kind`   */
} msvd_options;

/* solver.hpp:93-102 RecordRow */
typedef struct msvd_record_row {
    int32_t iter;
    int32_t pad_;
    int64_t matvecs_a;
    int64_t matvecs_at;
    double wall_ms;
    double theta;
    double resid;
    double relerr;     /* -1 when no truth */
    double sin_angle;  /* -1 when no truth */
} msvd_record_row;

/* solver.hpp:87-90 GroundTruth (host memory) */
typedef struct msvd_truth {
    double sigma_min;
    const double* v_min;  /* length n, host */
} msvd_truth;

/* store_iterates sink: kind 0 = trial basis T (n x k), kind 1 = target block V
 * (n x b); data is host memory, column-major, valid during the call only.    */
typedef void (*msvd_iterate_fn)(void* user, int32_t kind, int32_t iter,
                                const double* data, int64_t rows, int64_t cols);

/* solver.hpp:118-137 SolveResult.  Arrays are caller-owned HOST buffers;
 * optional ones may be NULL.                                                  */
typedef struct msvd_result {
    double* sigma;              /* [b]  ascending from the smallest           */
    double* v;                  /* [n*b] column-major, ordered like sigma     */
    msvd_record_row* rows;      /* [rows_capacity]                            */
    int32_t rows_capacity;      /* >= max_iter + 1 to receive every row       */
    int32_t rows_count;         /* out: record.rows.size()                    */
    int32_t status;             /* out: 0 converged, 1 max_iter_reached       */
    int32_t iterations;         /* out: rows_count - 1                        */
    double* vtilde;             /* optional [n*n] column-major Preconditioner::vtilde */
    double* sigma_tilde;        /* optional [n]                               */
    double sigma_max_estimate;  /* out */
    int32_t floored;            /* out */
    int32_t sketch_skipped;     /* out */
    int64_t floor_count;        /* out */
    int64_t sketch_dim;         /* out (0 when skipped) */
    int32_t zeta;               /* out (0 when skipped) */
    int32_t pad_;
    int64_t verify_count;       /* out */
    double max_cache_drift;     /* out */
    int64_t degenerate_replacements; /* out */
    msvd_iterate_fn iterate_cb; /* store_iterates sink, may be NULL           */
    void* iterate_user;
    /* timing breakdown (device events, ms); not part of the reference record */
    double t_sketch_ms, t_svd_ms, t_init_ms, t_loop_ms, t_total_ms;
} msvd_result;

typedef struct msvd_ctx msvd_ctx;
typedef struct msvd_matrix msvd_matrix;

/* Communicator for row-sharded runs.  kind 0 = single rank,
 * 1 = NCCL (unique id from rank 0, 128 bytes), 2 = in-process fake group
 * (several host threads on one GPU, host-mediated reductions; for tests).   */
typedef struct msvd_ctx_desc {
    int32_t device;             /* CUDA ordinal                               */
    int32_t comm_kind;          /* 0 none, 1 nccl, 2 fake                     */
    int32_t nranks;
    int32_t rank;
    uint8_t nccl_id[128];       /* comm_kind 1                                */
    void* fake_group;           /* comm_kind 2: from msvd_fake_group_create   */
    void* stream;               /* cudaStream_t or NULL (library creates one) */
} msvd_ctx_desc;

/* ---- library / context ------------------------------------------------ */
int32_t msvd_abi_version(void);
const char* msvd_last_error(void);
const char* msvd_status_name(int32_t status);
void msvd_options_default(msvd_options* o);
/* solver.hpp:83-85 */
double msvd_default_tolerance(int64_t n);
/* Host-only validation of solver.cpp:306-315 + prepare() 128-145 checks; the
 * same status solve would return before touching the device.               */
int32_t msvd_validate_options(int64_t m, int64_t n, const msvd_options* o,
                              const msvd_truth* truth);
/* row range [row0, row0+rows) owned by `rank` when m rows are split evenly */
void msvd_shard_rows(int64_t m, int32_t nranks, int32_t rank, int64_t* row0,
                     int64_t* rows);

int32_t msvd_get_nccl_unique_id(uint8_t out[128]);
int32_t msvd_fake_group_create(int32_t nranks, void** group);
int32_t msvd_fake_group_destroy(void* group);
int32_t msvd_ctx_create(const msvd_ctx_desc* desc, msvd_ctx** out);
int32_t msvd_ctx_destroy(msvd_ctx* ctx);
int32_t msvd_ctx_synchronize(msvd_ctx* ctx);

/* ---- operator (operator.hpp:41-56 DenseOperator over device memory) ----- */
/* Borrowed device pointer, row-major m_local x n with leading dim ld; row0 =
 * global index of the first local row (keys the sketch), m_global = total.  */
int32_t msvd_matrix_attach(msvd_ctx* ctx, const double* dA, int64_t m_local,
                           int64_t n, int64_t ld, int64_t row0,
                           int64_t m_global, msvd_matrix** out);
int32_t msvd_matrix_detach(msvd_matrix* mat);
/* operator.hpp:58-74 CsrOperator over device memory (csr.hpp:10-25
 * CsrMatrix): borrowed row offsets (int64, m_local + 1), column indices
 * (index_bytes = 4 or 8, sorted and unique per row) and values (nnz), local
 * rows [row0, row0 + m_local) of an m_global x n operator.  Validated like
 * CsrMatrix::validate (csr.cpp:9-31: DimensionError / NumericalError with
 * the reference's messages); the transpose is built once here so adjoint
 * products are deterministic gathers.  Every entry point taking an
 * msvd_matrix (products, sketch, solves, lanczos) accepts it; the handle
 * must be released with msvd_matrix_detach.  Limits: < 2^31 local rows,
 * < 2^32 local nonzeros.                                                    */
int32_t msvd_csr_attach(msvd_ctx* ctx, const int64_t* dRowOffsets,
                        const void* dColIndices, int32_t index_bytes,
                        const double* dValues, int64_t m_local, int64_t n,
                        int64_t nnz, int64_t row0, int64_t m_global,
                        msvd_matrix** out);
/* operator.cpp:7-12 apply_block: dY (m_local x b) = A dX (n x b)           */
int32_t msvd_apply(msvd_matrix* mat, const double* dX, int64_t b, double* dY);
/* operator.cpp:14-19 apply_adjoint_block: dX (n x b) = A^T dY (m_local x b),
 * summed over ranks (allreduce) for sharded matrices.                       */
int32_t msvd_apply_adjoint(msvd_matrix* mat, const double* dY, int64_t b,
                           double* dX);
/* operator.cpp:151-161 column_norms: dNorms (n)                             */
int32_t msvd_column_norms(msvd_matrix* mat, double* dNorms);

/* ---- hot-path primitives --------------------------- */
/* sketch.cpp:36-60 build_sparsestack into device arrays (m*zeta each)       */
int32_t msvd_build_sparsestack(msvd_ctx* ctx, int64_t d, int64_t m, int32_t zeta,
                               uint64_t seed, uint32_t* dPositions,
                               int8_t* dSigns);
/* sketch.cpp:75-95 / 120-126 sketch_apply(S, A): dSA (d x n, col-major),
 * reduced over ranks.                                                       */
int32_t msvd_sketch(msvd_matrix* mat, int64_t d, int32_t zeta, uint64_t seed,
                    double* dSA);
/* precond.cpp:11-36 build_preconditioner from dSA (rows x n col-major):
 * dVt (n x n col-major), dSig (n), floored values raised.                   */
int32_t msvd_precond_build(msvd_ctx* ctx, const double* dSA, int64_t rows,
                           int64_t n, double* dVt, double* dSig,
                           double* sigma_max_estimate, int64_t* floor_count);
/* precond.cpp:38-48 precond_apply per column: dW = Vt diag(sig^-2) Vt^T dR  */
int32_t msvd_precond_apply(msvd_ctx* ctx, const double* dVt, const double* dSig,
                           int64_t n, const double* dR, int64_t b, double* dW);
/* svd.cpp:21-55 householder_qr R factor of a tall dT (rows x k col-major),
 * computed as a TSQR; dR (k x k col-major, upper).  Row signs are the
 * reference's only up to +-1 (R^T R identical).                             */
int32_t msvd_tsqr_r(msvd_ctx* ctx, const double* dT, int64_t rows, int64_t k,
                    double* dR);
/* The two passes of an iteration as primitives.
 * msvd_gram_apply -- residual_of solver.cpp:357-369 with the recurrence
 *   products :421/:462 (kernel K2): dY (m_local x q) = dT (m_local x k,
 *   col-major) dC (k x q, col-major) and dG (n x b) = A^T dY[:, 0:b], summed
 *   over ranks; b <= q <= 2b.  dC == NULL: Y = T (q == k == b), dY unused.  */
int32_t msvd_gram_apply(msvd_matrix* mat, const double* dT, int64_t k,
                        const double* dC, int64_t q, int64_t b, double* dG,
                        double* dY);
/* msvd_aw_tsqr -- solver.cpp:412-416 (kernel K3): dAW (m_local x b) = A dW,
 *   and dR (k x k, k = kl + b, upper) = the Householder R factor of the trial
 *   block [dLead (m_local x kl) | AW] (svd.cpp:21-55, row signs up to +-1),
 *   merged over CTAs and ranks.  kl = 0: dLead unused.                      */
int32_t msvd_aw_tsqr(msvd_matrix* mat, const double* dW, int64_t b,
                     const double* dLead, int64_t kl, double* dAW, double* dR);
/* msvd_aw_gram -- the one-pass primitive: dAW (m_local x b) = A dW and
 *   dZ (n x b) = A^T (A dW), summed over ranks, from ONE pass over A.  Where
 *   the register-resident kernel does not fit (b * ceil(n/64) > 16 lanes'
 *   worth) it makes the two passes instead.                                 */
int32_t msvd_aw_gram(msvd_matrix* mat, const double* dW, int64_t b, double* dAW,
                     double* dZ);
/* msvd_aw_gram_ex -- the one-pass check refresh (solver.cpp:439 evaluated on
 *   the next pass): dAW = A dW, dZ (n x b) = A^T (A dW) and dZE (n x b) =
 *   A^T dE for dE (m_local x b, col-major; the solver passes E = A V' of the
 *   previous check iterate), all from ONE pass over A, summed over ranks.
 *   MSVD_ERR_INVALID where the shape has no such kernel (b > 4, wide n).    */
int32_t msvd_aw_gram_ex(msvd_matrix* mat, const double* dW, int64_t b, const double* dE,
                        double* dAW, double* dZ, double* dZE);
/* svd.cpp:180-252 dense_svd(B, false) of a small square dB (k x k, k<=32)
 * already reduced to R: sigma descending, V sign-fixed.                     */
int32_t msvd_small_svd(msvd_ctx* ctx, const double* dB, int64_t k,
                       double* dSigma, double* dV);
/* solver.cpp:177-211 check_convergence, evaluated by the device solver's own
 * stop rule (the control kernel's code) on a HOST history of `len` rows:
 * flags[4] = {tol_ok, resid_stalled, progress_stalled, stop}.  Throws
 * (DimensionError) like the reference when i + 1 >= len.                   */
int32_t msvd_check_convergence(msvd_ctx* ctx, const double* resid_hist, const double* theta_hist,
                               int64_t len, int32_t i, double sigma1_estimate, double tol,
                               double factor, int32_t use_stagnation, int32_t* flags);

/* ---- raw binary A interchange -----------------------
 * The dense-matrix counterpart of write_matrix_market_array / read (io.cpp:
 * 174-184, :96-172) without the text: a 32-byte header ("MSVDRAW1", int64 m,
 * int64 n, int32 layout = 0 row-major, int32 0) then m*n little-endian fp64,
 * row-major.  Exact round trip; a row range is one contiguous byte range.
 * Errors: MSVD_ERR_IO (IoError) for open / read / write / format failures.  */
int32_t msvd_raw_write(const char* path, const double* hA, int64_t m, int64_t n,
                       int64_t ld);
int32_t msvd_raw_info(const char* path, int64_t* m, int64_t* n);
/* rows [row0, row0 + rows) into host memory (leading dimension ld)          */
int32_t msvd_raw_read_rows(const char* path, int64_t row0, int64_t rows,
                           double* hA, int64_t ld);
/* the same rows straight into device memory (row-major, leading dimension
 * ld), through pinned staging buffers: a rank's shard of a row-sharded run */
int32_t msvd_raw_load_device(msvd_ctx* ctx, const char* path, int64_t row0,
                             int64_t rows, double* dA, int64_t ld);

/* ---- Krylov baseline (baselines.cpp:51-166 lanczos_gk) ----------------- */
/* baselines.hpp:20-23 LanczosStatus */
typedef enum msvd_lanczos_status {
    MSVD_LANCZOS_COMPLETED = 0,
    MSVD_LANCZOS_INVARIANT_SUBSPACE = 1
} msvd_lanczos_status;

/* baselines.hpp:25-33 LanczosResult.  Arrays are caller-owned HOST buffers;
 * the bases are optional (NULL skips the copy).                             */
typedef struct msvd_lanczos_result {
    double sigma_min;           /* out: smallest Ritz value of the final section */
    double* v;                  /* [n] matching right Ritz vector, unit norm     */
    msvd_record_row* rows;      /* [rows_capacity], one row per step             */
    int32_t rows_capacity;      /* >= iters to receive every row                 */
    int32_t rows_count;         /* out */
    int32_t status;             /* out: msvd_lanczos_status                      */
    int32_t steps;              /* out: sections evaluated                       */
    double* v_basis;            /* optional [n * iters], first `steps` columns   */
    double* u_basis;            /* optional [m_local * iters], first `steps` cols */
} msvd_lanczos_result;

/* baselines.cpp:51-166 lanczos_gk(a, iters, v0, truth, record_timing):
 * Golub-Kahan bidiagonalization from v0 (HOST, length n) with two-pass
 * reorthogonalization of both Krylov bases, on the device; the smallest
 * singular triplet of each bidiagonal section is found by bisection on its
 * Golub-Kahan tridiagonal plus inverse iteration (LAPACK dbdsvdx's route)
 * instead of the reference's dense Jacobi SVD of the section.              */
int32_t msvd_lanczos_gk(msvd_matrix* mat, int32_t iters, const double* v0,
                        const msvd_truth* truth, int32_t record_timing,
                        msvd_lanczos_result* res);

/* ---- full solve (solver.cpp:301-477, 479-489) ------------------------- */
int32_t msvd_lobpcg_solve(msvd_matrix* mat, const msvd_options* opts,
                          const msvd_truth* truth, msvd_result* res);
/* solver.cpp:479-484 (block size forced to 1) */
int32_t msvd_rlobpcg_single(msvd_matrix* mat, const msvd_options* opts,
                            const msvd_truth* truth, msvd_result* res);
/* solver.cpp:486-489 (precond_kind forced to randomized) */
int32_t msvd_rlobpcg_block(msvd_matrix* mat, const msvd_options* opts,
                           const msvd_truth* truth, msvd_result* res);
/* End-to-end convenience: A in HOST memory (row-major, pinned or pageable);
 * copies the local rows to the device inside the call, then solves.        */
int32_t msvd_solve_host(msvd_ctx* ctx, const double* hA, int64_t m_local,
                        int64_t n, int64_t ld, int64_t row0, int64_t m_global,
                        const msvd_options* opts, const msvd_truth* truth,
                        msvd_result* res);

/* sizeof of {msvd_options, msvd_record_row, msvd_truth, msvd_result,
 * msvd_ctx_desc, msvd_lanczos_result} into out[0..n) (binding self-check;
 * host only). */
void msvd_abi_sizes(int64_t* out, int32_t n);

/* Number of library kernels launched since ctx creation (bench evidence). */
int64_t msvd_launch_count(msvd_ctx* ctx);
/* Per-kernel-class device time with CUDA events on the ctx stream.  Slots:
 * 0 apply (A W), 1 gram (A^T Y), 2 tsqr, 3 rayleigh-ritz, 4 sketch,
 * 5 precond build (SVD), 6 precond apply, 7 cgs2, 8 reduce, 9 control.
 * enable: 0 off, 1 the A-pass classes only (apply, gram: two events per pass,
 * negligible overhead), 2 every class.  Enabling resets the accumulators;
 * read synchronizes the stream.                                             */
int32_t msvd_ctx_profile(msvd_ctx* ctx, int32_t enable);
/* Bit mask of the A-pass kernel variants launched on ctx since the last reset
 * (test evidence that a shape took the path it is meant to):
 *   1 apply_rows (producer warp)      2 apply_self (TMA, one warp per row)
 *   4 apply_pair (warp pair per row)  8 apply_pair EX (b = 1 check refresh)
 *  16 (retired: the four-warp team check refresh)   32 apply ticket (b >= 5)
 *  64 gram (A^T Y pass)              128 separate TSQR pass
 * 256 the preconditioner from the Cholesky-QR route (no n x n SVD)
 * 512 (retired: the team one-pass pass)
 * 1024 apply_split (b = 2..4 one-pass pass: dot, acc and producer warps)
 * 2048 apply_split EX (b = 2..4 check refresh in the split-role form)
 * reset != 0 clears the mask after reading it.                             */
int64_t msvd_ctx_kernel_paths(msvd_ctx* ctx, int32_t reset);
int32_t msvd_ctx_profile_read(msvd_ctx* ctx, double* ms, int64_t* counts, int32_t nslots);

#ifdef __cplusplus
}
#endif

#endif /* MSVD_H_ */
