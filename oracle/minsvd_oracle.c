/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into, or called by, the
 * product path (paper_2602_16797_b200/, libmsvd_cuda.so).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs load it.
 *
 * A plain-C restatement of the reference's RLOBPCG algorithm for the hot path
 * (minsvd, /root/reference/proj): SplitMix64 streams, the SparseStack sketch,
 * Householder QR + one-sided Jacobi SVD, the randomized preconditioner and the
 * block LOBPCG driver with its record/stop logic.  Every routine keeps the
 * reference's floating-point operation order (no FMA: built with
 * -ffp-contract=off, like the reference's x86-64 baseline build), so its
 * outputs are BIT-IDENTICAL to the reference's; tests/test_oracle.py pins that
 * against oracle/_ref (the reference compiled from its own sources) and the
 * committed golden vectors in tests/golden/.  Parity status: PINNED.
 *
 * Matrices are column-major (minsvd::DenseMatrix, dense.hpp:14-50).
 * Errors unwind with longjmp to the exported entry point and map onto the
 * msvd_status codes of include/msvd.h (errors.hpp:9-38).
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "msvd.h"

#define EPS 2.220446049250313e-16 /* std::numeric_limits<double>::epsilon() */
#define GOLDEN 0x9E3779B97F4A7C15ULL

/* ------------------------------------------------------------------ errors */

static __thread jmp_buf *g_jmp;
static __thread char g_msg[512];
static __thread int g_code;
/* The input generators (haar_orthonormal, synth, assemble) split their column
 * loops over OpenMP threads: each output column is still computed by one thread
 * in the serial operation order, so the bytes do not depend on the thread count
 * (tests/test_oracle.py pins them to the reference).  Everything else, the
 * solver included, stays single-threaded like the reference. */
static __thread int g_par;

typedef struct blk { struct blk *next; void *pad; } blk; /* 16-byte header */
static __thread blk *g_arena;

static void raise_err(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_msg, sizeof g_msg, fmt, ap);
    va_end(ap);
    g_code = code;
    longjmp(*g_jmp, 1);
}

/* zeroed allocation owned by the current call; freed by arena_release */
static void *zalloc(size_t bytes) {
    blk *b = (blk *)calloc(1, sizeof(blk) + (bytes ? bytes : 1));
    if (!b) raise_err(MSVD_ERR_INVALID, "oracle: out of memory");
    b->next = g_arena;
    g_arena = b;
    return (void *)(b + 1);
}

static void arena_release(void) {
    while (g_arena) {
        blk *n = g_arena->next;
        free(g_arena);
        g_arena = n;
    }
}

#define ENTER()                          \
    jmp_buf jb__;                        \
    jmp_buf *saved__ = g_jmp;            \
    blk *arena__ = g_arena;              \
    g_arena = NULL;                      \
    g_jmp = &jb__;                       \
    if (setjmp(jb__)) {                  \
        g_par = 0;                       \
        arena_release();                 \
        g_arena = arena__;               \
        g_jmp = saved__;                 \
        return g_code;                   \
    }
#define LEAVE()          \
    do {                 \
        arena_release(); \
        g_arena = arena__; \
        g_jmp = saved__; \
        return 0;        \
    } while (0)

const char *orc_last_error(void) { return g_msg; }

/* ---------------------------------------------------- SplitMix64 (rng.hpp) */

typedef struct {
    uint64_t s;
    double spare;
    int have_spare;
} sm64;

static uint64_t sm_mix(uint64_t z) { /* rng.hpp:55-59 */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static sm64 sm_plain(uint64_t seed) { sm64 r = {seed, 0.0, 0}; return r; }      /* rng.hpp:16 */
static sm64 sm_keyed(uint64_t seed, uint64_t key) {                             /* rng.hpp:18-19 */
    sm64 r = {sm_mix(seed + GOLDEN * (key + 1)), 0.0, 0};
    return r;
}
static uint64_t sm_u64(sm64 *r) { r->s += GOLDEN; return sm_mix(r->s); }     /* rng.hpp:21-24 */
static uint64_t sm_below(sm64 *r, uint64_t bound) {                           /* rng.hpp:27-32 */
    const uint64_t lim = UINT64_MAX - UINT64_MAX % bound;
    uint64_t x = sm_u64(r);
    while (x >= lim) x = sm_u64(r);
    return x % bound;
}
static double sm_unit(sm64 *r) { return (double)((sm_u64(r) >> 11) + 1) * 0x1.0p-53; } /* :35-37 */
static double sm_gauss(sm64 *r) {                                             /* rng.hpp:40-52 */
    if (r->have_spare) { r->have_spare = 0; return r->spare; }
    double u1 = sm_unit(r), u2 = sm_unit(r);
    double rad = sqrt(-2.0 * log(u1));
    double ang = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(ang);
    r->have_spare = 1;
    return rad * cos(ang);
}

/* --------------------------------------------------- dense (dense.cpp) */

typedef struct { int64_t r, c; double *p; } mat; /* column-major */

static mat mnew(int64_t r, int64_t c) {
    if (r < 0 || c < 0) raise_err(MSVD_ERR_DIMENSION, "DenseMatrix: negative dimension");
    mat m = {r, c, (double *)zalloc(sizeof(double) * (size_t)(r * c))};
    return m;
}
static double *col(mat m, int64_t j) { return m.p + j * m.r; }
#define AT(m, i, j) ((m).p[(j) * (m).r + (i)])
static mat mcopy(mat a) { mat o = mnew(a.r, a.c); memcpy(o.p, a.p, sizeof(double) * (size_t)(a.r * a.c)); return o; }
static mat mview(double *p, int64_t r, int64_t c) { mat m = {r, c, p}; return m; }
static mat meye(int64_t n) { mat m = mnew(n, n); for (int64_t i = 0; i < n; ++i) AT(m, i, i) = 1.0; return m; }

static double vdot(const double *a, const double *b, int64_t n) { /* dense.cpp:9-14 */
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
static double vnorm(const double *a, int64_t n) { return sqrt(vdot(a, a, n)); } /* :16-18 */
static void vscale(double *a, int64_t n, double s) { for (int64_t i = 0; i < n; ++i) a[i] *= s; }
static int finite_all(const double *a, int64_t n) {
    for (int64_t i = 0; i < n; ++i) if (!isfinite(a[i])) return 0;
    return 1;
}

/* y = M x, column sweeps (dense.cpp:50-60) */
static void matvec(mat m, const double *x, double *y) {
    for (int64_t i = 0; i < m.r; ++i) y[i] = 0.0;
    for (int64_t j = 0; j < m.c; ++j) {
        const double xj = x[j];
        const double *c = col(m, j);
        for (int64_t i = 0; i < m.r; ++i) y[i] += xj * c[i];
    }
}
/* y = M^T x, column dots (dense.cpp:62-73) */
static void matvec_t(mat m, const double *x, double *y) {
    for (int64_t j = 0; j < m.c; ++j) y[j] = vdot(col(m, j), x, m.r);
}
/* C = A B, skipping zero coefficients (dense.cpp:75-89) */
static mat matmul(mat a, mat b) {
    if (a.c != b.r) raise_err(MSVD_ERR_DIMENSION, "matmul: dimension mismatch");
    mat c = mnew(a.r, b.c);
#pragma omp parallel for schedule(static) if (g_par && a.r * a.c > 65536)
    for (int64_t j = 0; j < b.c; ++j) {
        double *cj = col(c, j);
        for (int64_t k = 0; k < a.c; ++k) {
            const double bkj = AT(b, k, j);
            if (bkj == 0.0) continue;
            const double *ak = col(a, k);
            for (int64_t i = 0; i < a.r; ++i) cj[i] += bkj * ak[i];
        }
    }
    return c;
}
static mat transpose(mat a) {
    mat t = mnew(a.c, a.r);
    for (int64_t j = 0; j < a.c; ++j)
        for (int64_t i = 0; i < a.r; ++i) AT(t, j, i) = AT(a, i, j);
    return t;
}
static double colnorm_from(mat a, int64_t j, int64_t from) { /* svd.cpp:12-17 */
    const double *c = col(a, j);
    double s = 0.0;
    for (int64_t i = from; i < a.r; ++i) s += c[i] * c[i];
    return sqrt(s);
}
static double max_colnorm(mat a) { /* solver.cpp:16-27 */
    double best = 0.0;
    for (int64_t j = 0; j < a.c; ++j) {
        double v = colnorm_from(a, j, 0);
        if (v > best) best = v;
    }
    return best;
}

/* --------------------------------------------------------- QR + SVD (svd.cpp) */

typedef struct { mat a; double *beta; } hqr;

/* Householder QR, reflectors stored below the diagonal (svd.cpp:21-55) */
static hqr qr_factor(mat a_in) {
    if (!finite_all(a_in.p, a_in.r * a_in.c)) raise_err(MSVD_ERR_NUMERICAL, "householder_qr: non-finite entry");
    const int64_t m = a_in.r, n = a_in.c;
    if (m < n) raise_err(MSVD_ERR_DIMENSION, "householder_qr: requires rows >= cols");
    hqr q = {mcopy(a_in), (double *)zalloc(sizeof(double) * (size_t)(n ? n : 1))};
    mat w = q.a;
    for (int64_t k = 0; k < n; ++k) {
        double *ck = col(w, k);
        const double xn = colnorm_from(w, k, k);
        if (xn == 0.0) { q.beta[k] = 0.0; continue; }
        const double alpha = ck[k] >= 0.0 ? -xn : xn;
        const double v0 = ck[k] - alpha;
        for (int64_t i = k + 1; i < m; ++i) ck[i] /= v0;
        q.beta[k] = -v0 / alpha;
        ck[k] = alpha;
        const double beta = q.beta[k];
#pragma omp parallel for schedule(static) if (g_par && (m - k) * (n - k) > 65536)
        for (int64_t j = k + 1; j < n; ++j) {
            double *cj = col(w, j);
            double s = cj[k];
            for (int64_t i = k + 1; i < m; ++i) s += ck[i] * cj[i];
            s *= beta;
            cj[k] -= s;
            for (int64_t i = k + 1; i < m; ++i) cj[i] -= s * ck[i];
        }
    }
    return q;
}
static mat qr_rfactor(hqr q) { /* svd.cpp:57-63 */
    const int64_t n = q.a.c;
    mat r = mnew(n, n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i <= j; ++i) AT(r, i, j) = AT(q.a, i, j);
    return r;
}
/* Q [B; 0] (svd.cpp:65-88) */
static mat qr_q_times(hqr q, mat b) {
    const int64_t m = q.a.r, n = q.a.c;
    if (b.r != n) raise_err(MSVD_ERR_DIMENSION, "qr_apply_q: dimension mismatch");
    mat y = mnew(m, b.c);
    for (int64_t j = 0; j < b.c; ++j)
        for (int64_t i = 0; i < n; ++i) AT(y, i, j) = AT(b, i, j);
    for (int64_t k = n - 1; k >= 0; --k) {
        const double beta = q.beta[k];
        if (beta == 0.0) continue;
        const double *vk = col(q.a, k);
#pragma omp parallel for schedule(static) if (g_par && (m - k) * y.c > 65536)
        for (int64_t j = 0; j < y.c; ++j) {
            double *cj = col(y, j);
            double s = cj[k];
            for (int64_t i = k + 1; i < m; ++i) s += vk[i] * cj[i];
            s *= beta;
            cj[k] -= s;
            for (int64_t i = k + 1; i < m; ++i) cj[i] -= s * vk[i];
        }
    }
    return y;
}

/* cyclic one-sided Jacobi on the columns of b, rotations accumulated in v
 * (svd.cpp:99-150: tolerance 1e-15, 60 sweeps, row-cyclic pair order)       */
static void jacobi_sweeps(mat b, mat v) {
    const int64_t s = b.r, n = b.c;
    double worst = 0.0;
    for (int sweep = 0; sweep < 60; ++sweep) {
        worst = 0.0;
        for (int64_t p = 0; p + 1 < n; ++p) {
            for (int64_t q = p + 1; q < n; ++q) {
                double *bp = col(b, p), *bq = col(b, q);
                double app = 0.0, aqq = 0.0, apq = 0.0;
                for (int64_t i = 0; i < s; ++i) {
                    app += bp[i] * bp[i];
                    aqq += bq[i] * bq[i];
                    apq += bp[i] * bq[i];
                }
                if (app == 0.0 || aqq == 0.0 || apq == 0.0) continue;
                const double rel = fabs(apq) / sqrt(app * aqq);
                if (rel > worst) worst = rel;
                if (rel <= 1e-15) continue;
                const double tau = (aqq - app) / (2.0 * apq);
                const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double sn = c * t;
                for (int64_t i = 0; i < s; ++i) {
                    const double xp = bp[i], xq = bq[i];
                    bp[i] = c * xp - sn * xq;
                    bq[i] = sn * xp + c * xq;
                }
                double *vp = col(v, p), *vq = col(v, q);
                for (int64_t i = 0; i < n; ++i) {
                    const double xp = vp[i], xq = vq[i];
                    vp[i] = c * xp - sn * xq;
                    vq[i] = sn * xp + c * xq;
                }
            }
        }
        if (worst <= 1e-15) return;
    }
    raise_err(MSVD_ERR_NUMERICAL, "one_sided_jacobi: no convergence after 60 sweeps (n=%lld, worst pair cosine=%f)",
              (long long)n, worst);
}

typedef struct { double *sigma; mat v; } svdres;

/* dense_svd(m, want_u=false) (svd.cpp:180-252): QR-reduce tall inputs,
 * Jacobi, stable descending sort, largest-|entry|-positive column signs     */
static svdres svd_values_right(mat a) {
    if (!finite_all(a.p, a.r * a.c)) raise_err(MSVD_ERR_NUMERICAL, "dense_svd: non-finite entry");
    const int64_t rows = a.r, n = a.c;
    if (rows < n) raise_err(MSVD_ERR_DIMENSION, "dense_svd: requires rows >= cols");
    if (n == 0) raise_err(MSVD_ERR_DIMENSION, "dense_svd: empty matrix");
    mat b = rows > n ? qr_rfactor(qr_factor(a)) : mcopy(a);
    mat v = meye(n);
    jacobi_sweeps(b, v);
    double *sig = (double *)zalloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) sig[j] = colnorm_from(b, j, 0);
    int64_t *ord = (int64_t *)zalloc(sizeof(int64_t) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) ord[j] = j;
    for (int64_t j = 1; j < n; ++j) { /* stable insertion sort, descending */
        int64_t key = ord[j], i = j - 1;
        while (i >= 0 && sig[key] > sig[ord[i]]) { ord[i + 1] = ord[i]; --i; }
        ord[i + 1] = key;
    }
    svdres out = {(double *)zalloc(sizeof(double) * (size_t)n), mnew(n, n)};
    for (int64_t j = 0; j < n; ++j) {
        out.sigma[j] = sig[ord[j]];
        memcpy(col(out.v, j), col(v, ord[j]), sizeof(double) * (size_t)n);
    }
    for (int64_t j = 0; j < n; ++j) {
        double *c = col(out.v, j);
        int64_t imax = 0;
        double amax = -1.0;
        for (int64_t i = 0; i < n; ++i) if (fabs(c[i]) > amax) { amax = fabs(c[i]); imax = i; }
        if (c[imax] < 0.0) for (int64_t i = 0; i < n; ++i) c[i] = -c[i];
    }
    return out;
}

/* ---------------------------------------------------- sketch (sketch.cpp) */

typedef struct { int64_t d, m; int zeta; uint32_t *pos; int8_t *sgn; } sstack;

static sstack sstack_build(int64_t d, int64_t m, int zeta, uint64_t seed) { /* :36-60 */
    if (d <= 0 || m <= 0) raise_err(MSVD_ERR_DIMENSION, "build_sparsestack: dimensions must be positive");
    if (zeta <= 0 || zeta > d) raise_err(MSVD_ERR_DIMENSION, "build_sparsestack: zeta must be in [1, d]");
    if (d % zeta != 0)
        raise_err(MSVD_ERR_DIMENSION, "build_sparsestack: zeta must divide d; use round_up_to_multiple(d, zeta) = %lld",
                  (long long)(d + (zeta - d % zeta)));
    sstack s = {d, m, zeta, (uint32_t *)zalloc(sizeof(uint32_t) * (size_t)(m * zeta)),
                (int8_t *)zalloc((size_t)(m * zeta))};
    const uint64_t blk_rows = (uint64_t)(d / zeta);
    for (int64_t j = 0; j < m; ++j) {
        sm64 r = sm_keyed(seed, (uint64_t)j);
        for (int k = 0; k < zeta; ++k) {
            s.pos[j * zeta + k] = (uint32_t)sm_below(&r, blk_rows);
            s.sgn[j * zeta + k] = (sm_u64(&r) >> 63) ? -1 : 1;
        }
    }
    return s;
}

/* S A for a dense column-major A, columns outer, rows ascending (:75-95) */
static mat sstack_apply(sstack s, mat a) {
    if (a.r != s.m)
        raise_err(MSVD_ERR_DIMENSION, "sketch_apply: operand has %lld rows, embedding expects %lld",
                  (long long)a.r, (long long)s.m);
    mat out = mnew(s.d, a.c);
    const double val = 1.0 / sqrt((double)s.zeta);
    const int64_t blk_rows = s.d / s.zeta;
    for (int64_t j = 0; j < a.c; ++j) {
        const double *aj = col(a, j);
        double *oj = col(out, j);
        for (int64_t r = 0; r < s.m; ++r) {
            const double x = aj[r];
            if (x == 0.0) continue;
            for (int k = 0; k < s.zeta; ++k)
                oj[blk_rows * k + s.pos[r * s.zeta + k]] += (double)s.sgn[r * s.zeta + k] * val * x;
        }
    }
    return out;
}

/* ------------------------------------------------------- CSR (csr.cpp) */

typedef struct { int64_t rows, cols; const int64_t *rp, *ci; const double *v; } csr;

static int64_t csr_nnz(csr a) { return a.rp[a.rows]; }

/* CsrMatrix::validate (csr.cpp:9-31), same checks in the same order */
static void csr_validate(csr a, int64_t nnz) {
    if (a.rows < 0 || a.cols < 0) raise_err(MSVD_ERR_DIMENSION, "CsrMatrix: negative dimension");
    if (a.rp[0] != 0 || a.rp[a.rows] != nnz)
        raise_err(MSVD_ERR_DIMENSION, "CsrMatrix: row_offsets endpoints inconsistent with nnz");
    for (int64_t i = 0; i < a.rows; ++i) {
        if (a.rp[i] > a.rp[i + 1])
            raise_err(MSVD_ERR_DIMENSION, "CsrMatrix: row_offsets not nondecreasing at row %lld", (long long)i);
        for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const int64_t j = a.ci[k];
            if (j < 0 || j >= a.cols)
                raise_err(MSVD_ERR_DIMENSION, "CsrMatrix: column index out of range in row %lld", (long long)i);
            if (k > a.rp[i] && a.ci[k - 1] >= j)
                raise_err(MSVD_ERR_DIMENSION, "CsrMatrix: column indices not strictly increasing in row %lld",
                          (long long)i);
        }
    }
    for (int64_t k = 0; k < nnz; ++k)
        if (!isfinite(a.v[k])) raise_err(MSVD_ERR_NUMERICAL, "CsrMatrix: non-finite value");
}
/* CsrMatrix::matvec (csr.cpp:33-44) */
static void csr_matvec(csr a, const double *x, double *y) {
    for (int64_t i = 0; i < a.rows; ++i) {
        double s = 0.0;
        for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k) s += a.v[k] * x[a.ci[k]];
        y[i] = s;
    }
}
/* CsrMatrix::matvec_adjoint (csr.cpp:46-57): scatter, zero y_i skipped */
static void csr_matvec_t(csr a, const double *y, double *x) {
    for (int64_t j = 0; j < a.cols; ++j) x[j] = 0.0;
    for (int64_t i = 0; i < a.rows; ++i) {
        const double yi = y[i];
        if (yi == 0.0) continue;
        for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k) x[a.ci[k]] += a.v[k] * yi;
    }
}
/* CsrMatrix::to_dense (csr.cpp:59-65) */
static mat csr_dense(csr a) {
    mat d = mnew(a.rows, a.cols);
    for (int64_t i = 0; i < a.rows; ++i)
        for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k) AT(d, i, a.ci[k]) = a.v[k];
    return d;
}
/* sketch_apply(S, CsrMatrix) (sketch.cpp:97-118): rows outer, x = v * val */
static mat sstack_apply_csr(sstack s, csr a) {
    if (a.rows != s.m)
        raise_err(MSVD_ERR_DIMENSION, "sketch_apply: operand has %lld rows, embedding expects %lld",
                  (long long)a.rows, (long long)s.m);
    mat out = mnew(s.d, a.cols);
    const double val = 1.0 / sqrt((double)s.zeta);
    const int64_t blk_rows = s.d / s.zeta;
    for (int64_t r = 0; r < a.rows; ++r)
        for (int64_t p = a.rp[r]; p < a.rp[r + 1]; ++p) {
            const double x = a.v[p] * val;
            double *oj = col(out, a.ci[p]);
            for (int k = 0; k < s.zeta; ++k)
                oj[blk_rows * k + s.pos[r * s.zeta + k]] += (double)s.sgn[r * s.zeta + k] * x;
        }
    return out;
}

/* ------------------------------------- LinearOperator (operator.hpp:15-39) */

typedef struct { int is_csr; mat d; csr s; } op;

static int64_t op_rows(op a) { return a.is_csr ? a.s.rows : a.d.r; }
static int64_t op_cols(op a) { return a.is_csr ? a.s.cols : a.d.c; }
static void op_apply(op a, const double *x, double *y) { if (a.is_csr) csr_matvec(a.s, x, y); else matvec(a.d, x, y); }
static void op_adjoint(op a, const double *y, double *x) {
    if (a.is_csr) csr_matvec_t(a.s, y, x); else matvec_t(a.d, y, x);
}
static mat op_dense(op a) { return a.is_csr ? csr_dense(a.s) : a.d; }
static mat op_sketch(sstack s, op a) { return a.is_csr ? sstack_apply_csr(s, a.s) : sstack_apply(s, a.d); }
/* column_norms: DenseOperator (operator.cpp:39-48), CsrOperator (:98-104) */
static void op_colnorms(op a, double *out) {
    const int64_t n = op_cols(a);
    if (!a.is_csr) {
        for (int64_t j = 0; j < n; ++j) out[j] = colnorm_from(a.d, j, 0);
        return;
    }
    for (int64_t j = 0; j < n; ++j) out[j] = 0.0;
    const int64_t nnz = csr_nnz(a.s);
    for (int64_t k = 0; k < nnz; ++k) out[a.s.ci[k]] += a.s.v[k] * a.s.v[k];
    for (int64_t j = 0; j < n; ++j) out[j] = sqrt(out[j]);
}

/* -------------------------------------------------- preconditioner (precond.cpp) */

typedef struct { mat vt; double *sig; double smax; int floored; int64_t nfloor; } pcond;

static pcond pcond_build(mat sa) { /* precond.cpp:11-36 */
    const int64_t n = sa.c;
    if (n < 1) raise_err(MSVD_ERR_DIMENSION, "build_preconditioner: empty sketch");
    if (sa.r < n) raise_err(MSVD_ERR_DIMENSION, "build_preconditioner: sketch has fewer rows than columns");
    svdres s = svd_values_right(sa);
    pcond p = {s.v, s.sigma, s.sigma[0], 0, 0};
    if (p.smax == 0.0) raise_err(MSVD_ERR_NUMERICAL, "build_preconditioner: sketched matrix is exactly zero");
    const double floor_v = sqrt((double)n) * EPS * p.smax;
    for (int64_t j = 0; j < n; ++j)
        if (p.sig[j] < floor_v) { p.sig[j] = floor_v; p.floored = 1; ++p.nfloor; }
    return p;
}

static void pcond_apply(pcond p, const double *r, double *out) { /* precond.cpp:38-48 */
    const int64_t n = p.vt.c;
    double *t = (double *)zalloc(sizeof(double) * (size_t)n);
    matvec_t(p.vt, r, t);
    for (int64_t j = 0; j < n; ++j) { const double s = p.sig[j]; t[j] /= s * s; }
    matvec(p.vt, t, out);
}

/* --------------------------------------------------------- solver (solver.cpp) */

/* BCGS2 with seeded Gaussian replacement of degenerate columns (:213-261) */
static void cgs2_project(double *x, int64_t n, mat basis, mat w, int64_t upto) {
    for (int64_t l = 0; l < basis.c; ++l) {
        const double *c = col(basis, l);
        const double pr = vdot(c, x, n);
        for (int64_t i = 0; i < n; ++i) x[i] -= pr * c[i];
    }
    for (int64_t l = 0; l < upto; ++l) {
        const double *c = col(w, l);
        const double pr = vdot(c, x, n);
        for (int64_t i = 0; i < n; ++i) x[i] -= pr * c[i];
    }
}
static int64_t cgs2_block(mat w, mat basis, sm64 *rng) {
    const int64_t n = w.r;
    if (basis.c > 0 && basis.r != n) raise_err(MSVD_ERR_DIMENSION, "cgs2: basis row count mismatch");
    const double drop = (double)n * EPS * max_colnorm(w);
    int64_t replaced = 0;
    double *x = (double *)zalloc(sizeof(double) * (size_t)(n ? n : 1));
    for (int64_t j = 0; j < w.c; ++j) {
        memcpy(x, col(w, j), sizeof(double) * (size_t)n);
        cgs2_project(x, n, basis, w, j);
        cgs2_project(x, n, basis, w, j);
        double nrm = vnorm(x, n);
        if (nrm <= drop) {
            int ok = 0;
            for (int att = 0; att < 8 && !ok; ++att) {
                for (int64_t i = 0; i < n; ++i) x[i] = sm_gauss(rng);
                cgs2_project(x, n, basis, w, j);
                cgs2_project(x, n, basis, w, j);
                nrm = vnorm(x, n);
                ok = nrm > 1e-3 * sqrt((double)n);
            }
            if (!ok) raise_err(MSVD_ERR_NUMERICAL, "cgs2: could not complete an orthonormal block");
            ++replaced;
        }
        vscale(x, n, 1.0 / nrm);
        memcpy(col(w, j), x, sizeof(double) * (size_t)n);
    }
    return replaced;
}

/* orthonormal basis of span(g) for the history update (:77-119) */
static mat orth_coef(mat g) {
    const int64_t rows = g.r, cols = g.c;
    mat q = mnew(rows, cols);
    const double sref = max_colnorm(g);
    double *w = (double *)zalloc(sizeof(double) * (size_t)(rows ? rows : 1));
    double *e = (double *)zalloc(sizeof(double) * (size_t)(rows ? rows : 1));
    for (int64_t j = 0; j < cols; ++j) {
        memcpy(w, col(g, j), sizeof(double) * (size_t)rows);
        for (int pass = 0; pass < 2; ++pass)
            for (int64_t l = 0; l < j; ++l) {
                double pr = 0.0;
                for (int64_t i = 0; i < rows; ++i) pr += AT(q, i, l) * w[i];
                for (int64_t i = 0; i < rows; ++i) w[i] -= pr * AT(q, i, l);
            }
        const double nrm = vnorm(w, rows);
        if (nrm <= 1e-14 * (sref > 1.0 ? sref : 1.0)) {
            int placed = 0;
            for (int64_t cand = 0; cand < rows && !placed; ++cand) {
                for (int64_t i = 0; i < rows; ++i) e[i] = 0.0;
                e[cand] = 1.0;
                for (int pass = 0; pass < 2; ++pass)
                    for (int64_t l = 0; l < j; ++l) {
                        double pr = 0.0;
                        for (int64_t i = 0; i < rows; ++i) pr += AT(q, i, l) * e[i];
                        for (int64_t i = 0; i < rows; ++i) e[i] -= pr * AT(q, i, l);
                    }
                const double en = vnorm(e, rows);
                if (en > 1e-8) { vscale(e, rows, 1.0 / en); memcpy(w, e, sizeof(double) * (size_t)rows); placed = 1; }
            }
            if (!placed) raise_err(MSVD_ERR_NUMERICAL, "solver: history update basis collapsed");
        } else {
            vscale(w, rows, 1.0 / nrm);
        }
        memcpy(col(q, j), w, sizeof(double) * (size_t)rows);
    }
    return q;
}

/* stop rule on record histories (:177-211); flags tol/resid/progress/stop */
static void stop_rule(const double *rh, const double *th, int64_t len, int i, double s1, double tol,
                      double factor, int use_stag, int *f) {
    if (i + 1 >= len) raise_err(MSVD_ERR_DIMENSION, "check_convergence: history shorter than the loop counter");
    f[0] = f[1] = f[2] = f[3] = 0;
    f[0] = rh[i + 1] <= s1 * s1 * tol;
    if (!use_stag) { f[3] = f[0]; return; }
    if (i >= 4) f[1] = factor * rh[i + 1] >= rh[i - 4];
    if (i >= 9) {
        const double dn = th[i] > 0.0 ? th[i] : 1.0;
        const double dt = th[i - 4] > 0.0 ? th[i - 4] : 1.0;
        const double recent = (th[i - 4] - th[i + 1]) / dn;
        const double earlier = (th[i - 9] - th[i - 4]) / dt;
        f[2] = factor * recent >= earlier;
    }
    f[3] = f[0] && f[1] && f[2];
}

static mat cols_of(mat a, int64_t j0, int64_t cnt) {
    mat o = mnew(a.r, cnt);
    memcpy(o.p, col(a, j0), sizeof(double) * (size_t)(a.r * cnt));
    return o;
}
static mat hcat3(mat a, mat b, mat c) {
    mat o = mnew(a.r, a.c + b.c + c.c);
    int64_t at = 0;
    memcpy(col(o, at), a.p, sizeof(double) * (size_t)(a.r * a.c));
    at += a.c;
    if (b.c) memcpy(col(o, at), b.p, sizeof(double) * (size_t)(a.r * b.c));
    at += b.c;
    if (c.c) memcpy(col(o, at), c.p, sizeof(double) * (size_t)(a.r * c.c));
    return o;
}
static mat apply_cols(op a, mat x) { /* operator.cpp:7-12 apply_block, column by column */
    mat y = mnew(op_rows(a), x.c);
    for (int64_t j = 0; j < x.c; ++j) op_apply(a, col(x, j), col(y, j));
    return y;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec * 1e3 + (double)ts.tv_nsec * 1e-6;
}

typedef struct {
    msvd_result *res;
    int64_t b, n;
    long mva, mvat;
    double *rh, *th;
    int64_t nrow;
    const msvd_truth *truth;
    double t0;
    int timing;
} recorder;

static void record_row(recorder *R, int iter, mat vcur, const double *theta, double resid) { /* :376-397 */
    msvd_record_row row;
    memset(&row, 0, sizeof row);
    row.iter = iter;
    row.matvecs_a = R->mva;
    row.matvecs_at = R->mvat;
    row.wall_ms = R->timing ? now_ms() - R->t0 : 0.0;
    row.theta = theta[R->b - 1];
    row.resid = resid;
    row.relerr = -1.0;
    row.sin_angle = -1.0;
    if (R->truth) {
        const double sn = R->truth->sigma_min;
        row.relerr = sn > 0.0 ? fabs(row.theta - sn) / sn : fabs(row.theta);
        double c = 0.0;
        const double *vc = col(vcur, R->b - 1);
        for (int64_t i = 0; i < R->n; ++i) c += vc[i] * R->truth->v_min[i];
        c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
        const double s2 = 1.0 - c * c;
        row.sin_angle = sqrt(s2 > 0.0 ? s2 : 0.0);
    }
    if (R->nrow < R->res->rows_capacity) R->res->rows[R->nrow] = row;
    R->rh[R->nrow] = resid;
    R->th[R->nrow] = theta[0];
    R->nrow++;
}

/* R = A^T AV - theta^2 V per column (:357-369) */
static mat residual_block(op a, mat v, mat av, const double *th, long *mvat) {
    mat r = mnew(v.r, v.c);
    for (int64_t j = 0; j < v.c; ++j) {
        double *rc = col(r, j);
        op_adjoint(a, col(av, j), rc);
        ++*mvat;
        const double t2 = th[j] * th[j];
        const double *vc = col(v, j);
        for (int64_t i = 0; i < v.r; ++i) rc[i] -= t2 * vc[i];
    }
    return r;
}

static void emit(msvd_result *res, int kind, int iter, mat m) {
    if (res->iterate_cb) res->iterate_cb(res->iterate_user, kind, iter, m.p, m.r, m.c);
}

/* lobpcg_solve (solver.cpp:301-477) on a dense column-major A */
static void solve_op(op a, const msvd_options *o, const msvd_truth *truth, msvd_result *res) {
    const int64_t m = op_rows(a), n = op_cols(a), b = o->block_size;
    if (m < n) raise_err(MSVD_ERR_DIMENSION, "solver: matrix must have at least as many rows as columns");
    if (b < 1) raise_err(MSVD_ERR_DIMENSION, "solver: block size must be positive");
    if (n < 3 * b) raise_err(MSVD_ERR_DIMENSION, "solver: need at least 3x block size columns");
    const double tol = o->tol < 0.0 ? 2.0 * sqrt((double)n) * EPS : o->tol;
    if (!(tol >= 0.0 && tol < 1.0)) raise_err(MSVD_ERR_NUMERICAL, "solver: tol must lie in [0, 1)");
    const int max_iter = o->max_iter < 0 ? (b == 1 ? 200 : 100) : o->max_iter;
    if (max_iter < 0 || o->check_every < 1)
        raise_err(MSVD_ERR_NUMERICAL, "solver: max_iter must be >= 0 and check_every >= 1");
    if (truth && !truth->v_min) raise_err(MSVD_ERR_DIMENSION, "solver: ground-truth vector length mismatch");

    recorder R;
    memset(&R, 0, sizeof R);
    R.t0 = now_ms();
    R.timing = o->record_timing;
    R.res = res;
    R.b = b;
    R.n = n;
    R.truth = truth;
    R.rh = (double *)zalloc(sizeof(double) * (size_t)(max_iter + 2));
    R.th = (double *)zalloc(sizeof(double) * (size_t)(max_iter + 2));

    /* prepare (:128-145) */
    pcond P;
    int64_t dim = 0;
    int skipped = 0;
    if (o->sketch_dim < 0 && m <= 4 * n) {
        skipped = 1;
        P = pcond_build(op_dense(a));
    } else {
        if (o->sketch_dim < 0 && o->zeta <= 0)
            raise_err(MSVD_ERR_DIMENSION, "round_up_to_multiple: zeta must be positive");
        int64_t d = o->sketch_dim < 0 ? (4 * n % o->zeta == 0 ? 4 * n : 4 * n + (o->zeta - 4 * n % o->zeta))
                                      : o->sketch_dim;
        if (d < n) raise_err(MSVD_ERR_DIMENSION, "solver: sketch dimension below column count");
        sstack s = sstack_build(d, m, o->zeta, o->seed);
        P = pcond_build(op_sketch(s, a));
        dim = d;
    }
    if (b > n) raise_err(MSVD_ERR_DIMENSION, "sketch_and_solve_init: block size out of range");
    mat v = mnew(n, b);
    for (int64_t j = 0; j < b; ++j) memcpy(col(v, j), col(P.vt, n - b + j), sizeof(double) * (size_t)n);
    const double sigma1 = P.smax;

    res->sigma_max_estimate = sigma1;
    res->sketch_skipped = skipped;
    res->sketch_dim = dim;
    res->zeta = skipped ? 0 : o->zeta;
    res->floored = P.floored;
    res->floor_count = P.nfloor;
    res->verify_count = 0;
    res->max_cache_drift = 0.0;
    res->degenerate_replacements = 0;
    if (res->vtilde) memcpy(res->vtilde, P.vt.p, sizeof(double) * (size_t)(n * n));
    if (res->sigma_tilde) memcpy(res->sigma_tilde, P.sig, sizeof(double) * (size_t)n);

    double *dinv = NULL;
    if (o->precond_kind == MSVD_PRECOND_DIAGONAL) {
        dinv = (double *)zalloc(sizeof(double) * (size_t)n);
        op_colnorms(a, dinv);
        for (int64_t j = 0; j < n; ++j) {
            const double c = dinv[j];
            dinv[j] = c > 0.0 ? 1.0 / (c * c) : 1.0;
        }
    }
    sm64 rng = sm_keyed(o->seed, 0x9e3779b97f4a7c15ULL);

    mat av = apply_cols(a, v);
    R.mva += b;
    svdres rr0 = svd_values_right(av);
    v = matmul(v, rr0.v);
    av = matmul(av, rr0.v);
    double *theta = rr0.sigma;

    mat r = residual_block(a, v, av, theta, &R.mvat);
    record_row(&R, 0, v, theta, max_colnorm(r));
    if (o->store_iterates) emit(res, 1, 0, v);

    mat x = mnew(n, 0), ax = mnew(m, 0);
    int status = 1;
    for (int i = 0; i < max_iter; ++i) {
        mat w;
        if (o->precond_kind == MSVD_PRECOND_NONE) {
            w = mcopy(r);
        } else if (o->precond_kind == MSVD_PRECOND_DIAGONAL) {
            w = mnew(n, b);
            for (int64_t j = 0; j < b; ++j)
                for (int64_t q = 0; q < n; ++q) AT(w, q, j) = AT(r, q, j) * dinv[q];
        } else {
            w = mnew(n, b);
            for (int64_t j = 0; j < b; ++j) pcond_apply(P, col(r, j), col(w, j));
        }
        if (!finite_all(w.p, n * b))
            raise_err(MSVD_ERR_NUMERICAL, "solver: non-finite preconditioned residual at iteration %d", i);
        res->degenerate_replacements += cgs2_block(w, hcat3(v, x, mnew(n, 0)), &rng);

        mat t = hcat3(v, x, w);
        mat at = hcat3(av, ax, apply_cols(a, w));
        R.mva += b;
        if (!finite_all(at.p, at.r * at.c))
            raise_err(MSVD_ERR_NUMERICAL, "solver: non-finite trial products at iteration %d", i);

        const int64_t k = t.c;
        svdres rr = svd_values_right(at);
        mat ct = cols_of(rr.v, k - b, b);
        double *theta_next = rr.sigma + (k - b);
        mat v_next = matmul(t, ct);
        mat av_next = matmul(at, ct);

        r = residual_block(a, v_next, av_next, theta_next, &R.mvat);
        record_row(&R, i + 1, v_next, theta_next, max_colnorm(r));
        if (o->store_iterates) { emit(res, 0, i, t); emit(res, 1, i + 1, v_next); }

        if (o->verify_cached_products && (i + 1) % 25 == 0) {
            mat fresh = apply_cols(a, v_next);
            res->verify_count += b;
            double drift = 0.0;
            for (int64_t q = 0; q < m * b; ++q) {
                const double dd = fabs(fresh.p[q] - av_next.p[q]);
                if (dd > drift) drift = dd;
            }
            if (drift > res->max_cache_drift) res->max_cache_drift = drift;
            if (drift > 1e-10 * sigma1)
                raise_err(MSVD_ERR_NUMERICAL, "solver: cached product drifted from a fresh one at iteration %d", i);
        }

        int stop = 0;
        if (i % o->check_every == 0) {
            int f[4];
            stop_rule(R.rh, R.th, R.nrow, i, sigma1, tol, o->stagnation_factor, o->use_stagnation, f);
            stop = f[3];
        }
        if (stop) {
            v = v_next; av = av_next; theta = theta_next;
            status = 0;
            break;
        }
        const int64_t lead = k - b;
        mat g = mnew(lead, b);
        for (int64_t j = 0; j < lead; ++j)
            for (int64_t l = 0; l < b; ++l) AT(g, j, l) = AT(rr.v, l, j);
        mat q = orth_coef(g);
        mat mix = matmul(cols_of(rr.v, 0, lead), q);
        x = matmul(t, mix);
        ax = matmul(at, mix);
        v = v_next; av = av_next; theta = theta_next;
    }

    for (int64_t j = 0; j < b; ++j) {
        res->sigma[j] = theta[b - 1 - j];
        memcpy(res->v + j * n, col(v, b - 1 - j), sizeof(double) * (size_t)n);
    }
    res->status = status;
    res->rows_count = (int32_t)R.nrow;
    res->iterations = (int32_t)R.nrow - 1;
}

/* ------------------------------------------ lanczos_gk (baselines.cpp) */

/* two full MGS passes against the first `used` columns (baselines.cpp:19-31) */
static void reorth_mgs(double *w, int64_t len, mat basis, int64_t used) {
    for (int pass = 0; pass < 2; ++pass)
        for (int64_t l = 0; l < used; ++l) {
            const double *c = col(basis, l);
            double proj = 0.0;
            for (int64_t i = 0; i < len; ++i) proj += c[i] * w[i];
            for (int64_t i = 0; i < len; ++i) w[i] -= proj * c[i];
        }
}

/* lanczos_gk (baselines.cpp:51-166) on a dense column-major A */
static void lanczos_op(op a, int iters, const double *v0, const msvd_truth *truth, int timing,
                       msvd_lanczos_result *res) {
    const int64_t m = op_rows(a), n = op_cols(a);
    if (m < n) raise_err(MSVD_ERR_DIMENSION, "lanczos_gk: matrix must be tall");
    if (iters < 1 || iters > n) raise_err(MSVD_ERR_DIMENSION, "lanczos_gk: step count must lie in [1, cols]");
    const double v0n = vnorm(v0, n);
    if (v0n == 0.0) raise_err(MSVD_ERR_NUMERICAL, "lanczos_gk: starting vector is zero");
    if (truth && !truth->v_min) raise_err(MSVD_ERR_DIMENSION, "lanczos_gk: ground-truth vector length mismatch");
    const double t0 = now_ms();

    mat vb = mnew(n, iters + 1), ub = mnew(m, iters);
    double *alpha = (double *)zalloc(sizeof(double) * (size_t)iters);
    double *beta = (double *)zalloc(sizeof(double) * (size_t)iters);
    double *v = (double *)zalloc(sizeof(double) * (size_t)n);
    memcpy(v, v0, sizeof(double) * (size_t)n);
    vscale(v, n, 1.0 / v0n);
    memcpy(col(vb, 0), v, sizeof(double) * (size_t)n);

    double *u = (double *)zalloc(sizeof(double) * (size_t)m);
    op_apply(a, v, u);
    long mva = 1, mvat = 0;
    const double a1 = vnorm(u, m);
    res->rows_count = 0;
    res->steps = 0;
    res->status = MSVD_LANCZOS_COMPLETED;
    if (a1 == 0.0) { /* v0 is an exact null vector of A */
        res->sigma_min = 0.0;
        memcpy(res->v, v, sizeof(double) * (size_t)n);
        res->status = MSVD_LANCZOS_INVARIANT_SUBSPACE;
        return;
    }
    alpha[0] = a1;
    vscale(u, m, 1.0 / a1);
    memcpy(col(ub, 0), u, sizeof(double) * (size_t)m);
    double coeff = a1;

    double *w = (double *)zalloc(sizeof(double) * (size_t)n);
    double *vest = (double *)zalloc(sizeof(double) * (size_t)n);
    double *un = (double *)zalloc(sizeof(double) * (size_t)m);
    for (int j = 1; j <= iters; ++j) {
        op_adjoint(a, col(ub, j - 1), w);
        ++mvat;
        const double *vp = col(vb, j - 1);
        for (int64_t i = 0; i < n; ++i) w[i] += -alpha[j - 1] * vp[i];
        reorth_mgs(w, n, vb, j);
        const double bj = vnorm(w, n);
        if (bj > coeff) coeff = bj;
        beta[j - 1] = bj;

        mat sec = mnew(j, j); /* bidiagonal_section (baselines.cpp:33-40) */
        for (int i = 0; i < j; ++i) {
            AT(sec, i, i) = alpha[i];
            if (i + 1 < j) AT(sec, i, i + 1) = beta[i];
        }
        svdres s = svd_values_right(sec);
        const double theta = s.sigma[j - 1];
        const double *y = col(s.v, j - 1);
        memset(vest, 0, sizeof(double) * (size_t)n);
        for (int l = 0; l < j; ++l) {
            const double *c = col(vb, l);
            for (int64_t i = 0; i < n; ++i) vest[i] += y[l] * c[i];
        }
        const double resid = alpha[j - 1] * bj * fabs(y[j - 1]);

        msvd_record_row row;
        memset(&row, 0, sizeof row);
        row.iter = j;
        row.matvecs_a = mva;
        row.matvecs_at = mvat;
        row.wall_ms = timing ? now_ms() - t0 : 0.0;
        row.theta = theta;
        row.resid = resid;
        row.relerr = -1.0;
        row.sin_angle = -1.0;
        if (truth) {
            const double sn = truth->sigma_min;
            row.relerr = sn > 0.0 ? fabs(theta - sn) / sn : fabs(theta);
            double c = vdot(vest, truth->v_min, n);
            c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
            const double s2 = 1.0 - c * c;
            row.sin_angle = sqrt(s2 > 0.0 ? s2 : 0.0);
        }
        if (res->rows_count < res->rows_capacity) res->rows[res->rows_count] = row;
        res->rows_count++;
        res->sigma_min = theta;
        memcpy(res->v, vest, sizeof(double) * (size_t)n);
        res->steps = j;

        if (bj <= 64.0 * EPS * coeff) { res->status = MSVD_LANCZOS_INVARIANT_SUBSPACE; break; }
        if (j == iters) break;

        vscale(w, n, 1.0 / bj);
        memcpy(col(vb, j), w, sizeof(double) * (size_t)n);
        op_apply(a, w, un);
        ++mva;
        const double *up = col(ub, j - 1);
        for (int64_t i = 0; i < m; ++i) un[i] += -bj * up[i];
        reorth_mgs(un, m, ub, j);
        const double aj = vnorm(un, m);
        if (aj > coeff) coeff = aj;
        if (aj <= 64.0 * EPS * coeff) { res->status = MSVD_LANCZOS_INVARIANT_SUBSPACE; break; }
        alpha[j] = aj;
        vscale(un, m, 1.0 / aj);
        memcpy(col(ub, j), un, sizeof(double) * (size_t)m);
    }
    if (res->v_basis) memcpy(res->v_basis, vb.p, sizeof(double) * (size_t)(n * res->steps));
    if (res->u_basis) memcpy(res->u_basis, ub.p, sizeof(double) * (size_t)(m * res->steps));
}

/* ---------------------------------------------------------------- exports */

int orc_lanczos_gk(const double *a_colmajor, int64_t m, int64_t n, int iters, const double *v0,
                   const msvd_truth *truth, int record_timing, msvd_lanczos_result *res) {
    ENTER();
    op a = {0, mview((double *)a_colmajor, m, n), {0, 0, NULL, NULL, NULL}};
    lanczos_op(a, iters, v0, truth, record_timing, res);
    LEAVE();
}

/* CsrOperator (operator.hpp:58-74): validated at construction (csr.cpp:9-31) */
static op csr_op(int64_t m, int64_t n, const int64_t *rp, const int64_t *ci, const double *v, int64_t nnz) {
    op a = {1, {0, 0, NULL}, {m, n, rp, ci, v}};
    csr_validate(a.s, nnz);
    return a;
}

int orc_lanczos_gk_csr(int64_t m, int64_t n, const int64_t *rp, const int64_t *ci, const double *v, int64_t nnz,
                       int iters, const double *v0, const msvd_truth *truth, int record_timing,
                       msvd_lanczos_result *res) {
    ENTER();
    lanczos_op(csr_op(m, n, rp, ci, v, nnz), iters, v0, truth, record_timing, res);
    LEAVE();
}

int orc_lobpcg_solve_csr(int64_t m, int64_t n, const int64_t *rp, const int64_t *ci, const double *v, int64_t nnz,
                         const msvd_options *o, const msvd_truth *truth, msvd_result *res) {
    ENTER();
    solve_op(csr_op(m, n, rp, ci, v, nnz), o, truth, res);
    LEAVE();
}

/* sketch_apply(S, CsrMatrix) of rows [row0, row0 + m) keyed by global row */
int orc_sketch_csr(int64_t d, int zeta, uint64_t seed, int64_t m, int64_t n, const int64_t *rp, const int64_t *ci,
                   const double *v, int64_t nnz, int64_t row0, double *sa) {
    ENTER();
    op a = csr_op(m, n, rp, ci, v, nnz);
    sstack full = sstack_build(d, row0 + m, zeta, seed);
    sstack s = {d, m, zeta, full.pos + row0 * zeta, full.sgn + row0 * zeta};
    mat out = sstack_apply_csr(s, a.s);
    memcpy(sa, out.p, sizeof(double) * (size_t)(d * n));
    LEAVE();
}

/* y = A x, x = A^T y, column norms of a CSR operator (checker primitives) */
int orc_csr_products(int64_t m, int64_t n, const int64_t *rp, const int64_t *ci, const double *v, int64_t nnz,
                     const double *x, double *y, const double *yin, double *xout, double *norms) {
    ENTER();
    op a = csr_op(m, n, rp, ci, v, nnz);
    if (x && y) csr_matvec(a.s, x, y);
    if (yin && xout) csr_matvec_t(a.s, yin, xout);
    if (norms) op_colnorms(a, norms);
    LEAVE();
}

void orc_splitmix_draws(uint64_t seed, uint64_t key, int keyed, int kind, int64_t count, double *out_f,
                        uint64_t *out_u, uint64_t bound) {
    sm64 r = keyed ? sm_keyed(seed, key) : sm_plain(seed);
    for (int64_t i = 0; i < count; ++i) {
        if (kind == 0) out_u[i] = sm_u64(&r);
        else if (kind == 1) out_u[i] = sm_below(&r, bound);
        else if (kind == 2) out_f[i] = sm_unit(&r);
        else out_f[i] = sm_gauss(&r);
    }
}

int orc_build_sparsestack(int64_t d, int64_t m, int zeta, uint64_t seed, uint32_t *pos, int8_t *sgn) {
    ENTER();
    sstack s = sstack_build(d, m, zeta, seed);
    memcpy(pos, s.pos, sizeof(uint32_t) * (size_t)(m * zeta));
    memcpy(sgn, s.sgn, (size_t)(m * zeta));
    LEAVE();
}

/* sketch of a row block [row0, row0+rows) of a larger A whose S columns are
 * keyed by GLOBAL row index (the row-sharded form).  Column-major
 * local block.  row0 = 0, rows = m is sketch_apply itself.                  */
int orc_sketch_rows(int64_t d, int zeta, uint64_t seed, const double *a, int64_t rows, int64_t n,
                    int64_t row0, double *sa) {
    ENTER();
    sstack full = sstack_build(d, row0 + rows, zeta, seed);
    sstack s = {d, rows, zeta, full.pos + row0 * zeta, full.sgn + row0 * zeta};
    mat out = sstack_apply(s, mview((double *)a, rows, n));
    memcpy(sa, out.p, sizeof(double) * (size_t)(d * n));
    LEAVE();
}

int orc_householder_r(const double *a, int64_t m, int64_t k, double *r) {
    ENTER();
    mat rr = qr_rfactor(qr_factor(mview((double *)a, m, k)));
    memcpy(r, rr.p, sizeof(double) * (size_t)(k * k));
    LEAVE();
}

int orc_dense_svd(const double *a, int64_t rows, int64_t n, double *sigma, double *v) {
    ENTER();
    svdres s = svd_values_right(mview((double *)a, rows, n));
    memcpy(sigma, s.sigma, sizeof(double) * (size_t)n);
    memcpy(v, s.v.p, sizeof(double) * (size_t)(n * n));
    LEAVE();
}

int orc_build_preconditioner(const double *sa, int64_t rows, int64_t n, double *vt, double *sig, double *smax,
                             int64_t *nfloor) {
    ENTER();
    pcond p = pcond_build(mview((double *)sa, rows, n));
    memcpy(vt, p.vt.p, sizeof(double) * (size_t)(n * n));
    memcpy(sig, p.sig, sizeof(double) * (size_t)n);
    *smax = p.smax;
    *nfloor = p.nfloor;
    LEAVE();
}

int orc_precond_apply(const double *vt, const double *sig, int64_t n, const double *r, int64_t b, double *w) {
    ENTER();
    pcond p = {mview((double *)vt, n, n), (double *)sig, 0.0, 0, 0};
    for (int64_t j = 0; j < b; ++j) pcond_apply(p, r + j * n, w + j * n);
    LEAVE();
}

int orc_check_convergence(const double *resid, const double *theta, int64_t len, int i, double s1, double tol,
                          double factor, int use_stag, int *flags) {
    ENTER();
    stop_rule(resid, theta, len, i, s1, tol, factor, use_stag, flags);
    LEAVE();
}

int orc_cgs2(double *w, int64_t n, int64_t c, const double *basis, int64_t nb, uint64_t seed, int64_t *replaced) {
    ENTER();
    sm64 rng = sm_keyed(seed, 0x9e3779b97f4a7c15ULL);
    *replaced = cgs2_block(mview(w, n, c), mview((double *)basis, n, nb), &rng);
    LEAVE();
}

int orc_orth_coefficients(const double *g, int64_t rows, int64_t cols, double *q) {
    ENTER();
    mat qq = orth_coef(mview((double *)g, rows, cols));
    memcpy(q, qq.p, sizeof(double) * (size_t)(rows * cols));
    LEAVE();
}

/* haar_orthonormal (matgen.cpp:126-139): Q of a SplitMix64 Gaussian, R_jj>0 */
static mat haar(int64_t m, int64_t n, uint64_t seed) {
    if (m < n) raise_err(MSVD_ERR_DIMENSION, "haar_orthonormal: need rows >= columns");
    if (n < 1) raise_err(MSVD_ERR_DIMENSION, "haar_orthonormal: need at least one column");
    sm64 r = sm_plain(seed);
    mat g = mnew(m, n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) AT(g, i, j) = sm_gauss(&r);
    hqr q = qr_factor(g);
    mat qm = qr_q_times(q, meye(n));
    for (int64_t j = 0; j < n; ++j)
        if (AT(q.a, j, j) < 0.0) {
            double *c = col(qm, j);
            for (int64_t i = 0; i < m; ++i) c[i] = -c[i];
        }
    return qm;
}

int orc_haar_orthonormal(int64_t m, int64_t n, uint64_t seed, double *q) {
    ENTER();
    g_par = 1;
    mat h = haar(m, n, seed);
    memcpy(q, h.p, sizeof(double) * (size_t)(m * n));
    g_par = 0;
    LEAVE();
}

/* synth(explicit_list) dense assembly (matgen.cpp:141-176): A = U diag(s) V^T */
int orc_synth_dense(const double *sigma, int64_t n, int64_t m, uint64_t seed, double *a_colmajor, double *v_min) {
    ENTER();
    g_par = 1;
    if (n < 2) raise_err(MSVD_ERR_DIMENSION, "spectrum: need at least two values");
    for (int64_t i = 0; i < n; ++i) {
        if (!(sigma[i] > 0.0)) raise_err(MSVD_ERR_NUMERICAL, "spectrum: values must be strictly positive");
        if (i > 0 && sigma[i] > sigma[i - 1]) raise_err(MSVD_ERR_NUMERICAL, "spectrum: values must be nonincreasing");
    }
    if (m < n) raise_err(MSVD_ERR_DIMENSION, "synth: need rows >= columns");
    sm64 ku = sm_keyed(seed, 0x55u), kv = sm_keyed(seed, 0x56u);
    mat u = haar(m, n, sm_u64(&ku));
    mat v = haar(n, n, sm_u64(&kv));
    memcpy(v_min, col(v, n - 1), sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) {
        double *c = col(u, j);
        for (int64_t i = 0; i < m; ++i) c[i] *= sigma[j];
    }
    mat a = matmul(u, transpose(v));
    memcpy(a_colmajor, a.p, sizeof(double) * (size_t)(m * n));
    g_par = 0;
    LEAVE();
}

/* Same assembly without spectrum validation: configs with exact zeros (C3)
 * are assembled directly, since spectrum() rejects them (matgen.cpp:41-47). */
int orc_assemble_svd(const double *sigma, int64_t n, int64_t m, uint64_t seed, double *a_colmajor, double *v_min) {
    ENTER();
    g_par = 1;
    if (m < n) raise_err(MSVD_ERR_DIMENSION, "synth: need rows >= columns");
    sm64 ku = sm_keyed(seed, 0x55u), kv = sm_keyed(seed, 0x56u);
    mat u = haar(m, n, sm_u64(&ku));
    mat v = haar(n, n, sm_u64(&kv));
    memcpy(v_min, col(v, n - 1), sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) {
        double *c = col(u, j);
        for (int64_t i = 0; i < m; ++i) c[i] *= sigma[j];
    }
    mat a = matmul(u, transpose(v));
    memcpy(a_colmajor, a.p, sizeof(double) * (size_t)(m * n));
    g_par = 0;
    LEAVE();
}

/* ------------------------------------------------ harness-only generator
 * NOT a reference recipe: a fast, bit-reproducible stand-in for synth() at the
 * sizes where matgen's serial Householder QR of an m x n Gaussian would take
 * many minutes (the full-n parity fixtures: C3 at n = 2000, C5 at n = 1000).
 *
 *   X  m x n Gaussian, column j from SplitMix64(seed, 0x1000 + j) (rng.hpp)
 *   G  = X^T X, accumulated over fixed 512-row chunks in chunk order
 *   R  = chol(G) (upper), so U = X R^{-1} is orthonormal to ~kappa(X)^2 u
 *        (kappa(X) ~ 1.2-1.6 for the tall Gaussians used here)
 *   V  = haar_orthonormal(n, n, SplitMix64(seed, 0x56)) (matgen.cpp:126-139)
 *   A  = X M with M = R^{-1} diag(sigma) V^T, so A = U diag(sigma) V^T
 *
 * Every output element is computed by one thread in a fixed operation order
 * (no FMA: -ffp-contract=off), so the bytes depend only on (sigma, m, seed),
 * never on the thread count; the fixtures pin them by SHA-256.  Exact zeros
 * in sigma give exactly zero rows of diag(sigma) V^T, hence an exact
 * rank deficiency of M up to the rounding of the triangular solve.        */
static double dot4(const double *a, const double *b, int64_t len) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t i = 0;
    for (; i + 4 <= len; i += 4) {
        s0 += a[i] * b[i];
        s1 += a[i + 1] * b[i + 1];
        s2 += a[i + 2] * b[i + 2];
        s3 += a[i + 3] * b[i + 3];
    }
    for (; i < len; ++i) s0 += a[i] * b[i];
    return (s0 + s1) + (s2 + s3);
}

int orc_synth_fast(const double *sigma, int64_t n, int64_t m, uint64_t seed, double *a_colmajor, double *v_out) {
    ENTER();
    g_par = 1;
    if (n < 1 || m < n) raise_err(MSVD_ERR_DIMENSION, "synth_fast: need rows >= columns >= 1");
    mat x = mnew(m, n);
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t j = 0; j < n; ++j) {
        sm64 r = sm_keyed(seed, 0x1000u + (uint64_t)j);
        double *c = col(x, j);
        for (int64_t i = 0; i < m; ++i) c[i] = sm_gauss(&r);
    }
    /* G (upper triangle) = sum over 512-row chunks, in chunk order */
    mat g = mnew(n, n);
    const int64_t CH = 512;
    for (int64_t r0 = 0; r0 < m; r0 += CH) {
        const int64_t len = (m - r0 < CH) ? m - r0 : CH;
#pragma omp parallel for schedule(dynamic, 8)
        for (int64_t q = 0; q < n; ++q) {
            const double *xq = col(x, q) + r0;
            for (int64_t p = 0; p <= q; ++p) AT(g, p, q) += dot4(col(x, p) + r0, xq, len);
        }
    }
    /* right-looking Cholesky, R stored transposed (rt(l, k) = R(k, l)) */
    mat rt = mnew(n, n);
    for (int64_t k = 0; k < n; ++k) {
        const double d = AT(g, k, k);
        if (!(d > 0.0)) raise_err(MSVD_ERR_NUMERICAL, "synth_fast: Gram matrix not positive definite");
        const double rkk = sqrt(d);
        AT(rt, k, k) = rkk;
        for (int64_t j = k + 1; j < n; ++j) AT(rt, j, k) = AT(g, k, j) / rkk;
        const double *rk = col(rt, k);
#pragma omp parallel for schedule(static) if ((n - k) * (n - k) > 16384)
        for (int64_t j = k + 1; j < n; ++j)
            for (int64_t i = k + 1; i <= j; ++i) AT(g, i, j) -= rk[i] * rk[j];
    }
    sm64 kv = sm_keyed(seed, 0x56u);
    mat v = haar(n, n, sm_u64(&kv));
    memcpy(v_out, v.p, sizeof(double) * (size_t)(n * n));
    /* M = R^{-1} diag(sigma) V^T, column by column (back substitution) */
    mat mm = mnew(n, n);
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t j = 0; j < n; ++j) {
        double *mj = col(mm, j);
        for (int64_t k = n - 1; k >= 0; --k) {
            const double *rk = col(rt, k); /* rk[l] = R(k, l) */
            double s = sigma[k] * AT(v, j, k);
            for (int64_t l = k + 1; l < n; ++l) s -= rk[l] * mj[l];
            mj[k] = s / rk[k];
        }
    }
    /* A = X M over 128-row blocks; A(i, j) = sum_k M(k, j) X(i, k), k ascending */
    const int64_t RB = 128;
    const int64_t nblk = (m + RB - 1) / RB;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t bi = 0; bi < nblk; ++bi) {
        const int64_t i0 = bi * RB, len = (m - i0 < RB) ? m - i0 : RB;
        for (int64_t j = 0; j < n; ++j) {
            double acc[128];
            for (int64_t i = 0; i < len; ++i) acc[i] = 0.0;
            const double *mj = col(mm, j);
            for (int64_t k = 0; k < n; ++k) {
                const double c = mj[k];
                const double *xk = col(x, k) + i0;
                for (int64_t i = 0; i < len; ++i) acc[i] += c * xk[i];
            }
            memcpy(a_colmajor + j * m + i0, acc, sizeof(double) * (size_t)len);
        }
    }
    g_par = 0;
    LEAVE();
}

int orc_lobpcg_solve(const double *a, int64_t m, int64_t n, const msvd_options *o, const msvd_truth *truth,
                     msvd_result *res) {
    ENTER();
    mat d = mview((double *)a, m, n);
    if (!finite_all(d.p, m * n)) raise_err(MSVD_ERR_NUMERICAL, "DenseOperator: non-finite entry");
    op A = {0, d, {0, 0, NULL, NULL, NULL}};
    solve_op(A, o, truth, res);
    LEAVE();
}
