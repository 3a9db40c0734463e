// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (minsvd, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// Python tests and bench.py's reference arm call the reference's own code path
// (lobpcg_solve, sketch_apply, dense_svd, ...) on raw arrays.  Nothing here
// re-implements any algorithm; each function only converts raw pointers to
// minsvd types and back.
#include <cstring>
#include <exception>
#include <string>

#include "minsvd/baselines.hpp"
#include "minsvd/errors.hpp"
#include "minsvd/matgen.hpp"
#include "minsvd/operator.hpp"
#include "minsvd/precond.hpp"
#include "minsvd/rng.hpp"
#include "minsvd/sketch.hpp"
#include "minsvd/solver.hpp"
#include "minsvd/svd.hpp"
#include "msvd.h"

using namespace minsvd;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const DimensionError*>(&e)) return MSVD_ERR_DIMENSION;
    if (dynamic_cast<const IoError*>(&e)) return MSVD_ERR_IO;
    if (dynamic_cast<const NumericalError*>(&e)) return MSVD_ERR_NUMERICAL;
    if (dynamic_cast<const ConvergenceError*>(&e)) return MSVD_ERR_CONVERGENCE;
    return MSVD_ERR_INVALID;
}

DenseMatrix wrap(const double* a, index_t m, index_t n) {
    DenseMatrix d(m, n);
    if (m * n > 0) std::memcpy(d.data(), a, sizeof(double) * static_cast<size_t>(m * n));
    return d;
}

void unwrap(const DenseMatrix& d, double* out) {
    if (d.rows() * d.cols() > 0)
        std::memcpy(out, d.data(), sizeof(double) * static_cast<size_t>(d.rows() * d.cols()));
}

SolverOptions to_opts(const msvd_options* o) {
    SolverOptions s;
    s.tol = o->tol;
    s.max_iter = o->max_iter;
    s.check_every = o->check_every;
    s.stagnation_factor = o->stagnation_factor;
    s.block_size = o->block_size;
    s.seed = o->seed;
    s.sketch_dim = o->sketch_dim;
    s.zeta = o->zeta;
    s.use_stagnation = o->use_stagnation != 0;
    s.record_timing = o->record_timing != 0;
    s.verify_cached_products = o->verify_cached_products != 0;
    s.store_iterates = o->store_iterates != 0;
    return s;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// matgen.cpp:141-176 synth(explicit_list, m, seed), dense assembly.
int ref_synth_dense(const double* sigma, int64_t n, int64_t m, uint64_t seed,
                    double* a_colmajor, double* v_min) {
    try {
        SpectrumSpec spec;
        spec.kind = SpectrumKind::explicit_list;
        spec.values.assign(sigma, sigma + n);
        SyntheticProblem p = synth(spec, m, seed, false, false);
        unwrap(p.a->to_dense(), a_colmajor);
        std::memcpy(v_min, p.v_min.data(), sizeof(double) * static_cast<size_t>(n));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// matgen.cpp:126-139
int ref_haar_orthonormal(int64_t m, int64_t n, uint64_t seed, double* q) {
    try {
        unwrap(haar_orthonormal(m, n, seed), q);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// rng.hpp: raw stream draws for pinning the SplitMix64 restatement.
void ref_splitmix_draws(uint64_t seed, uint64_t key, int keyed, int kind, int64_t count,
                        double* out_f, uint64_t* out_u, uint64_t bound) {
    SplitMix64 r = keyed ? SplitMix64(seed, key) : SplitMix64(seed);
    for (int64_t i = 0; i < count; ++i) {
        if (kind == 0) out_u[i] = r.next_u64();
        else if (kind == 1) out_u[i] = r.next_below(bound);
        else if (kind == 2) out_f[i] = r.next_unit();
        else out_f[i] = r.next_gaussian();
    }
}

// sketch.cpp:36-60
int ref_build_sparsestack(int64_t d, int64_t m, int zeta, uint64_t seed, uint32_t* pos,
                          int8_t* sign) {
    try {
        SparseStackEmbedding s = build_sparsestack(d, m, zeta, seed);
        std::memcpy(pos, s.positions.data(), sizeof(uint32_t) * s.positions.size());
        std::memcpy(sign, s.signs.data(), s.signs.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// sketch.cpp:75-95 (dense operand), A column-major m x n -> SA d x n.
int ref_sketch_apply(int64_t d, int zeta, uint64_t seed, const double* a, int64_t m,
                     int64_t n, double* sa) {
    try {
        SparseStackEmbedding s = build_sparsestack(d, m, zeta, seed);
        unwrap(sketch_apply(s, DenseOperator(wrap(a, m, n))), sa);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// svd.cpp:21-63 householder_qr + qr_r
int ref_householder_r(const double* a, int64_t m, int64_t k, double* r) {
    try {
        unwrap(qr_r(householder_qr(wrap(a, m, k))), r);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// svd.cpp:180-252 dense_svd(want_u = false)
int ref_dense_svd(const double* a, int64_t rows, int64_t n, double* sigma, double* v) {
    try {
        SvdResult s = dense_svd(wrap(a, rows, n), false);
        std::memcpy(sigma, s.sigma.data(), sizeof(double) * static_cast<size_t>(n));
        unwrap(s.v, v);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// precond.cpp:11-36
int ref_build_preconditioner(const double* sa, int64_t rows, int64_t n, double* vt,
                             double* sig, double* smax, int64_t* floor_count) {
    try {
        Preconditioner p = build_preconditioner(wrap(sa, rows, n));
        unwrap(p.vtilde, vt);
        std::memcpy(sig, p.sigma_tilde.data(), sizeof(double) * static_cast<size_t>(n));
        *smax = p.sigma_max_estimate;
        *floor_count = p.floor_count;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// precond.cpp:38-48, applied per column of r (n x b)
int ref_precond_apply(const double* vt, const double* sig, int64_t n, const double* r,
                      int64_t b, double* w) {
    try {
        Preconditioner p;
        p.vtilde = wrap(vt, n, n);
        p.sigma_tilde.assign(sig, sig + n);
        for (int64_t j = 0; j < b; ++j) {
            Vector col(r + j * n, r + (j + 1) * n);
            Vector out = precond_apply(p, col);
            std::memcpy(w + j * n, out.data(), sizeof(double) * static_cast<size_t>(n));
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// solver.cpp:177-211; flags = {tol_ok, resid_stalled, progress_stalled, stop}
int ref_check_convergence(const double* resid, const double* theta, int64_t len, int i,
                          double sigma1, double tol, double factor, int use_stagnation,
                          int* flags) {
    try {
        std::vector<double> r(resid, resid + len), t(theta, theta + len);
        StopDecision d = check_convergence(r, t, i, sigma1, tol, factor, use_stagnation != 0);
        flags[0] = d.tol_ok;
        flags[1] = d.resid_stalled;
        flags[2] = d.progress_stalled;
        flags[3] = d.stop;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// solver.cpp:213-261, w (n x c) in place against basis (n x nb); rng keyed
// like the solver's replacement stream (seed, 0x9e3779b97f4a7c15).
int ref_cgs2(double* w, int64_t n, int64_t c, const double* basis, int64_t nb,
             uint64_t seed, int64_t* replaced) {
    try {
        DenseMatrix wm = wrap(w, n, c);
        DenseMatrix bm = nb > 0 ? wrap(basis, n, nb) : DenseMatrix(n, 0);
        SplitMix64 rng(seed, 0x9e3779b97f4a7c15ull);
        *replaced = cgs2(wm, bm, rng);
        unwrap(wm, w);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

namespace {
CsrMatrix wrap_csr(int64_t m, int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t nnz) {
    CsrMatrix c;
    c.rows = m;
    c.cols = n;
    c.row_offsets.assign(rp, rp + m + 1);
    c.col_indices.assign(ci, ci + nnz);
    c.values.assign(v, v + nnz);
    return c;
}
int solve_on(const LinearOperator& op, int64_t n, const msvd_options* o, const msvd_truth* truth,
             msvd_result* res);
int lanczos_on(const LinearOperator& op, int64_t n, int iters, const double* v0, const msvd_truth* truth,
               int record_timing, msvd_lanczos_result* res);
}  // namespace

// solver.cpp:301-477 lobpcg_solve on a DenseOperator (A column-major m x n).
int ref_lobpcg_solve(const double* a, int64_t m, int64_t n, const msvd_options* o,
                     const msvd_truth* truth, msvd_result* res) {
    try {
        DenseOperator op(wrap(a, m, n));
        return solve_on(op, n, o, truth, res);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// the same on a CsrOperator (operator.hpp:58-74; validated at construction)
int ref_lobpcg_solve_csr(int64_t m, int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                         int64_t nnz, const msvd_options* o, const msvd_truth* truth, msvd_result* res) {
    try {
        CsrOperator op(wrap_csr(m, n, rp, ci, v, nnz));
        return solve_on(op, n, o, truth, res);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// sketch.cpp:97-118 sketch_apply(S, CsrMatrix)
int ref_sketch_csr(int64_t d, int zeta, uint64_t seed, int64_t m, int64_t n, const int64_t* rp,
                   const int64_t* ci, const double* v, int64_t nnz, double* sa) {
    try {
        SparseStackEmbedding s = build_sparsestack(d, m, zeta, seed);
        unwrap(sketch_apply(s, wrap_csr(m, n, rp, ci, v, nnz)), sa);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// csr.cpp:33-57 matvec / matvec_adjoint, operator.cpp:98-104 column_norms
int ref_csr_products(int64_t m, int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                     int64_t nnz, const double* x, double* y, const double* yin, double* xout,
                     double* norms) {
    try {
        CsrOperator op(wrap_csr(m, n, rp, ci, v, nnz));
        if (x && y) {
            Vector r = op.apply(Vector(x, x + n));
            std::memcpy(y, r.data(), sizeof(double) * r.size());
        }
        if (yin && xout) {
            Vector r = op.apply_adjoint(Vector(yin, yin + m));
            std::memcpy(xout, r.data(), sizeof(double) * r.size());
        }
        if (norms) {
            Vector r = op.column_norms();
            std::memcpy(norms, r.data(), sizeof(double) * r.size());
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_lanczos_gk_csr(int64_t m, int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                       int64_t nnz, int iters, const double* v0, const msvd_truth* truth,
                       int record_timing, msvd_lanczos_result* res) {
    try {
        CsrOperator op(wrap_csr(m, n, rp, ci, v, nnz));
        return lanczos_on(op, n, iters, v0, truth, record_timing, res);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"

namespace {
int solve_on(const LinearOperator& op, int64_t n, const msvd_options* o, const msvd_truth* truth,
             msvd_result* res) {
    try {
        SolverOptions opts = to_opts(o);
        GroundTruth gt;
        const GroundTruth* gtp = nullptr;
        if (truth) {
            gt.sigma_min = truth->sigma_min;
            gt.v_min.assign(truth->v_min, truth->v_min + n);
            gtp = &gt;
        }
        PrecondKind kind = o->precond_kind == MSVD_PRECOND_NONE       ? PrecondKind::none
                           : o->precond_kind == MSVD_PRECOND_DIAGONAL ? PrecondKind::diagonal
                                                                      : PrecondKind::randomized;
        SolveResult r = lobpcg_solve(op, kind, opts, gtp);
        const index_t b = static_cast<index_t>(r.sigma.size());
        std::memcpy(res->sigma, r.sigma.data(), sizeof(double) * static_cast<size_t>(b));
        unwrap(r.v, res->v);
        res->rows_count = static_cast<int32_t>(r.record.rows.size());
        res->iterations = static_cast<int32_t>(r.iterations());
        for (size_t i = 0; i < r.record.rows.size() && static_cast<int32_t>(i) < res->rows_capacity;
             ++i) {
            const RecordRow& src = r.record.rows[i];
            msvd_record_row& dst = res->rows[i];
            dst.iter = src.iter;
            dst.matvecs_a = src.matvecs_a;
            dst.matvecs_at = src.matvecs_at;
            dst.wall_ms = src.wall_ms;
            dst.theta = src.theta;
            dst.resid = src.resid;
            dst.relerr = src.relerr;
            dst.sin_angle = src.sin_angle;
        }
        res->status = r.status == SolveStatus::converged ? 0 : 1;
        if (res->vtilde) unwrap(r.precond.vtilde, res->vtilde);
        if (res->sigma_tilde)
            std::memcpy(res->sigma_tilde, r.precond.sigma_tilde.data(),
                        sizeof(double) * r.precond.sigma_tilde.size());
        res->sigma_max_estimate = r.sigma_max_estimate;
        res->floored = r.precond.floored;
        res->floor_count = r.precond.floor_count;
        res->sketch_skipped = r.sketch_skipped;
        res->sketch_dim = r.sketch_dim;
        res->zeta = r.zeta;
        res->verify_count = r.verify_count;
        res->max_cache_drift = r.max_cache_drift;
        res->degenerate_replacements = r.degenerate_replacements;
        if (res->iterate_cb) {
            for (size_t i = 0; i < r.trail_t.size(); ++i)
                res->iterate_cb(res->iterate_user, 0, static_cast<int32_t>(i), r.trail_t[i].data(),
                                r.trail_t[i].rows(), r.trail_t[i].cols());
            for (size_t i = 0; i < r.trail_v.size(); ++i)
                res->iterate_cb(res->iterate_user, 1, static_cast<int32_t>(i), r.trail_v[i].data(),
                                r.trail_v[i].rows(), r.trail_v[i].cols());
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// baselines.cpp:51-166 lanczos_gk on a DenseOperator (A column-major m x n).
int lanczos_on(const LinearOperator& op, int64_t n, int iters, const double* v0, const msvd_truth* truth,
               int record_timing, msvd_lanczos_result* res) {
    try {
        GroundTruth gt;
        const GroundTruth* gtp = nullptr;
        if (truth) {
            gt.sigma_min = truth->sigma_min;
            gt.v_min.assign(truth->v_min, truth->v_min + n);
            gtp = &gt;
        }
        Vector v(v0, v0 + n);
        LanczosResult r = lanczos_gk(op, iters, v, gtp, record_timing != 0);
        res->sigma_min = r.sigma_min;
        std::memcpy(res->v, r.v.data(), sizeof(double) * r.v.size());
        res->rows_count = static_cast<int32_t>(r.record.rows.size());
        for (size_t i = 0; i < r.record.rows.size() && static_cast<int32_t>(i) < res->rows_capacity;
             ++i) {
            const RecordRow& src = r.record.rows[i];
            msvd_record_row& dst = res->rows[i];
            dst.iter = src.iter;
            dst.matvecs_a = src.matvecs_a;
            dst.matvecs_at = src.matvecs_at;
            dst.wall_ms = src.wall_ms;
            dst.theta = src.theta;
            dst.resid = src.resid;
            dst.relerr = src.relerr;
            dst.sin_angle = src.sin_angle;
        }
        res->status = r.status == LanczosStatus::completed ? MSVD_LANCZOS_COMPLETED
                                                           : MSVD_LANCZOS_INVARIANT_SUBSPACE;
        res->steps = r.steps;
        if (res->v_basis) unwrap(r.v_basis, res->v_basis);
        if (res->u_basis) unwrap(r.u_basis, res->u_basis);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // namespace

extern "C" {
int ref_lanczos_gk(const double* a, int64_t m, int64_t n, int iters, const double* v0,
                   const msvd_truth* truth, int record_timing, msvd_lanczos_result* res) {
    try {
        DenseOperator op(wrap(a, m, n));
        return lanczos_on(op, n, iters, v0, truth, record_timing, res);
    } catch (const std::exception& e) {
        return fail(e);
    }
}
}  // extern "C"
