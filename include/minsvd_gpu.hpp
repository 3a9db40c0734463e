// minsvd_gpu.hpp -- the reference's C++ solve API (minsvd, solver.hpp /
// operator.hpp / errors.hpp) over the C ABI of libmsvd_cuda.so.
//
// Header-only.  Same names, argument meaning and error behaviour as
//   /root/reference/proj/include/minsvd/solver.hpp:25-190
//   /root/reference/proj/include/minsvd/operator.hpp:15-56
//   /root/reference/proj/include/minsvd/errors.hpp:9-38
// with one substitution: the operator is a DeviceDenseOperator over device
// memory (row-major A), and every product runs on the GPU.  There is no CPU
// path; a solve on anything else is rejected with DimensionError.
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "msvd.h"

namespace minsvd {
namespace gpu {

using index_t = std::ptrdiff_t;
using Vector = std::vector<double>;

// ---- errors.hpp:9-38 ------------------------------------------------------
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class DimensionError : public Error {
public:
    explicit DimensionError(const std::string& m) : Error(m) {}
};
class IoError : public Error {
public:
    explicit IoError(const std::string& m) : Error(m) {}
};
class NumericalError : public Error {
public:
    explicit NumericalError(const std::string& m) : Error(m) {}
};
class ConvergenceError : public Error {
public:
    explicit ConvergenceError(const std::string& m) : Error(m) {}
};

inline void check(int32_t rc) {
    if (rc == MSVD_OK) return;
    const std::string msg = msvd_last_error();
    switch (rc) {
        case MSVD_ERR_DIMENSION: throw DimensionError(msg);
        case MSVD_ERR_IO: throw IoError(msg);
        case MSVD_ERR_NUMERICAL: throw NumericalError(msg);
        case MSVD_ERR_CONVERGENCE: throw ConvergenceError(msg);
        default: throw Error(msg);
    }
}

// ---- solver.hpp ------------------------------------------------------------
enum class PrecondKind { none = MSVD_PRECOND_NONE, diagonal = MSVD_PRECOND_DIAGONAL, randomized = MSVD_PRECOND_RANDOMIZED };

struct SolverOptions {
    double tol = -1.0;
    int max_iter = -1;
    int check_every = 5;
    double stagnation_factor = 1.1;
    index_t block_size = 1;
    std::uint64_t seed = 0;
    index_t sketch_dim = -1;
    int zeta = 4;
    bool use_stagnation = true;
    bool record_timing = true;
    bool verify_cached_products = false;
    bool store_iterates = false;

    msvd_options to_abi(PrecondKind kind) const {
        msvd_options o;
        o.tol = tol;
        o.max_iter = max_iter;
        o.check_every = check_every;
        o.stagnation_factor = stagnation_factor;
        o.block_size = block_size;
        o.seed = seed;
        o.sketch_dim = sketch_dim;
        o.zeta = zeta;
        o.use_stagnation = use_stagnation;
        o.record_timing = record_timing;
        o.verify_cached_products = verify_cached_products;
        o.store_iterates = store_iterates;
        o.precond_kind = static_cast<int32_t>(kind);
        return o;
    }
};

inline double default_tolerance(index_t n) {
    return 2.0 * std::sqrt(static_cast<double>(n)) * std::numeric_limits<double>::epsilon();
}

struct GroundTruth {
    double sigma_min = 0.0;
    Vector v_min;
};

struct RecordRow {
    int iter = 0;
    long matvecs_a = 0;
    long matvecs_at = 0;
    double wall_ms = 0.0;
    double theta = 0.0;
    double resid = 0.0;
    double relerr = -1.0;
    double sin_angle = -1.0;
};

struct ConvergenceRecord {
    std::vector<RecordRow> rows;
    bool has_truth = false;
};

enum class SolveStatus { converged, max_iter_reached };

struct SolveResult {
    std::vector<double> v;  // n x b, column-major, ordered like sigma
    index_t n = 0, b = 0;
    Vector sigma;           // ascending from the smallest
    SolveStatus status = SolveStatus::max_iter_reached;
    ConvergenceRecord record;
    double sigma_max_estimate = 0.0;
    bool sketch_skipped = false;
    index_t sketch_dim = 0;
    int zeta = 0;
    long verify_count = 0;
    double max_cache_drift = 0.0;
    index_t degenerate_replacements = 0;
    index_t floor_count = 0;
    std::vector<std::vector<double>> trail_t, trail_v;
    index_t iterations() const { return static_cast<index_t>(record.rows.size()) - 1; }
};

// ---- device context + operator (operator.hpp:41-56 DenseOperator) --------
class Context {
public:
    explicit Context(int device = 0, void* stream = nullptr) {
        msvd_ctx_desc d{};
        d.device = device;
        d.stream = stream;
        check(msvd_ctx_create(&d, &ctx_));
    }
    Context(const msvd_ctx_desc& d) { check(msvd_ctx_create(&d, &ctx_)); }
    ~Context() { msvd_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    msvd_ctx* get() const { return ctx_; }
    void synchronize() const { check(msvd_ctx_synchronize(ctx_)); }

private:
    msvd_ctx* ctx_ = nullptr;
};

// Common handle of the device operators: the products and passes of one
// LinearOperator (operator.hpp:15-39) over device memory.
class DeviceOperator {
public:
    virtual ~DeviceOperator() { msvd_matrix_detach(mat_); }
    DeviceOperator(const DeviceOperator&) = delete;
    DeviceOperator& operator=(const DeviceOperator&) = delete;

    index_t rows() const { return m_; }
    index_t cols() const { return n_; }
    virtual index_t nnz() const = 0;
    // device-to-device block products (column-major blocks)
    void apply_block(const double* dX, index_t b, double* dY) const { check(msvd_apply(mat_, dX, b, dY)); }
    void apply_adjoint_block(const double* dY, index_t b, double* dX) const {
        check(msvd_apply_adjoint(mat_, dY, b, dX));
    }
    void column_norms(double* dNorms) const { check(msvd_column_norms(mat_, dNorms)); }
    // the iteration's two passes as primitives: K2 Y = T C and
    // G = A^T Y[:, :b]; K3 A W with the TSQR R of [lead | A W]; the one-pass
    // A W plus A^T A W
    void gram_apply(const double* dT, index_t k, const double* dC, index_t q, index_t b, double* dG,
                    double* dY) const {
        check(msvd_gram_apply(mat_, dT, k, dC, q, b, dG, dY));
    }
    void aw_tsqr(const double* dW, index_t b, const double* dLead, index_t kl, double* dAW, double* dR) const {
        check(msvd_aw_tsqr(mat_, dW, b, dLead, kl, dAW, dR));
    }
    void aw_gram(const double* dW, index_t b, double* dAW, double* dZ) const {
        check(msvd_aw_gram(mat_, dW, b, dAW, dZ));
    }
    msvd_matrix* get() const { return mat_; }

protected:
    DeviceOperator(index_t m, index_t n) : m_(m), n_(n) {}
    msvd_matrix* mat_ = nullptr;
    index_t m_, n_;
};

// operator.hpp:41-56 DenseOperator: borrowed device pointer, rows
// [row0, row0 + m_local) of an m_global x n row-major matrix (leading dim ld)
class DeviceDenseOperator final : public DeviceOperator {
public:
    DeviceDenseOperator(const Context& ctx, const double* dA, index_t m_local, index_t n, index_t ld,
                        index_t row0 = 0, index_t m_global = -1)
        : DeviceOperator(m_global < 0 ? m_local : m_global, n) {
        check(msvd_matrix_attach(ctx.get(), dA, m_local, n, ld, row0, m_, &mat_));
    }
    index_t nnz() const override { return m_ * n_; }
};

// operator.hpp:58-74 CsrOperator: borrowed device CSR arrays of the local
// rows (row offsets int64, column indices of index_bytes = 4 or 8, values);
// validated like CsrMatrix::validate at construction
class DeviceCsrOperator final : public DeviceOperator {
public:
    DeviceCsrOperator(const Context& ctx, const int64_t* dRowOffsets, const void* dColIndices, int index_bytes,
                      const double* dValues, index_t m_local, index_t n, index_t nnz, index_t row0 = 0,
                      index_t m_global = -1)
        : DeviceOperator(m_global < 0 ? m_local : m_global, n), nnz_(nnz) {
        check(msvd_csr_attach(ctx.get(), dRowOffsets, dColIndices, index_bytes, dValues, m_local, n, nnz, row0, m_,
                              &mat_));
    }
    index_t nnz() const override { return nnz_; }

private:
    index_t nnz_;
};

namespace detail {
inline void iterate_sink(void* user, int32_t kind, int32_t, const double* data, int64_t rows, int64_t cols) {
    auto* r = static_cast<SolveResult*>(user);
    (kind == 0 ? r->trail_t : r->trail_v).emplace_back(data, data + rows * cols);
}

inline SolveResult run(int32_t (*fn)(msvd_matrix*, const msvd_options*, const msvd_truth*, msvd_result*),
                       const DeviceOperator& a, PrecondKind kind, const SolverOptions& opts,
                       const GroundTruth* truth, bool force_single) {
    msvd_options o = opts.to_abi(kind);
    if (force_single) o.block_size = 1;
    const index_t b = o.block_size > 0 ? o.block_size : 1;
    const int max_iter = o.max_iter >= 0 ? o.max_iter : (b == 1 ? 200 : 100);
    SolveResult out;
    out.n = a.cols();
    out.b = b;
    out.sigma.assign(static_cast<size_t>(b), 0.0);
    out.v.assign(static_cast<size_t>(b * a.cols()), 0.0);
    std::vector<msvd_record_row> rows(static_cast<size_t>(max_iter + 2));
    msvd_result r{};
    r.sigma = out.sigma.data();
    r.v = out.v.data();
    r.rows = rows.data();
    r.rows_capacity = static_cast<int32_t>(rows.size());
    r.iterate_cb = &iterate_sink;
    r.iterate_user = &out;
    msvd_truth t{};
    if (truth) {
        if (static_cast<index_t>(truth->v_min.size()) != a.cols())
            throw DimensionError("solver: ground-truth vector length mismatch");
        t.sigma_min = truth->sigma_min;
        t.v_min = truth->v_min.data();
    }
    check(fn(a.get(), &o, truth ? &t : nullptr, &r));
    out.status = r.status == 0 ? SolveStatus::converged : SolveStatus::max_iter_reached;
    out.record.has_truth = truth != nullptr;
    for (int i = 0; i < r.rows_count && i < r.rows_capacity; ++i) {
        const msvd_record_row& s = rows[static_cast<size_t>(i)];
        out.record.rows.push_back(RecordRow{s.iter, static_cast<long>(s.matvecs_a), static_cast<long>(s.matvecs_at),
                                            s.wall_ms, s.theta, s.resid, s.relerr, s.sin_angle});
    }
    out.sigma_max_estimate = r.sigma_max_estimate;
    out.sketch_skipped = r.sketch_skipped != 0;
    out.sketch_dim = r.sketch_dim;
    out.zeta = r.zeta;
    out.verify_count = static_cast<long>(r.verify_count);
    out.max_cache_drift = r.max_cache_drift;
    out.degenerate_replacements = r.degenerate_replacements;
    out.floor_count = r.floor_count;
    return out;
}
}  // namespace detail

// solver.hpp:172-181
inline SolveResult lobpcg_solve(const DeviceOperator& a, PrecondKind kind, const SolverOptions& opts,
                                const GroundTruth* truth = nullptr) {
    return detail::run(&msvd_lobpcg_solve, a, kind, opts, truth, false);
}
inline SolveResult rlobpcg_single(const DeviceOperator& a, const SolverOptions& opts,
                                  const GroundTruth* truth = nullptr) {
    return detail::run(&msvd_rlobpcg_single, a, PrecondKind::randomized, opts, truth, true);
}
inline SolveResult rlobpcg_block(const DeviceOperator& a, const SolverOptions& opts,
                                 const GroundTruth* truth = nullptr) {
    return detail::run(&msvd_rlobpcg_block, a, PrecondKind::randomized, opts, truth, false);
}

// ---- baselines.hpp:12-42 ---------------------------------------------------
inline SolveResult lobpcg_generic(const DeviceOperator& a, PrecondKind kind, const SolverOptions& opts,
                                  const GroundTruth* truth = nullptr) {
    return lobpcg_solve(a, kind, opts, truth);
}

enum class LanczosStatus { completed, invariant_subspace };

struct LanczosResult {
    double sigma_min = 0.0;
    Vector v;
    ConvergenceRecord record;
    LanczosStatus status = LanczosStatus::completed;
    int steps = 0;
    std::vector<double> v_basis;  // n x steps, column-major
    std::vector<double> u_basis;  // m_local x steps, column-major
};

// baselines.cpp:51-166 on the device (msvd_lanczos_gk)
inline LanczosResult lanczos_gk(const DeviceOperator& a, int iters, const Vector& v0,
                                const GroundTruth* truth = nullptr, bool record_timing = true,
                                index_t m_local = -1) {
    if (static_cast<index_t>(v0.size()) != a.cols())
        throw DimensionError("lanczos_gk: starting vector length mismatch");
    if (truth && static_cast<index_t>(truth->v_min.size()) != a.cols())
        throw DimensionError("lanczos_gk: ground-truth vector length mismatch");
    const index_t ml = m_local < 0 ? a.rows() : m_local;
    LanczosResult out;
    out.v.assign(static_cast<size_t>(a.cols()), 0.0);
    const size_t cap = static_cast<size_t>(iters > 0 ? iters : 1);
    std::vector<msvd_record_row> rows(cap);
    out.v_basis.assign(static_cast<size_t>(a.cols()) * cap, 0.0);
    out.u_basis.assign(static_cast<size_t>(ml) * cap, 0.0);
    msvd_lanczos_result r{};
    r.v = out.v.data();
    r.rows = rows.data();
    r.rows_capacity = static_cast<int32_t>(cap);
    r.v_basis = out.v_basis.data();
    r.u_basis = out.u_basis.data();
    msvd_truth t{};
    if (truth) {
        t.sigma_min = truth->sigma_min;
        t.v_min = truth->v_min.data();
    }
    check(msvd_lanczos_gk(a.get(), iters, v0.data(), truth ? &t : nullptr, record_timing ? 1 : 0, &r));
    out.sigma_min = r.sigma_min;
    out.status = r.status == MSVD_LANCZOS_COMPLETED ? LanczosStatus::completed : LanczosStatus::invariant_subspace;
    out.steps = r.steps;
    out.record.has_truth = truth != nullptr;
    for (int i = 0; i < r.rows_count && i < r.rows_capacity; ++i) {
        const msvd_record_row& s = rows[static_cast<size_t>(i)];
        out.record.rows.push_back(RecordRow{s.iter, static_cast<long>(s.matvecs_a), static_cast<long>(s.matvecs_at),
                                            s.wall_ms, s.theta, s.resid, s.relerr, s.sin_angle});
    }
    out.v_basis.resize(static_cast<size_t>(a.cols()) * r.steps);
    out.u_basis.resize(static_cast<size_t>(ml) * r.steps);
    return out;
}

}  // namespace gpu
}  // namespace minsvd
