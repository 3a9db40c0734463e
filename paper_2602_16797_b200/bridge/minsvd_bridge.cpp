// The device solver behind the reference's own C++ types (include/minsvd_bridge.hpp).
//
// Built against the reference's headers and library (the integration a
// maintainer adds to proj/: INTEGRATION.md section 3); every product and the
// whole gpu_* solve run in libmsvd_cuda.so through its C ABI (include/msvd.h).
#include "minsvd_bridge.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>

namespace minsvd {
namespace {

// errors.hpp:9-38 from the ABI status (include/msvd.h msvd_status)
void check(int32_t rc) {
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

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(std::string("msvd bridge: ") + what + ": " + cudaGetErrorString(e));
}

msvd_options to_abi(const SolverOptions& o, PrecondKind kind) {
    msvd_options a;
    msvd_options_default(&a);
    a.tol = o.tol;
    a.max_iter = o.max_iter;
    a.check_every = o.check_every;
    a.stagnation_factor = o.stagnation_factor;
    a.block_size = static_cast<int64_t>(o.block_size);
    a.seed = o.seed;
    a.sketch_dim = static_cast<int64_t>(o.sketch_dim);
    a.zeta = o.zeta;
    a.use_stagnation = o.use_stagnation ? 1 : 0;
    a.record_timing = o.record_timing ? 1 : 0;
    a.verify_cached_products = o.verify_cached_products ? 1 : 0;
    a.store_iterates = o.store_iterates ? 1 : 0;
    a.precond_kind = kind == PrecondKind::none ? MSVD_PRECOND_NONE
                     : kind == PrecondKind::diagonal ? MSVD_PRECOND_DIAGONAL
                                                     : MSVD_PRECOND_RANDOMIZED;
    return a;
}

DenseMatrix from_colmajor(const double* p, index_t rows, index_t cols) {
    DenseMatrix m(rows, cols);
    if (rows > 0 && cols > 0) std::memcpy(m.data(), p, sizeof(double) * static_cast<std::size_t>(rows * cols));
    return m;
}

// store_iterates sink (solver.cpp:424-427): trail_t / trail_v as DenseMatrix
void iterate_sink(void* user, int32_t kind, int32_t, const double* data, int64_t rows, int64_t cols) {
    auto* r = static_cast<SolveResult*>(user);
    (kind == 0 ? r->trail_t : r->trail_v).push_back(from_colmajor(data, rows, cols));
}

const DeviceDenseOperatorAdapter* device_operator(const LinearOperator& a) {
    const LinearOperator* op = &a;
    if (const auto* counting = dynamic_cast<const CountingOperator*>(op)) op = &counting->inner();  // sketch.cpp:121
    const auto* dev = dynamic_cast<const DeviceDenseOperatorAdapter*>(op);
    if (!dev)
        throw DimensionError("gpu_lobpcg_solve: the device solver takes a DeviceDenseOperatorAdapter "
                             "(no CPU fallback)");
    return dev;
}

}  // namespace

// ------------------------------------------------------------------ operator
DeviceDenseOperatorAdapter::DeviceDenseOperatorAdapter(msvd_ctx* ctx, const double* dA, index_t m_local, index_t n,
                                                       index_t ld, index_t row0, index_t m_global)
    : ctx_(ctx), m_(m_local), n_(n), mglob_(m_global < 0 ? m_local : m_global) {
    attach(dA, ld, row0);
}

DeviceDenseOperatorAdapter::DeviceDenseOperatorAdapter(msvd_ctx* ctx, const DenseMatrix& a)
    : ctx_(ctx), m_(a.rows()), n_(a.cols()), mglob_(a.rows()) {
    // DenseOperator's constructor rejects non-finite data (operator.cpp:35-37);
    // the device solve checks it again on its own
    const std::size_t count = static_cast<std::size_t>(m_ * n_);
    std::vector<double> rm(count);
    for (index_t j = 0; j < n_; ++j) {
        const double* c = a.col(j);
        for (index_t i = 0; i < m_; ++i) rm[static_cast<std::size_t>(i * n_ + j)] = c[i];
    }
    cuda(cudaMalloc(&owned_, sizeof(double) * std::max<std::size_t>(count, 1)), "cudaMalloc");
    if (count) cuda(cudaMemcpy(owned_, rm.data(), sizeof(double) * count, cudaMemcpyHostToDevice), "upload A");
    attach(owned_, n_, 0);
}

void DeviceDenseOperatorAdapter::attach(const double* dA, index_t ld, index_t row0) {
    dA_ = dA;
    ld_ = m_ > 1 ? ld : n_;
    check(msvd_matrix_attach(ctx_, dA, m_, n_, ld_, row0, mglob_, &mat_));
}

DeviceDenseOperatorAdapter::~DeviceDenseOperatorAdapter() {
    if (mat_) msvd_matrix_detach(mat_);
    for (double* b : buf_)
        if (b) cudaFree(b);
    if (owned_) cudaFree(owned_);
}

double* DeviceDenseOperatorAdapter::scratch(std::size_t doubles, int which) const {
    if (cap_[which] < doubles) {
        if (buf_[which]) cudaFree(buf_[which]);
        buf_[which] = nullptr;
        cuda(cudaMalloc(&buf_[which], sizeof(double) * std::max<std::size_t>(doubles, 1)), "cudaMalloc");
        cap_[which] = doubles;
    }
    return buf_[which];
}

DenseMatrix DeviceDenseOperatorAdapter::apply_block(const DenseMatrix& x) const {
    if (x.rows() != n_) throw DimensionError("apply_block: dimension mismatch");
    const index_t b = x.cols();
    DenseMatrix y(m_, b);
    if (b == 0) return y;
    double* dx = scratch(static_cast<std::size_t>(n_ * b), 0);
    double* dy = scratch(static_cast<std::size_t>(m_ * b), 1);
    cuda(cudaMemcpy(dx, x.data(), sizeof(double) * n_ * b, cudaMemcpyHostToDevice), "H2D x");
    check(msvd_apply(mat_, dx, b, dy));
    check(msvd_ctx_synchronize(ctx_));
    cuda(cudaMemcpy(y.data(), dy, sizeof(double) * m_ * b, cudaMemcpyDeviceToHost), "D2H y");
    return y;
}

DenseMatrix DeviceDenseOperatorAdapter::apply_adjoint_block(const DenseMatrix& y) const {
    if (y.rows() != m_) throw DimensionError("apply_adjoint_block: dimension mismatch");
    const index_t b = y.cols();
    DenseMatrix x(n_, b);
    if (b == 0) return x;
    double* dy = scratch(static_cast<std::size_t>(m_ * b), 1);
    double* dx = scratch(static_cast<std::size_t>(n_ * b), 0);
    cuda(cudaMemcpy(dy, y.data(), sizeof(double) * m_ * b, cudaMemcpyHostToDevice), "H2D y");
    check(msvd_apply_adjoint(mat_, dy, b, dx));
    check(msvd_ctx_synchronize(ctx_));
    cuda(cudaMemcpy(x.data(), dx, sizeof(double) * n_ * b, cudaMemcpyDeviceToHost), "D2H x");
    return x;
}

Vector DeviceDenseOperatorAdapter::apply(const Vector& x) const {
    if (static_cast<index_t>(x.size()) != n_) throw DimensionError("dense_matvec: dimension mismatch");
    DenseMatrix xm(n_, 1);
    xm.set_col(0, x);
    return apply_block(xm).col_copy(0);
}

Vector DeviceDenseOperatorAdapter::apply_adjoint(const Vector& y) const {
    if (static_cast<index_t>(y.size()) != m_) throw DimensionError("dense_matvec_adjoint: dimension mismatch");
    DenseMatrix ym(m_, 1);
    ym.set_col(0, y);
    return apply_adjoint_block(ym).col_copy(0);
}

Vector DeviceDenseOperatorAdapter::column_norms() const {
    double* d = scratch(static_cast<std::size_t>(n_), 0);
    check(msvd_column_norms(mat_, d));
    check(msvd_ctx_synchronize(ctx_));
    Vector out(static_cast<std::size_t>(n_));
    cuda(cudaMemcpy(out.data(), d, sizeof(double) * n_, cudaMemcpyDeviceToHost), "D2H norms");
    return out;
}

DenseMatrix DeviceDenseOperatorAdapter::to_dense() const {
    std::vector<double> rm(static_cast<std::size_t>(m_ * n_));
    check(msvd_ctx_synchronize(ctx_));
    if (m_ > 0 && n_ > 0)
        cuda(cudaMemcpy2D(rm.data(), sizeof(double) * n_, dA_, sizeof(double) * ld_, sizeof(double) * n_, m_,
                          cudaMemcpyDeviceToHost),
             "D2H A");
    DenseMatrix a(m_, n_);
    for (index_t j = 0; j < n_; ++j)
        for (index_t i = 0; i < m_; ++i) a(i, j) = rm[static_cast<std::size_t>(i * n_ + j)];
    return a;
}

// -------------------------------------------------------------------- solves
SolveResult gpu_lobpcg_solve(const LinearOperator& a, PrecondKind kind, const SolverOptions& opts,
                             const GroundTruth* truth) {
    const DeviceDenseOperatorAdapter* dev = device_operator(a);
    const index_t n = dev->cols();
    msvd_options o = to_abi(opts, kind);
    const index_t b = std::max<index_t>(opts.block_size, 1);
    const int max_iter = opts.max_iter >= 0 ? opts.max_iter : (b == 1 ? 200 : 100);
    if (truth && static_cast<index_t>(truth->v_min.size()) != n)
        throw DimensionError("solver: ground-truth vector length mismatch");

    SolveResult r;
    std::vector<double> sigma(static_cast<std::size_t>(b)), v(static_cast<std::size_t>(n * b));
    std::vector<msvd_record_row> rows(static_cast<std::size_t>(std::max(max_iter, 0) + 2));
    r.precond.vtilde = DenseMatrix(n, n);
    r.precond.sigma_tilde.assign(static_cast<std::size_t>(n), 0.0);
    msvd_result res;
    std::memset(&res, 0, sizeof(res));
    res.sigma = sigma.data();
    res.v = v.data();
    res.rows = rows.data();
    res.rows_capacity = static_cast<int32_t>(rows.size());
    res.vtilde = r.precond.vtilde.data();
    res.sigma_tilde = r.precond.sigma_tilde.data();
    res.iterate_cb = opts.store_iterates ? iterate_sink : nullptr;
    res.iterate_user = &r;
    msvd_truth t{};
    if (truth) {
        t.sigma_min = truth->sigma_min;
        t.v_min = truth->v_min.data();
    }
    check(msvd_lobpcg_solve(dev->handle(), &o, truth ? &t : nullptr, &res));

    r.v = from_colmajor(v.data(), n, b);
    r.sigma = sigma;
    r.status = res.status == 0 ? SolveStatus::converged : SolveStatus::max_iter_reached;
    r.record.has_truth = truth != nullptr;
    for (int i = 0; i < res.rows_count && i < res.rows_capacity; ++i) {
        RecordRow row;
        row.iter = rows[static_cast<std::size_t>(i)].iter;
        row.matvecs_a = static_cast<long>(rows[static_cast<std::size_t>(i)].matvecs_a);
        row.matvecs_at = static_cast<long>(rows[static_cast<std::size_t>(i)].matvecs_at);
        row.wall_ms = rows[static_cast<std::size_t>(i)].wall_ms;
        row.theta = rows[static_cast<std::size_t>(i)].theta;
        row.resid = rows[static_cast<std::size_t>(i)].resid;
        row.relerr = rows[static_cast<std::size_t>(i)].relerr;
        row.sin_angle = rows[static_cast<std::size_t>(i)].sin_angle;
        r.record.rows.push_back(row);
    }
    r.precond.sigma_max_estimate = res.sigma_max_estimate;
    r.precond.floored = res.floored != 0;
    r.precond.floor_count = static_cast<index_t>(res.floor_count);
    r.sigma_max_estimate = res.sigma_max_estimate;
    r.sketch_skipped = res.sketch_skipped != 0;
    r.sketch_dim = static_cast<index_t>(res.sketch_dim);
    r.zeta = res.zeta;
    r.verify_count = static_cast<long>(res.verify_count);
    r.max_cache_drift = res.max_cache_drift;
    r.degenerate_replacements = static_cast<index_t>(res.degenerate_replacements);
    return r;
}

SolveResult gpu_rlobpcg_single(const LinearOperator& a, const SolverOptions& opts, const GroundTruth* truth) {
    SolverOptions o = opts;
    o.block_size = 1;  // solver.cpp:479-484
    return gpu_lobpcg_solve(a, PrecondKind::randomized, o, truth);
}

SolveResult gpu_rlobpcg_block(const LinearOperator& a, const SolverOptions& opts, const GroundTruth* truth) {
    return gpu_lobpcg_solve(a, PrecondKind::randomized, opts, truth);
}

StopDecision gpu_check_convergence(const std::vector<double>& resid_hist, const std::vector<double>& theta_hist,
                                   int i, double sigma1_estimate, double tol, double factor, bool use_stagnation) {
    static thread_local msvd_ctx* ctx = nullptr;
    if (!ctx) {
        msvd_ctx_desc desc;
        std::memset(&desc, 0, sizeof(desc));
        cuda(cudaGetDevice(&desc.device), "cudaGetDevice");
        check(msvd_ctx_create(&desc, &ctx));
    }
    const int64_t len = static_cast<int64_t>(std::min(resid_hist.size(), theta_hist.size()));
    int32_t f[4] = {0, 0, 0, 0};
    check(msvd_check_convergence(ctx, resid_hist.data(), theta_hist.data(), len, i, sigma1_estimate, tol, factor,
                                 use_stagnation ? 1 : 0, f));
    StopDecision d;
    d.tol_ok = f[0] != 0;
    d.resid_stalled = f[1] != 0;
    d.progress_stalled = f[2] != 0;
    d.stop = f[3] != 0;
    return d;
}

}  // namespace minsvd
