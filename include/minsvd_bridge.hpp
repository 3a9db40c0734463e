// minsvd_bridge.hpp -- the device solver behind the reference's OWN C++ types.
//
// Where include/minsvd_gpu.hpp mirrors the reference API in a parallel
// namespace for callers that do not link the reference, this header plugs the
// device path INTO the reference: it is compiled against the reference's
// headers (/root/reference/proj/include) and links the reference library, so
//
//   * DeviceDenseOperatorAdapter IS a minsvd::LinearOperator
//     (operator.hpp:15-39): the reference's own solvers, CountingOperator
//     (operator.hpp:102-128) and every caller that takes a
//     `const LinearOperator&` can hold it, and its products run on the GPU;
//   * gpu_lobpcg_solve / gpu_rlobpcg_single / gpu_rlobpcg_block take the
//     reference's SolverOptions / GroundTruth and return the reference's
//     SolveResult (solver.hpp:118-137) -- DenseMatrix v, the Preconditioner
//     (vtilde, sigma_tilde, floor data), the ConvergenceRecord whose to_csv()
//     (solver.cpp:149-171) is the reference's own, counters and trails --
//     with the whole solve on the device (libmsvd_cuda.so).
//
// Errors are the reference's exception classes (errors.hpp:9-38), mapped from
// the C ABI status codes.  There is no CPU fallback: gpu_* reject any operator
// that is not a DeviceDenseOperatorAdapter (or a CountingOperator over one,
// unwrapped as sketch.cpp:121-122 does) with DimensionError.
#pragma once

#include <memory>

#include "minsvd/operator.hpp"
#include "minsvd/solver.hpp"
#include "msvd.h"

namespace minsvd {

/// A dense operator over device memory: row-major A (m_local x n, leading
/// dimension ld) on the context's GPU, rows [row0, row0 + m_local) of an
/// m_global-row matrix for row-sharded runs.  Products are deterministic for
/// a fixed device and rank count (operator.hpp:10-14).  rows() is this
/// rank's row count: apply() returns the local rows, apply_adjoint() the
/// n-vector summed over ranks.
class DeviceDenseOperatorAdapter final : public LinearOperator {
public:
    /// Borrow device memory (the caller keeps it alive and unchanged).
    DeviceDenseOperatorAdapter(msvd_ctx* ctx, const double* dA, index_t m_local, index_t n, index_t ld,
                               index_t row0 = 0, index_t m_global = -1);
    /// Upload a host DenseMatrix (column-major, dense.hpp:14-50) as a
    /// row-major device copy owned by the adapter.
    DeviceDenseOperatorAdapter(msvd_ctx* ctx, const DenseMatrix& a);
    ~DeviceDenseOperatorAdapter() override;
    DeviceDenseOperatorAdapter(const DeviceDenseOperatorAdapter&) = delete;
    DeviceDenseOperatorAdapter& operator=(const DeviceDenseOperatorAdapter&) = delete;

    index_t rows() const override { return m_; }
    index_t cols() const override { return n_; }
    index_t nnz() const override { return m_ * n_; }
    Vector apply(const Vector& x) const override;
    Vector apply_adjoint(const Vector& y) const override;
    /// One device pass for all columns (operator.cpp:7-19 loops per column).
    DenseMatrix apply_block(const DenseMatrix& x) const override;
    DenseMatrix apply_adjoint_block(const DenseMatrix& y) const override;
    Vector column_norms() const override;
    DenseMatrix to_dense() const override;

    msvd_matrix* handle() const { return mat_; }
    msvd_ctx* context() const { return ctx_; }
    index_t m_global() const { return mglob_; }

private:
    void attach(const double* dA, index_t ld, index_t row0);
    double* scratch(std::size_t doubles, int which) const;

    msvd_ctx* ctx_ = nullptr;
    msvd_matrix* mat_ = nullptr;
    const double* dA_ = nullptr;
    double* owned_ = nullptr;
    index_t m_ = 0, n_ = 0, ld_ = 0, mglob_ = 0;
    mutable double* buf_[2] = {nullptr, nullptr};
    mutable std::size_t cap_[2] = {0, 0};
};

/// solver.hpp:172-173 lobpcg_solve with the whole solve on the device.
SolveResult gpu_lobpcg_solve(const LinearOperator& a, PrecondKind kind, const SolverOptions& opts,
                             const GroundTruth* truth = nullptr);
/// solver.hpp:176-177 (block size forced to 1).
SolveResult gpu_rlobpcg_single(const LinearOperator& a, const SolverOptions& opts,
                               const GroundTruth* truth = nullptr);
/// solver.hpp:180-181 (randomized preconditioner).
SolveResult gpu_rlobpcg_block(const LinearOperator& a, const SolverOptions& opts,
                              const GroundTruth* truth = nullptr);

/// The device stop rule (the control kernel's __device__ decision) on a
/// synthetic history, for the reference's check_convergence tests
/// (solver.hpp:152-155, test_solver.cpp:84-145).
StopDecision gpu_check_convergence(const std::vector<double>& resid_hist, const std::vector<double>& theta_hist,
                                   int i, double sigma1_estimate, double tol, double factor, bool use_stagnation);

}  // namespace minsvd
