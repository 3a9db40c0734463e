// Cholesky factor and its inverse for the preconditioner route
// (precond_chol.cu): G = R^T R (G symmetric positive definite, n <= 2048)
// and X = R^-1, both upper triangular, column-major.
//
// The factor comes from cuSOLVER potrf.  Its inverse is NOT a triangular
// solve with the identity (cuBLAS trsm: 0.55 ms at n = 1000; trtri 1.2 ms,
// scripts/micro_dense.cu): the 32 x 32 diagonal blocks are inverted by one
// warp each, and the inverse is assembled bottom-up with batched DMMA GEMMs,
// inv([A B; 0 C]) = [inv(A), -inv(A) B inv(C); 0, inv(C)], one level per
// doubling of the block size (the matrix padded with the identity to
// 32 * 2^L columns so every level is a regular strided batch).
//
// (A cooperative right-looking blocked Cholesky on 32 x 32 blocks measured
// slower than potrf -- 3.4 vs 1.1 ms at n = 1000, 96 grid-wide barriers -- and
// was removed in round 2.)

#include <cstdlib>
#include <string>

#include "common.cuh"
#include "msvd_internal.h"

namespace msvd {
namespace {

constexpr int kB = 32;        // block size

// Dinv[K] = inverse of the upper triangular 32 x 32 diagonal block K of R
// (one warp per block, lane = column, back substitution)
__global__ void __launch_bounds__(32) leaf_inverse_kernel(const double* R, int np, double* Dinv) {
    __shared__ double B[kB * kB];
    const int K = blockIdx.x, lane = threadIdx.x;
    const double* RKK = R + static_cast<int64_t>(K) * kB * (np + 1);
    for (int i = lane; i < kB * kB; i += 32) {
        const int r = i % kB, c = i / kB;
        B[i] = r <= c ? RKK[r + c * static_cast<int64_t>(np)] : 0.0;
    }
    __syncwarp();
    double x[kB];
#pragma unroll
    for (int i = kB - 1; i >= 0; --i) {
        double s = (i == lane) ? 1.0 : 0.0;
#pragma unroll
        for (int l = i + 1; l < kB; ++l) s -= B[i + l * kB] * x[l];
        x[i] = i <= lane ? s / B[i + i * kB] : 0.0;
    }
    double* D = Dinv + static_cast<int64_t>(K) * kB * kB;
#pragma unroll
    for (int i = 0; i < kB; ++i) D[i + lane * kB] = x[i];
}

// M (np x np): strictly lower triangle zeroed
__global__ void zero_lower_np_kernel(double* M, int np) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < static_cast<int64_t>(np) * np && i % np > i / np) M[i] = 0.0;
}

// X (np x np) := block-diagonal of the Dinv blocks, zero elsewhere
__global__ void place_diag_kernel(const double* Dinv, int np, double* X) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<int64_t>(np) * np) return;
    const int r = static_cast<int>(i % np), c = static_cast<int>(i / np);
    X[i] = (r / kB == c / kB) ? Dinv[static_cast<int64_t>(r / kB) * kB * kB + (r % kB) + (c % kB) * kB] : 0.0;
}

// Gp (np x np) = [G 0; 0 I]
__global__ void pad_kernel(const double* G, int64_t n, int np, double* Gp) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<int64_t>(np) * np) return;
    const int64_t r = i % np, c = i / np;
    Gp[i] = (r < n && c < n) ? G[r + c * n] : (r == c ? 1.0 : 0.0);
}
// out (n x n) = top-left block of Xp (np x np)
__global__ void unpad_kernel(const double* Xp, int np, int64_t n, double* out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n * n) return;
    out[i] = Xp[(i % n) + (i / n) * static_cast<int64_t>(np)];
}

unsigned blocks_of(int64_t count) { return static_cast<unsigned>(ceil_div(count, 256)); }

__global__ void info_to_flag_kernel(int* f) { *f = (*f == 0) ? 1 : 0; }

}  // namespace

int chol_pad_dim(int64_t n) {
    int np = kB;
    while (np < n) np *= 2;
    return np;
}

// R (n x n upper, lower zeroed) with R^T R = G and Rinv = R^-1 (n x n upper).
// ws: >= 3 np^2 + np * kB doubles (np = chol_pad_dim(n)).  Returns the
// success flag on the device (1 = G positive definite to working precision).
void chol_inverse(Ctx& c, const double* G, int64_t n, double* R, double* Rinv, double* ws, int* dflag) {
    if (!c.blas) {
        if (cublasCreate(&c.blas) != CUBLAS_STATUS_SUCCESS) fail(MSVD_ERR_CUDA, "cublasCreate failed");
        cublasSetPointerMode(c.blas, CUBLAS_POINTER_MODE_HOST);
    }
    if (cublasSetStream(c.blas, c.stream) != CUBLAS_STATUS_SUCCESS) fail(MSVD_ERR_CUDA, "cublasSetStream failed");
    const int np = chol_pad_dim(n);
    const int64_t nn = static_cast<int64_t>(np) * np;
    double* Gp = ws;            // np x np: padded G, then R
    double* X = Gp + nn;        // np x np: R^-1
    double* T = X + nn;         // np x np: GEMM scratch
    double* Dinv = T + nn;      // nb x 32 x 32
    pad_kernel<<<blocks_of(nn), 256, 0, c.stream>>>(G, n, np, Gp);
    {
        if (!c.solver && cusolverDnCreate(&c.solver) != CUSOLVER_STATUS_SUCCESS) fail(MSVD_ERR_CUDA, "cusolverDnCreate");
        if (cusolverDnSetStream(c.solver, c.stream) != CUSOLVER_STATUS_SUCCESS) fail(MSVD_ERR_CUDA, "cusolverDnSetStream");
        int lwork = 0;
        if (cusolverDnDpotrf_bufferSize(c.solver, CUBLAS_FILL_MODE_UPPER, np, Gp, np, &lwork) != CUSOLVER_STATUS_SUCCESS)
            fail(MSVD_ERR_CUDA, "potrf buffer size");
        // potrf's workspace: T (np x np, the GEMM scratch, free until the recursion)
        if (static_cast<int64_t>(lwork) > nn) fail(MSVD_ERR_CUDA, "potrf workspace larger than n^2");
        // dflag receives potrf's info (0 = ok); converted to 1 = ok below
        if (cusolverDnDpotrf(c.solver, CUBLAS_FILL_MODE_UPPER, np, Gp, np, T, lwork, dflag) !=
            CUSOLVER_STATUS_SUCCESS)
            fail(MSVD_ERR_CUDA, "potrf");
        info_to_flag_kernel<<<1, 1, 0, c.stream>>>(dflag);
        zero_lower_np_kernel<<<blocks_of(nn), 256, 0, c.stream>>>(Gp, np);
        leaf_inverse_kernel<<<np / kB, 32, 0, c.stream>>>(Gp, np, Dinv);
        c.launches += 3;
    }
    place_diag_kernel<<<blocks_of(nn), 256, 0, c.stream>>>(Dinv, np, X);
    c.launches += 3;
    // bottom-up: blocks of size s -> 2s: X12 = -X11 R12 X22 for every pair
    const double one = 1.0, zero = 0.0, mone = -1.0;
    for (int s = kB; s < np; s *= 2) {
        const int pairs = np / (2 * s);
        const long long stride = 2LL * s * (np + 1);  // from one pair's top-left corner to the next
        // T12 = R12 X22  (R12 at (0, s) of the pair, X22 at (s, s)); T at the same place in T
        if (cublasDgemmStridedBatched(c.blas, CUBLAS_OP_N, CUBLAS_OP_N, s, s, s, &one, Gp + static_cast<int64_t>(s) * np,
                                      np, stride, X + static_cast<int64_t>(s) * (np + 1), np, stride, &zero,
                                      T + static_cast<int64_t>(s) * np, np, stride, pairs) != CUBLAS_STATUS_SUCCESS)
            fail(MSVD_ERR_CUDA, "cuBLAS batched GEMM failed (triangular inverse)");
        // X12 = -X11 T12
        if (cublasDgemmStridedBatched(c.blas, CUBLAS_OP_N, CUBLAS_OP_N, s, s, s, &mone, X, np, stride,
                                      T + static_cast<int64_t>(s) * np, np, stride, &zero,
                                      X + static_cast<int64_t>(s) * np, np, stride, pairs) != CUBLAS_STATUS_SUCCESS)
            fail(MSVD_ERR_CUDA, "cuBLAS batched GEMM failed (triangular inverse)");
    }
    unpad_kernel<<<blocks_of(n * n), 256, 0, c.stream>>>(Gp, np, n, R);
    unpad_kernel<<<blocks_of(n * n), 256, 0, c.stream>>>(X, np, n, Rinv);
    MSVD_CUDA(cudaGetLastError());
    c.launches += 2;
}

}  // namespace msvd
