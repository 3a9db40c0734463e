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
// chol_coop_kernel below is a cooperative right-looking blocked Cholesky on
// 32 x 32 blocks; measured slower than potrf (3.4 vs 1.1 ms at n = 1000,
// 96 grid-wide barriers), it is kept only behind MSVD_CHOL_COOP = 1.
#include <cooperative_groups.h>

#include <cstdlib>
#include <string>

#include "common.cuh"
#include "msvd_internal.h"

namespace msvd {
namespace {

namespace cg = cooperative_groups;

constexpr int kB = 32;        // block size
constexpr int kCoopT = 256;   // threads per CTA (8 warps)

// out (32 x 32 block, column ld) = s * A^T B for 32 x 32 blocks A, B (lane = column of out):
// out(r, c) = s * sum_l A(l, r) B(l, c) [+ out(r, c) when acc]
__device__ __forceinline__ void block_atb(const double* A, int lda, const double* B, int ldb, double* out, int ldo,
                                          double s, bool acc, double* sh) {
    const int lane = threadIdx.x & 31;
    // A staged in shared memory (broadcast reads), B's column in registers
    for (int i = lane; i < kB * kB; i += 32) sh[i] = A[(i % kB) + (i / kB) * static_cast<int64_t>(lda)];
    double bc[kB];
#pragma unroll
    for (int l = 0; l < kB; ++l) bc[l] = B[l + lane * static_cast<int64_t>(ldb)];
    __syncwarp();
    for (int r = 0; r < kB; ++r) {
        double t = 0.0;
#pragma unroll
        for (int l = 0; l < kB; ++l) t += sh[l + r * kB] * bc[l];
        double* o = out + r + lane * static_cast<int64_t>(ldo);
        *o = acc ? *o + s * t : s * t;
    }
    __syncwarp();
}

// G (np x np, column-major, upper triangle used) -> R (upper, in place, lower
// zeroed) and Dinv[K] = R_KK^-1 for every diagonal block.  flag: 1 = success
__global__ void __launch_bounds__(kCoopT, 1) chol_coop_kernel(double* G, int np, double* Dinv, int* flag) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double shd[];  // 8 warps x one 32 x 32 staging block (64 KB, dynamic)
    double* sh[8];
    for (int w = 0; w < 8; ++w) sh[w] = shd + w * kB * kB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * 8 + warp, nwarps = gridDim.x * 8;
    const int nb = np / kB;
    for (int K = 0; K < nb; ++K) {
        double* GKK = G + static_cast<int64_t>(K) * kB * (np + 1);
        // A. diagonal block: warp 0 of CTA 0, lane = column
        if (blockIdx.x == 0 && warp == 0) {
            double col[kB];
#pragma unroll
            for (int i = 0; i < kB; ++i) col[i] = GKK[i + lane * static_cast<int64_t>(np)];
            bool ok = true;
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                double d = 0.0;
                if (lane == j) {
                    double s = col[j];
#pragma unroll
                    for (int i = 0; i < j; ++i) s -= col[i] * col[i];
                    d = s > 0.0 ? sqrt(s) : 0.0;
                }
                d = __shfl_sync(0xffffffffu, d, j);
                if (!(d > 0.0)) ok = false;
                double s = col[j];
#pragma unroll
                for (int i = 0; i < j; ++i) s -= __shfl_sync(0xffffffffu, col[i], j) * col[i];
                if (lane == j) col[j] = d;
                else if (lane > j) col[j] = d > 0.0 ? s / d : 0.0;
            }
            // write R_KK (upper, lower zeroed) and stage it for the inverse
            double* R = sh[0];
#pragma unroll
            for (int i = 0; i < kB; ++i) {
                const double v = i <= lane ? col[i] : 0.0;
                GKK[i + lane * static_cast<int64_t>(np)] = v;
                R[i + lane * kB] = v;
            }
            __syncwarp();
            // Dinv_K column lane: back substitution R x = e_lane
            double x[kB];
#pragma unroll
            for (int i = kB - 1; i >= 0; --i) {
                double s = (i == lane) ? 1.0 : 0.0;
#pragma unroll
                for (int l = i + 1; l < kB; ++l) s -= R[i + l * kB] * x[l];
                x[i] = i <= lane ? s / R[i + i * kB] : 0.0;
            }
            double* D = Dinv + static_cast<int64_t>(K) * kB * kB;
#pragma unroll
            for (int i = 0; i < kB; ++i) D[i + lane * kB] = x[i];
            if (!ok && lane == 0) *flag = 0;
            __syncwarp();
        }
        grid.sync();
        // B. row panel: R_KJ = Dinv_K^T G_KJ for J > K
        const double* D = Dinv + static_cast<int64_t>(K) * kB * kB;
        for (int J = K + 1 + gw; J < nb; J += nwarps) {
            double* GKJ = G + static_cast<int64_t>(K) * kB + static_cast<int64_t>(J) * kB * np;
            // out = D^T GKJ, written back in place through a staging copy of GKJ
            double* sB = sh[warp];
            for (int i = lane; i < kB * kB; i += 32) sB[i] = GKJ[(i % kB) + (i / kB) * static_cast<int64_t>(np)];
            __syncwarp();
            double bc[kB];
#pragma unroll
            for (int l = 0; l < kB; ++l) bc[l] = sB[l + lane * kB];
            __syncwarp();
            for (int i = lane; i < kB * kB; i += 32) sB[i] = D[i];
            __syncwarp();
            for (int r = 0; r < kB; ++r) {
                double t = 0.0;
#pragma unroll
                for (int l = 0; l < kB; ++l) t += sB[l + r * kB] * bc[l];
                GKJ[r + lane * static_cast<int64_t>(np)] = t;
            }
            __syncwarp();
        }
        grid.sync();
        // C. trailing update: G_IJ -= R_KI^T R_KJ for K < I <= J
        const int nt = nb - K - 1;
        const int tiles = nt * (nt + 1) / 2;
        for (int t = gw; t < tiles; t += nwarps) {
            // t -> (I, J), column-major over the upper triangle of the trailing blocks
            int jj = 0, base = 0;
            while (base + jj + 1 <= t) {
                base += jj + 1;
                ++jj;
            }
            const int I = K + 1 + (t - base), J = K + 1 + jj;
            block_atb(G + static_cast<int64_t>(K) * kB + static_cast<int64_t>(I) * kB * np, np,
                      G + static_cast<int64_t>(K) * kB + static_cast<int64_t>(J) * kB * np, np,
                      G + static_cast<int64_t>(I) * kB + static_cast<int64_t>(J) * kB * np, np, -1.0, true, sh[warp]);
        }
        grid.sync();
    }
    // zero the strictly lower triangle
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < static_cast<int64_t>(np) * np;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (i % np > i / np) G[i] = 0.0;
}

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
    const char* ce = std::getenv("MSVD_CHOL_COOP");
    if (ce && std::atoi(ce) == 1) {
        const int one_i = 1;
        MSVD_CUDA(cudaMemcpyAsync(dflag, &one_i, sizeof(int), cudaMemcpyHostToDevice, c.stream));
        int per_sm = 0;
        const size_t smem = sizeof(double) * 8 * kB * kB;
        optin_smem(c, chol_coop_kernel);
        MSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chol_coop_kernel, kCoopT, smem));
        if (per_sm < 1) fail(MSVD_ERR_CUDA, "msvd: cooperative Cholesky kernel cannot be resident");
        int npi = np;
        void* args[] = {&Gp, &npi, &Dinv, &dflag};
        MSVD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(chol_coop_kernel), c.num_sms, kCoopT, args,
                                              smem, c.stream));
        ++c.launches;
    } else {
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
