// Householder TSQR fold shared by the TSQR kernel, the Rayleigh-Ritz kernel
// and the A*W kernel with the fused TSQR epilogue.
#pragma once

#include "common.cuh"

namespace msvd {

// ---------------------------------------------------------------------------
// Householder fold of a 32-row block X into an upper-triangular R held in
// shared memory (column-major, leading dimension KM): the QR step of a TSQR
// on [R; X].  Lane i holds row i of X in x[].  The reflector sign convention
// follows svd.cpp:37 (alpha = -sign(x_k) ||x||), so every R produced here is
// the reference's householder_qr R up to roundoff and row signs -- and the
// Jacobi SVD that consumes it depends only on R^T R (svd.cpp:113-117).
// ---------------------------------------------------------------------------

template <int KM>
__device__ void fold_rows(double* R, double (&x)[KM], int k) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        if (j >= k) break;
        const double rjj = R[j + j * KM];
        const double xj = x[j];
        const double ss = warp_sum(xj * xj);
        const double nrm2 = rjj * rjj + ss;
        if (nrm2 == 0.0) continue;  // svd.cpp:33-36 (zero column: beta = 0)
        const double xnorm = sqrt(nrm2);
        const double alpha = rjj >= 0.0 ? -xnorm : xnorm;
        const double v0 = rjj - alpha;
        const double vi = xj / v0;
        const double beta = -v0 / alpha;
        double d[KM];
#pragma unroll
        for (int l = j + 1; l < KM; ++l) d[l] = l < k ? vi * x[l] : 0.0;
#pragma unroll
        for (int l = j + 1; l < KM; ++l)
            if (l < k) d[l] = warp_sum(d[l]);
#pragma unroll
        for (int l = j + 1; l < KM; ++l) {
            if (l < k) {
                const double rjl = R[j + l * KM];
                const double s = (rjl + d[l]) * beta;
                d[l] = rjl - s;  // new R(j, l)
                x[l] -= s * vi;
            }
        }
        x[j] = 0.0;
        __syncwarp();
        if (lane == 0) {
            R[j + j * KM] = alpha;
#pragma unroll
            for (int l = j + 1; l < KM; ++l)
                if (l < k) R[j + l * KM] = d[l];
        }
        __syncwarp();
    }
}

// rows of another upper-triangular R2 (ld KM) as the X block of a fold
template <int KM>
__device__ __forceinline__ void rows_of(const double* R2, int k, double (&x)[KM]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int l = 0; l < KM; ++l) x[l] = (lane < k && l >= lane && l < k) ? R2[lane + l * KM] : 0.0;
}

}  // namespace msvd
