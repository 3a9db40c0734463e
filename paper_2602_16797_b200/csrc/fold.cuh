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

namespace msvd {

// Shared-memory form of the same Householder fold, for wide trial blocks:
// lane l owns column l of the stacked [R; X] block, so each reflector costs
// plain FMAs over shared memory instead of k butterfly reductions.
//   Rs: k x k upper triangular, column-major, leading dimension KM
//   Xs: 32 x k rows, row-major, leading dimension XLD (= KM + 1: no conflicts)
// Same reflector convention as fold_rows (svd.cpp:37).
template <int KM>
__device__ void fold_smem(double* Rs, double* Xs, int k) {
    constexpr int XLD = KM + 1;
    const int lane = threadIdx.x & 31;
    __syncwarp();
    for (int j = 0; j < k; ++j) {
        double beta = 0.0, inv = 0.0;
        int skip = 0;
        if (lane == j) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                const double a0 = Xs[i * XLD + j], a1 = Xs[(i + 1) * XLD + j];
                const double a2 = Xs[(i + 2) * XLD + j], a3 = Xs[(i + 3) * XLD + j];
                s0 = fma(a0, a0, s0);
                s1 = fma(a1, a1, s1);
                s2 = fma(a2, a2, s2);
                s3 = fma(a3, a3, s3);
            }
            const double rjj = Rs[j + j * KM];
            const double nrm2 = rjj * rjj + ((s0 + s1) + (s2 + s3));
            if (nrm2 == 0.0) {
                skip = 1;  // svd.cpp:33-36
            } else {
                const double xnorm = sqrt(nrm2);
                const double alpha = rjj >= 0.0 ? -xnorm : xnorm;
                const double v0 = rjj - alpha;
                beta = -v0 / alpha;
                inv = 1.0 / v0;
                Rs[j + j * KM] = alpha;
            }
        }
        skip = __shfl_sync(kFull, skip, j);
        if (skip) continue;
        beta = __shfl_sync(kFull, beta, j);
        inv = __shfl_sync(kFull, inv, j);
        if (lane > j && lane < k) {
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                d0 = fma(Xs[i * XLD + j], Xs[i * XLD + lane], d0);
                d1 = fma(Xs[(i + 1) * XLD + j], Xs[(i + 1) * XLD + lane], d1);
                d2 = fma(Xs[(i + 2) * XLD + j], Xs[(i + 2) * XLD + lane], d2);
                d3 = fma(Xs[(i + 3) * XLD + j], Xs[(i + 3) * XLD + lane], d3);
            }
            const double rjl = Rs[j + lane * KM];
            const double s = (rjl + inv * ((d0 + d1) + (d2 + d3))) * beta;
            Rs[j + lane * KM] = rjl - s;
            const double si = s * inv;
#pragma unroll
            for (int i = 0; i < 32; ++i) Xs[i * XLD + lane] -= si * Xs[i * XLD + j];
        }
        __syncwarp();
    }
}

// the rows of an upper-triangular R2 (ld KM) as the X block of fold_smem
template <int KM>
__device__ __forceinline__ void load_rows_smem(const double* R2, int k, double* Xs) {
    constexpr int XLD = KM + 1;
    const int lane = threadIdx.x & 31;
    for (int l = 0; l < k; ++l) Xs[lane * XLD + l] = (lane < k && l >= lane) ? R2[lane + l * KM] : 0.0;
    __syncwarp();
}

}  // namespace msvd
