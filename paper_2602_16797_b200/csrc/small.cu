// TSQR, Rayleigh-Ritz and the n-scale control kernels.
//
// Everything between the two A passes stays on the device: the host only
// launches and, at check iterations, reads the stop/error words.
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "fold.cuh"
#include "msvd_internal.h"

namespace msvd {

namespace {

constexpr double kEps = 2.220446049250313e-16;

struct TsqrArgs {
    Cols T;
    int64_t m;
    int k;
    double* Rparts;  // [grid][k][k]
    DevState* st;
    int iter;
    const int* skip;  // nonzero: the Cholesky QR2 of the block was usable, nothing to do
};

// per-CTA TSQR: 8 warps fold 32-row tiles round-robin, then a 3-level tree
template <int KM>
__global__ void __launch_bounds__(256) tsqr_kernel(TsqrArgs a) {
    if (a.skip && *a.skip) return;
    __shared__ double Rw[8][KM * KM];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = lane; i < KM * KM; i += 32) Rw[warp][i] = 0.0;
    __syncwarp();
    const int64_t r0 = (a.m * blockIdx.x) / gridDim.x;
    const int64_t r1 = (a.m * (blockIdx.x + 1)) / gridDim.x;
    const int64_t ntiles = ceil_div(r1 - r0, 32);
    bool finite = true;
    for (int64_t t = warp; t < ntiles; t += 8) {
        const int64_t row = r0 + t * 32 + lane;
        double x[KM];
#pragma unroll
        for (int l = 0; l < KM; ++l) {
            x[l] = (l < a.k && row < r1) ? a.T.p[l][row] : 0.0;
            finite = finite && isfinite(x[l]);
        }
        fold_rows<KM>(Rw[warp], x, a.k);
    }
    if (!__all_sync(kFull, finite) && lane == 0 && a.st) {
        if (atomicCAS(&a.st->err_code, 0, kErrNonfiniteAT) == 0) a.st->err_iter = a.iter;
    }
    __syncthreads();
#pragma unroll
    for (int s = 1; s < 8; s <<= 1) {
        if ((warp % (2 * s)) == 0) {
            double x[KM];
            rows_of<KM>(Rw[warp + s], a.k, x);
            fold_rows<KM>(Rw[warp], x, a.k);
        }
        __syncthreads();
    }
    double* out = a.Rparts + static_cast<size_t>(blockIdx.x) * a.k * a.k;
    for (int i = threadIdx.x; i < a.k * a.k; i += blockDim.x) {
        const int r = i % a.k, cc = i / a.k;
        out[i] = r <= cc ? Rw[0][r + cc * KM] : 0.0;
    }
}

// Narrow trial blocks (k <= 8): the CTA's rows in chunks of 512 * RPT, each
// chunk folded into the CTA's R in ONE Householder step with the whole CTA
// (every thread holds RPT rows in registers; two fixed-order block
// reductions per reflector) -- fold_rows' arithmetic with the chunk as the
// X block, instead of a chain of 32-row warp folds.
template <int KM, int RPT>
__global__ void __launch_bounds__(512) tsqr_stacked_kernel(TsqrArgs a) {
    if (a.skip && *a.skip) return;
    __shared__ double R[KM * KM];
    __shared__ double red[2][16][KM + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NW = 16;
    const int k = a.k;
    for (int i = threadIdx.x; i < KM * KM; i += blockDim.x) R[i] = 0.0;
    const int64_t r0 = (a.m * blockIdx.x) / gridDim.x;
    const int64_t r1 = (a.m * (blockIdx.x + 1)) / gridDim.x;
    bool finite = true;
    int buf = 0;
    auto block_sums = [&](double (&v)[KM], int cnt, double (&out)[KM]) {
        double(*rb)[KM + 1] = red[buf];
        buf ^= 1;
#pragma unroll
        for (int l = 0; l < KM; ++l)
            if (l < cnt) {
                const double t = warp_sum(v[l]);
                if (lane == 0) rb[warp][l] = t;
            }
        __syncthreads();
#pragma unroll
        for (int l = 0; l < KM; ++l) {
            double t = 0.0;
            if (l < cnt)
#pragma unroll
                for (int w = 0; w < NW; ++w) t += rb[w][l];
            out[l] = t;
        }
    };
    __syncthreads();
    for (int64_t base = r0; base < r1; base += 512 * RPT) {
        double x[RPT][KM];
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int64_t row = base + threadIdx.x + 512 * i;
#pragma unroll
            for (int l = 0; l < KM; ++l) {
                x[i][l] = (l < k && row < r1) ? a.T.p[l][row] : 0.0;
                finite = finite && isfinite(x[i][l]);
            }
        }
#pragma unroll
        for (int j = 0; j < KM; ++j) {  // unrolled: x stays in registers (a runtime j would index it in local memory)
            if (j >= k) break;
            double v[KM], o[KM];
#pragma unroll
            for (int l = 0; l < KM; ++l) v[l] = 0.0;
#pragma unroll
            for (int i = 0; i < RPT; ++i) v[0] += x[i][j] * x[i][j];
            block_sums(v, 1, o);
            const double rjj = R[j + j * KM];
            const double nrm2 = rjj * rjj + o[0];
            if (nrm2 == 0.0) continue;  // svd.cpp:33-36
            const double xnorm = sqrt(nrm2);
            const double alpha = rjj >= 0.0 ? -xnorm : xnorm;
            const double v0 = rjj - alpha;
            const double beta = -v0 / alpha;
#pragma unroll
            for (int l = 0; l < KM; ++l) v[l] = 0.0;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const double vi = x[i][j] / v0;
#pragma unroll
                for (int l = 0; l < KM; ++l)
                    if (l > j && l < k) v[l] += vi * x[i][l];
            }
            block_sums(v, k, o);
            double sl[KM];
#pragma unroll
            for (int l = 0; l < KM; ++l) sl[l] = (l > j && l < k) ? (R[j + l * KM] + o[l]) * beta : 0.0;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const double vi = x[i][j] / v0;
#pragma unroll
                for (int l = 0; l < KM; ++l)
                    if (l > j && l < k) x[i][l] -= sl[l] * vi;
                x[i][j] = 0.0;
            }
            __syncthreads();  // every thread has read R's row j
            if (threadIdx.x == 0) {
                for (int l = j + 1; l < k; ++l) R[j + l * KM] -= sl[l];
                R[j + j * KM] = alpha;
            }
            __syncthreads();
        }
    }
    if (!__all_sync(kFull, finite) && lane == 0 && a.st) {
        if (atomicCAS(&a.st->err_code, 0, kErrNonfiniteAT) == 0) a.st->err_iter = a.iter;
    }
    double* out = a.Rparts + static_cast<size_t>(blockIdx.x) * k * k;
    for (int i = threadIdx.x; i < k * k; i += blockDim.x) {
        const int r = i % k, cc = i / k;
        out[i] = r <= cc ? R[r + cc * KM] : 0.0;
    }
}

// Wide trial blocks: 16 warps per CTA, shared-memory folds (fold_smem)
template <int KM>
__global__ void __launch_bounds__(512) tsqr_smem_kernel(TsqrArgs a) {
    if (a.skip && *a.skip) return;
    extern __shared__ __align__(16) double tsm[];
    constexpr int XLD = KM + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    double* Rw = tsm + warp * KM * KM;
    double* Xs = tsm + nw * KM * KM + warp * 32 * XLD;
    for (int i = lane; i < KM * KM; i += 32) Rw[i] = 0.0;
    const int64_t r0 = (a.m * blockIdx.x) / gridDim.x;
    const int64_t r1 = (a.m * (blockIdx.x + 1)) / gridDim.x;
    const int64_t ntiles = ceil_div(r1 - r0, 32);
    bool finite = true;
    for (int64_t t = warp; t < ntiles; t += nw) {
        const int64_t row = r0 + t * 32 + lane;
        double v[KM];  // all loads in flight before the first shared store
#pragma unroll
        for (int l = 0; l < KM; ++l) v[l] = (l < a.k && row < r1) ? a.T.p[l][row] : 0.0;
#pragma unroll
        for (int l = 0; l < KM; ++l)
            if (l < a.k) {
                finite = finite && isfinite(v[l]);
                Xs[lane * XLD + l] = v[l];
            }
        fold_smem<KM>(Rw, Xs, a.k);
    }
    if (!__all_sync(kFull, finite) && lane == 0 && a.st) {
        if (atomicCAS(&a.st->err_code, 0, kErrNonfiniteAT) == 0) a.st->err_iter = a.iter;
    }
    __syncthreads();
    for (int s = 1; s < nw; s <<= 1) {
        if ((warp % (2 * s)) == 0 && warp + s < nw) {
            load_rows_smem<KM>(tsm + (warp + s) * KM * KM, a.k, Xs);
            fold_smem<KM>(Rw, Xs, a.k);
        }
        __syncthreads();
    }
    double* out = a.Rparts + static_cast<size_t>(blockIdx.x) * a.k * a.k;
    for (int i = threadIdx.x; i < a.k * a.k; i += blockDim.x) {
        const int r = i % a.k, cc = i / a.k;
        out[i] = r <= cc ? tsm[r + cc * KM] : 0.0;
    }
}

// ---------------------------------------------------------------------------
// One-sided Jacobi SVD of a k x k (k <= 24) matrix in shared memory with a
// round-robin parallel pair order (one warp per pair, lanes over rows); the
// per-pair rotation, the 1e-15 tolerance, the 60-sweep cap and the
// convergence test are svd.cpp:99-150.  Then sigma = column norms, stable
// descending sort, largest-|entry|-positive signs (svd.cpp:200-248).
// Must be called by all threads of the CTA (blockDim >= 32 * 12).
// ---------------------------------------------------------------------------
template <int KM>
__device__ bool jacobi_svd(double* Bm, double* V, int k, double* sig, double* Vs, int* ord,
                           double* worst_s) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < KM * KM; i += blockDim.x) V[i] = ((i % KM) == (i / KM)) ? 1.0 : 0.0;
    const int K2 = k + (k & 1);
    bool converged = (k <= 1);
    __syncthreads();
    for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
        if (threadIdx.x == 0) *worst_s = 0.0;
        __syncthreads();
        for (int r = 0; r < K2 - 1; ++r) {
            if (warp < K2 / 2) {
                int p, q;
                if (warp == 0) {
                    p = r;
                    q = K2 - 1;
                } else {
                    p = (r + warp) % (K2 - 1);
                    q = (r - warp + (K2 - 1)) % (K2 - 1);
                }
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                if (q < k) {
                    const double bp = lane < k ? Bm[lane + p * KM] : 0.0;
                    const double bq = lane < k ? Bm[lane + q * KM] : 0.0;
                    const double app = warp_sum(bp * bp);
                    const double aqq = warp_sum(bq * bq);
                    const double apq = warp_sum(bp * bq);
                    if (!(app == 0.0 || aqq == 0.0 || apq == 0.0)) {
                        // svd.cpp:113-131 with the serial sqrt / divide chain shortened: the
                        // cosine test |apq| / sqrt(app aqq) > 1e-15 squared (no sqrt, no
                        // divide), t = sign(tau) / (|tau| + sqrt(1 + tau^2)) with tau =
                        // zeta / (2 apq) written as 2 apq sign(zeta) / (|zeta| + sqrt(zeta^2 +
                        // 4 apq^2)) (one sqrt, one divide), c = rsqrt(1 + t^2)
                        const bool big = apq * apq > 1e-30 * (app * aqq);
                        if (lane == 0 && big) *worst_s = 1.0;  // (every writer stores the same value)
                        if (big) {
                            const double zeta = aqq - app;
                            const double t = (zeta >= 0.0 ? 2.0 : -2.0) * apq /
                                             (fabs(zeta) + sqrt(fma(zeta, zeta, 4.0 * apq * apq)));
                            const double c = rsqrt(fma(t, t, 1.0));
                            const double sn = c * t;
                            if (lane < k) {
                                Bm[lane + p * KM] = c * bp - sn * bq;
                                Bm[lane + q * KM] = sn * bp + c * bq;
                                const double vp = V[lane + p * KM], vq = V[lane + q * KM];
                                V[lane + p * KM] = c * vp - sn * vq;
                                V[lane + q * KM] = sn * vp + c * vq;
                            }
                        }
                    }
                }
            }
            __syncthreads();
        }
        converged = *worst_s <= 1e-15;
        __syncthreads();
        if (threadIdx.x == 0) worst_s[1] = sweep + 1;  // sweeps used (diagnostics)
    }
    if (threadIdx.x < k) {
        double s = 0.0;
        for (int i = 0; i < k; ++i) s += Bm[i + threadIdx.x * KM] * Bm[i + threadIdx.x * KM];
        sig[threadIdx.x] = sqrt(s);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int j = 0; j < k; ++j) ord[j] = j;
        for (int j = 1; j < k; ++j) {
            const int key = ord[j];
            int i = j - 1;
            while (i >= 0 && sig[key] > sig[ord[i]]) {
                ord[i + 1] = ord[i];
                --i;
            }
            ord[i + 1] = key;
        }
    }
    __syncthreads();
    if (threadIdx.x < k) {
        const int j = threadIdx.x, src = ord[j];
        int imax = 0;
        double amax = -1.0;
        for (int i = 0; i < k; ++i) {
            const double v = fabs(V[i + src * KM]);
            if (v > amax) {
                amax = v;
                imax = i;
            }
        }
        const double sgn = V[imax + src * KM] < 0.0 ? -1.0 : 1.0;
        for (int i = 0; i < k; ++i) Vs[i + j * KM] = sgn * V[i + src * KM];
    }
    __syncthreads();
    const double s_sorted = threadIdx.x < k ? sig[ord[threadIdx.x]] : 0.0;
    __syncthreads();
    if (threadIdx.x < k) sig[threadIdx.x] = s_sorted;
    __syncthreads();
    return converged;
}

// ---------------------------------------------------------------------------
// Rayleigh-Ritz (solver.cpp:352-355 init, :417-421 and :453-462 iteration)
// ---------------------------------------------------------------------------
// Merge of the per-CTA R factors as ONE Householder QR of the stacked
// (nparts k) x k matrix with the whole CTA (small k): each reflector is two
// fixed-order block reductions instead of a chain of per-part warp folds.
// Same reflector arithmetic as fold_rows (svd.cpp:37 sign convention), so the
// merged R is the TSQR's up to roundoff.  Ms: rows x (KM + 1) scratch;
// red: 2 x 17 x (KM + 1) scratch.  Called by all threads; R -> Rout (ld KM).
// TOP: Rprev (shared memory, ld KM), an R already merged, is stacked on top,
// so parts that do not all fit in shared memory are merged group by group.
template <int KM, bool TOP = false>
__device__ void stacked_qr(const double* Rparts, int nparts, int k, double* Ms, double* red, double* Rout,
                           const double* Rprev = nullptr) {
    constexpr int LD = KM + 1;
    const int top = TOP ? k : 0;
    const int rows = top + nparts * k;
    const int nthr = blockDim.x, nw = nthr >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int idx = threadIdx.x; idx < rows * k; idx += nthr) {
        const int r = idx / k, l = idx - r * k;
        if (TOP && r < top) {
            Ms[r * LD + l] = l >= r ? Rprev[r + l * KM] : 0.0;
        } else {
            const int p = (r - top) / k, i = (r - top) - p * k;
            Ms[r * LD + l] = l >= i ? Rparts[static_cast<size_t>(p) * k * k + i + l * k] : 0.0;
        }
    }
    __syncthreads();
    int buf = 0;
    // sum over warps in fixed order of per-thread values v[0..cnt)
    auto block_sums = [&](double (&v)[KM], int cnt, double (&out)[KM]) {
        double* rb = red + buf * 17 * LD;
        buf ^= 1;
        if constexpr (KM <= 8) {  // few values: per-value butterflies, every thread adds the warps
#pragma unroll
            for (int l = 0; l < KM; ++l)
                if (l < cnt) {
                    const double t = warp_sum(v[l]);
                    if (lane == 0) rb[warp * LD + l] = t;
                }
            __syncthreads();
#pragma unroll
            for (int l = 0; l < KM; ++l) {
                double t = 0.0;
                if (l < cnt)
                    for (int w = 0; w < nw; ++w) t += rb[w * LD + l];
                out[l] = t;
            }
        } else {  // many: one transpose-reduce per warp, threads l < cnt add the warps
            double t16[16];
#pragma unroll
            for (int l = 0; l < 16; ++l) t16[l] = l < KM && l < cnt ? v[l < KM ? l : 0] : 0.0;
            const double t = warp_transpose_reduce<16>(t16);
            if (lane < cnt) rb[warp * LD + lane] = t;
            __syncthreads();
            if (threadIdx.x < cnt) {
                double sum = 0.0;
                for (int w = 0; w < nw; ++w) sum += rb[w * LD + threadIdx.x];
                rb[16 * LD + threadIdx.x] = sum;
            }
            __syncthreads();
#pragma unroll
            for (int l = 0; l < KM; ++l) out[l] = l < cnt ? rb[16 * LD + l] : 0.0;
        }
    };
    for (int j = 0; j < k; ++j) {
        double v[KM], o[KM];
#pragma unroll
        for (int l = 0; l < KM; ++l) v[l] = 0.0;
        for (int r = j + 1 + threadIdx.x; r < rows; r += nthr) v[0] += Ms[r * LD + j] * Ms[r * LD + j];
        block_sums(v, 1, o);
        const double rjj = Ms[j * LD + j];
        const double nrm2 = rjj * rjj + o[0];
        if (nrm2 == 0.0) continue;  // svd.cpp:33-36
        const double xnorm = sqrt(nrm2);
        const double alpha = rjj >= 0.0 ? -xnorm : xnorm;
        const double v0 = rjj - alpha;
        const double beta = -v0 / alpha;
#pragma unroll
        for (int l = 0; l < KM; ++l) v[l] = 0.0;
        for (int r = j + 1 + threadIdx.x; r < rows; r += nthr) {
            const double vr = Ms[r * LD + j] / v0;
#pragma unroll
            for (int l = 0; l < KM; ++l)
                if (l > j && l < k) v[l] += vr * Ms[r * LD + l];
        }
        block_sums(v, k, o);
        __syncthreads();  // every thread has read row j and column j before they change
        for (int r = j + 1 + threadIdx.x; r < rows; r += nthr) {
            const double vr = Ms[r * LD + j] / v0;
#pragma unroll
            for (int l = 0; l < KM; ++l)
                if (l > j && l < k) {
                    const double sl = (Ms[j * LD + l] + o[l]) * beta;
                    Ms[r * LD + l] -= sl * vr;
                }
            Ms[r * LD + j] = 0.0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
            for (int l = 0; l < KM; ++l)
                if (l > j && l < k) {
                    const double rjl = Ms[j * LD + l];
                    Ms[j * LD + l] = rjl - (rjl + o[l]) * beta;
                }
            Ms[j * LD + j] = alpha;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < KM * KM; i += nthr) {
        const int r = i % KM, c = i / KM;
        Rout[i] = (r < k && c < k && r <= c) ? Ms[r * LD + c] : 0.0;
    }
    __syncthreads();
}

// the rr kernel's fold scratch lives after its other shared arrays
template <int KM>
__device__ __forceinline__ double* rr_scratch(double* sh) {
    return sh + (16 * KM * KM + 3 * KM * KM + KM + 2 * KM * kMaxB + 2) + (KM + 1) / 2 + 2;
}
#define ord_end_scratch(sh, KM) rr_scratch<KM>(sh)
// doubles of the rr kernel's fixed shared layout (arrays + per-warp fold scratch)
template <int KM>
__host__ __device__ constexpr size_t rr_base_words() {
    return (16 * KM * KM + 3 * KM * KM + KM + 2 * KM * kMaxB + 2) + (KM + 1) / 2 + 2 + 16 * 32 * (KM + 1) + 8;
}

template <int KM>
__global__ void __launch_bounds__(512) rr_kernel(RRArgs a) {
    extern __shared__ __align__(16) double sh[];
    double* Rw = sh;                      // [16][KM*KM]
    double* Bm = Rw + 16 * KM * KM;       // KM*KM
    double* V = Bm + KM * KM;             // KM*KM
    double* Vs = V + KM * KM;             // KM*KM sorted/sign-fixed
    double* sig = Vs + KM * KM;           // KM
    double* q = sig + KM;                 // KM*KMAXB  orth coefficients (lead x b)
    double* mix = q + KM * kMaxB;         // KM*kMaxB
    double* worst = mix + KM * kMaxB;     // 1
    int* ord = reinterpret_cast<int*>(worst + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = a.k, b = a.b;

    // 1. merge the partial R factors.  Small k with room in shared memory:
    // one stacked Householder QR with the whole CTA; otherwise warp w folds
    // parts w, w+16, ... and a tree merges the warps.
    unsigned dyn_smem;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn_smem));
    const size_t stacked_words = static_cast<size_t>(a.nparts) * k * (KM + 1) + 2 * 17 * (KM + 1);
    const size_t base_words = rr_base_words<KM>();
    // KM = 16: the parts in groups that fit, each group stacked under the R so far
    const int64_t room = static_cast<int64_t>(dyn_smem / sizeof(double)) -
                         static_cast<int64_t>(base_words + 2 * 17 * (KM + 1));
    const int group = KM == 16 && room > 0 ? static_cast<int>(room / (k * (KM + 1))) - 1 : 0;
    if (a.chol_ok && *a.chol_ok) {  // the block's R from Cholesky QR2 (trial_qr.cu)
        for (int i = threadIdx.x; i < KM * KM; i += blockDim.x) {
            const int r = i % KM, c = i / KM;
            Bm[i] = (r < k && c < k && r <= c) ? a.chol_R[r + c * k] : 0.0;
        }
    } else if (KM <= 8 && (base_words + stacked_words) * sizeof(double) <= dyn_smem) {
        double* Ms = sh + base_words;
        stacked_qr<KM>(a.Rparts, a.nparts, k, Ms + 2 * 17 * (KM + 1), Ms, Bm);
    } else if (KM == 16 && group >= 8) {
        double* Ms = sh + base_words;
        stacked_qr<KM>(a.Rparts, min(group, a.nparts), k, Ms + 2 * 17 * (KM + 1), Ms, Bm);
        for (int p0 = group; p0 < a.nparts; p0 += group)
            stacked_qr<KM, true>(a.Rparts + static_cast<size_t>(p0) * k * k, min(group, a.nparts - p0), k,
                                 Ms + 2 * 17 * (KM + 1), Ms, Bm, Bm);
    } else {
    for (int i = lane; i < KM * KM; i += 32) Rw[warp * KM * KM + i] = 0.0;
    __syncwarp();
    const int nw = blockDim.x >> 5;
    double* Xs = ord_end_scratch(sh, KM) + warp * 32 * (KM + 1);
    double xn[KM];
    if (warp < a.nparts) {
        const double* R0 = a.Rparts + static_cast<size_t>(warp) * k * k;
#pragma unroll
        for (int l = 0; l < KM; ++l) xn[l] = (lane < k && l >= lane && l < k) ? R0[lane + l * k] : 0.0;
    }
    for (int pi = warp; pi < a.nparts; pi += nw) {
        const double* R2 = a.Rparts + static_cast<size_t>(pi) * k * k;
        if constexpr (KM >= 8) {
            double v[KM];
#pragma unroll
            for (int l = 0; l < KM; ++l) v[l] = (lane < k && l >= lane && l < k) ? R2[lane + l * k] : 0.0;
#pragma unroll
            for (int l = 0; l < KM; ++l)
                if (l < k) Xs[lane * (KM + 1) + l] = v[l];
            fold_smem<KM>(Rw + warp * KM * KM, Xs, k);
        } else {
            double x[KM];
#pragma unroll
            for (int l = 0; l < KM; ++l) x[l] = xn[l];
            if (pi + nw < a.nparts) {  // prefetch the next part while this one folds
                const double* Rn = a.Rparts + static_cast<size_t>(pi + nw) * k * k;
#pragma unroll
                for (int l = 0; l < KM; ++l) xn[l] = (lane < k && l >= lane && l < k) ? Rn[lane + l * k] : 0.0;
            }
            fold_rows<KM>(Rw + warp * KM * KM, x, k);
        }
    }
    __syncthreads();
    for (int s = 1; s < nw; s <<= 1) {
        if ((warp % (2 * s)) == 0 && warp + s < nw) {
            if constexpr (KM >= 8) {
                load_rows_smem<KM>(Rw + (warp + s) * KM * KM, k, Xs);
                fold_smem<KM>(Rw + warp * KM * KM, Xs, k);
            } else {
                double x[KM];
                rows_of<KM>(Rw + (warp + s) * KM * KM, k, x);
                fold_rows<KM>(Rw + warp * KM * KM, x, k);
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < KM * KM; i += blockDim.x) {
        const int r = i % KM, c = i / KM;
        Bm[i] = (r < k && c < k && r <= c) ? Rw[i] : 0.0;
    }
    }
    __syncthreads();
    if (a.R_out)
        for (int i = threadIdx.x; i < k * k; i += blockDim.x) a.R_out[i] = Bm[(i % k) + (i / k) * KM];
    if (a.mode == 2) return;

    // 2. SVD of R (svd.cpp:180-252)
    const bool ok = jacobi_svd<KM>(Bm, V, k, sig, Vs, ord, worst);
    if (!ok && threadIdx.x == 0) {
        if (atomicCAS(&a.st->err_code, 0, kErrJacobi) == 0) a.st->err_iter = a.iter;
    }
    if (a.sig_out && threadIdx.x < k) a.sig_out[threadIdx.x] = sig[threadIdx.x];
    if (a.Vfull_out)
        for (int i = threadIdx.x; i < k * k; i += blockDim.x) a.Vfull_out[i] = Vs[(i % k) + (i / k) * KM];

    // 3. target block: last b Ritz pairs
    const int lead = k - b;
    if (threadIdx.x < b) {
        const double th = sig[lead + threadIdx.x];
        a.theta_out[threadIdx.x] = th;
    }
    for (int i = threadIdx.x; i < k * b; i += blockDim.x) {
        const int r = i % k, j = i / k;
        a.Cm[r + j * k] = Vs[r + (lead + j) * KM];
    }
    // 4. history coefficients: q = orth_coefficients(C(0:b, 0:lead)^T), mix = V(:,0:lead) q
    if (a.mode == 1 && warp == 0) {
        // g (lead x b): g(j,l) = Vs(l, j); lane = row j of g
        double sref = 0.0;
        for (int l = 0; l < b; ++l) {
            const double gv = lane < lead ? Vs[l + lane * KM] : 0.0;
            sref = fmax(sref, sqrt(warp_sum(gv * gv)));
        }
        bool collapsed = false;
        for (int j = 0; j < b; ++j) {
            double w = lane < lead ? Vs[j + lane * KM] : 0.0;
            for (int pass = 0; pass < 2; ++pass)
                for (int l = 0; l < j; ++l) {
                    const double ql = lane < lead ? q[lane + l * KM] : 0.0;
                    const double pr = warp_sum(ql * w);
                    w -= pr * ql;
                }
            const double nrm = sqrt(warp_sum(w * w));
            if (nrm <= 1e-14 * fmax(1.0, sref)) {
                bool placed = false;
                for (int cand = 0; cand < lead && !placed; ++cand) {
                    double e = lane == cand ? 1.0 : 0.0;
                    for (int pass = 0; pass < 2; ++pass)
                        for (int l = 0; l < j; ++l) {
                            const double ql = lane < lead ? q[lane + l * KM] : 0.0;
                            const double pr = warp_sum(ql * e);
                            e -= pr * ql;
                        }
                    const double en = sqrt(warp_sum(e * e));
                    if (en > 1e-8) {
                        w = e * (1.0 / en);
                        placed = true;
                    }
                }
                if (!placed) collapsed = true;
            } else {
                w *= 1.0 / nrm;
            }
            if (lane < lead) q[lane + j * KM] = w;
            __syncwarp();
        }
        if (collapsed && lane == 0)
            if (atomicCAS(&a.st->err_code, 0, kErrOrth) == 0) a.st->err_iter = a.iter;
    }
    __syncthreads();
    if (a.mode == 1) {
        for (int i = threadIdx.x; i < k * b; i += blockDim.x) {
            const int r = i % k, j = i / k;
            double s = 0.0;
            for (int l = 0; l < lead; ++l) s += Vs[r + l * KM] * q[l + j * KM];
            mix[r + j * KM] = s;
            a.Cm[r + (b + j) * k] = s;
        }
    }
    __syncthreads();
    // 5. n-side products V' = T C, X' = T mix (dense.cpp:75-89 matmul); in
    //    one-pass mode the same combinations of the A^T A images Z
    const bool zmode = a.Z.p[0] != nullptr;
    for (int pass = 0; pass < (zmode ? 2 : 1); ++pass) {
        const Cols& src = pass == 0 ? a.T : a.Z;
        double* vo = pass == 0 ? a.Vout : a.ZVout;
        double* xo = pass == 0 ? a.Xout : a.ZXout;
        for (int64_t i = threadIdx.x; i < a.n; i += blockDim.x) {
            double t[KM];
#pragma unroll
            for (int l = 0; l < KM; ++l) t[l] = l < k ? src.p[l][i] : 0.0;
            for (int j = 0; j < b; ++j) {
                double v = 0.0, xv = 0.0;
#pragma unroll
                for (int l = 0; l < KM; ++l)
                    if (l < k) {
                        v = fma(Vs[l + (lead + j) * KM], t[l], v);
                        if (a.mode == 1) xv = fma(mix[l + j * KM], t[l], xv);
                    }
                vo[i + j * a.n] = v;
                if (a.mode == 1) xo[i + j * a.n] = xv;
            }
        }
    }
}

// m-side recurrence products without A: out[j][i] = sum_l T[l][i] Cm[l + j k]
// (solver.cpp:421, :462 -- AV' = AT C, AX' = AT mix).  K, Q are compile-time
// so the column pointers stay in registers; each thread handles kTcRows rows
// (stride blockDim) with all of their loads issued before the FMAs.
constexpr int kTcRows = 4;
template <int K, int Q>
__global__ void __launch_bounds__(256) tcombine_kernel(Cols T, const double* Cm, OutCols out, int64_t m) {
    __shared__ double Cs[K * Q];
    for (int i = threadIdx.x; i < K * Q; i += blockDim.x) Cs[i] = Cm[i];
    __syncthreads();
    const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x * kTcRows;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x * kTcRows + threadIdx.x; base < m;
         base += step) {
        double t[kTcRows][K];
#pragma unroll
        for (int u = 0; u < kTcRows; ++u) {
            const int64_t r = base + static_cast<int64_t>(u) * blockDim.x;
#pragma unroll
            for (int l = 0; l < K; ++l) t[u][l] = r < m ? __ldcs(T.p[l] + r) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kTcRows; ++u) {
            const int64_t r = base + static_cast<int64_t>(u) * blockDim.x;
            if (r < m) {
#pragma unroll
                for (int j = 0; j < Q; ++j) {
                    double y = 0.0;
#pragma unroll
                    for (int l = 0; l < K; ++l) y = fma(Cs[l + j * K], t[u][l], y);
                    out.p[j][r] = y;
                }
            }
        }
    }
}

// G = sum of per-CTA partials (fixed order); R = G - theta^2 V; partial norms.
// A block covers kRedCols columns with kRedGroups thread groups; group g sums
// partials g, g + kRedGroups, ... in order (all loads in flight together),
// and the group sums are added in fixed order.  Many small blocks, so the
// partials stream from L2 through many SMs at once.
constexpr int kRedCols = 64;
constexpr int kRedGroups = 16;
__global__ void __launch_bounds__(kRedCols * kRedGroups) reduce_g_kernel(const double* Gpart, int nparts, int64_t n,
                                                                         int b, const double* V, const DevState* st,
                                                                         int residual, double* Gout, double* nrm_part,
                                                                         const int* skip) {
    if (skip && *skip) return;
    __shared__ double part[kRedGroups][kRedCols];
    __shared__ double red[kRedCols / 32];
    const int j = blockIdx.y;
    const int t = threadIdx.x % kRedCols, grp = threadIdx.x / kRedCols;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kRedCols + t;
    double s = 0.0;
    if (i < n) {
#pragma unroll 16
        for (int p = grp; p < nparts; p += kRedGroups) s += Gpart[(static_cast<size_t>(p) * b + j) * n + i];
    }
    part[grp][t] = s;
    __syncthreads();
    if (grp != 0) return;
    double v = 0.0;
    if (i < n) {
        s = part[0][t];
#pragma unroll
        for (int g = 1; g < kRedGroups; ++g) s += part[g][t];
        if (residual) {
            const double th = st->theta[j];
            s -= (th * th) * V[i + j * n];
        }
        Gout[i + j * n] = s;
        v = s * s;
    }
    v = warp_sum(v);
    if ((t & 31) == 0) red[t >> 5] = v;
    named_sync(1, kRedCols);
    if (t == 0) {
        double tt = 0.0;
        for (int w = 0; w < kRedCols / 32; ++w) tt += red[w];
        nrm_part[j * gridDim.x + blockIdx.x] = tt;
    }
}

// one-pass check gate: the residual norm as control_kernel forms it, from the
// images' residual; far above the tolerance the stop test cannot pass, and
// the exact Gram pass is skipped
__global__ void gate_kernel(const double* nrm_part, int nblk, int b, DevState* st, double thresh) {
    if (threadIdx.x != 0) return;
    double best = 0.0;
    for (int j = 0; j < b; ++j) {
        double s = 0.0;
        for (int x = 0; x < nblk; ++x) s += nrm_part[j * nblk + x];
        best = fmax(best, sqrt(s));
    }
    st->skip_exact = best > thresh ? 1 : 0;
}

// the stop rule (solver.cpp:177-211) for loop counter i: flags = {tol_ok,
// resid_stalled, progress_stalled, stop}
__device__ void stop_rule(const double* rh, const double* th, int i, double sigma1, double tol, double factor,
                          int use_stag, int flags[4]) {
    const bool tol_ok = rh[i + 1] <= sigma1 * sigma1 * tol;
    bool rs = false, ps = false, stop = tol_ok;
    if (use_stag) {
        if (i >= 4) rs = factor * rh[i + 1] >= rh[i - 4];
        if (i >= 9) {
            const double dn = th[i] > 0.0 ? th[i] : 1.0;
            const double dt = th[i - 4] > 0.0 ? th[i - 4] : 1.0;
            const double recent = (th[i - 4] - th[i + 1]) / dn;
            const double earlier = (th[i - 9] - th[i - 4]) / dt;
            ps = factor * recent >= earlier;
        }
        stop = tol_ok && rs && ps;
    }
    flags[0] = tol_ok;
    flags[1] = rs;
    flags[2] = ps;
    flags[3] = stop;
}

__global__ void stop_rule_kernel(const double* rh, const double* th, int i, double sigma1, double tol,
                                 double factor, int use_stag, int* flags) {
    stop_rule(rh, th, i, sigma1, tol, factor, use_stag, flags);
}

// record row + stop rule (solver.cpp:376-397, :177-211)
__global__ void __launch_bounds__(256) control_kernel(ControlArgs a) {
    __shared__ double red[8];
    __shared__ double resid_s;
    if (threadIdx.x == 0) {
        double best = 0.0;
        for (int j = 0; j < a.b; ++j) {
            double s = 0.0;
            for (int x = 0; x < a.nblk; ++x) s += a.nrm_part[j * a.nblk + x];
            best = fmax(best, sqrt(s));
        }
        resid_s = best;
    }
    double c = 0.0;
    if (a.truth_v) {
        const double* vc = a.V + static_cast<int64_t>(a.b - 1) * a.n;
        for (int64_t i = threadIdx.x; i < a.n; i += blockDim.x) c += vc[i] * a.truth_v[i];
        c = warp_sum(c);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    DevState* st = a.st;
    msvd_record_row row;
    row.iter = a.row;
    row.pad_ = 0;
    row.matvecs_a = static_cast<int64_t>(a.b) * (a.row + 1);
    row.matvecs_at = static_cast<int64_t>(a.b) * (a.row + 1);
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    row.wall_ms = a.timing ? static_cast<double>(now - st->t0_ns) * 1e-6 : 0.0;
    row.theta = st->theta[a.b - 1];
    row.resid = resid_s;
    row.relerr = -1.0;
    row.sin_angle = -1.0;
    if (a.truth_v) {
        double cc = 0.0;
        for (int w = 0; w < 8; ++w) cc += red[w];
        cc = fmin(1.0, fmax(-1.0, cc));
        const double sn = a.truth_sigma;
        row.relerr = sn > 0.0 ? fabs(row.theta - sn) / sn : fabs(row.theta);
        row.sin_angle = sqrt(fmax(0.0, 1.0 - cc * cc));
    }
    a.rows[a.row] = row;
    a.rh[a.row] = resid_s;
    a.th[a.row] = st->theta[0];
    if (a.check == 2) {
        // early accept of a deferred check row (tolerance-only stop): the residual from the
        // carried images is within ~u sigma_1^2 of the exact one, so a value a factor four
        // under the threshold decides the test without the refresh pass
        st->stop = resid_s <= 0.25 * a.sigma1 * a.sigma1 * a.tol ? 1 : 0;
    } else if (a.check) {
        int f[4];
        stop_rule(a.rh, a.th, a.row - 1, a.sigma1, a.tol, a.factor, a.use_stag, f);
        st->stop = f[3];
    }
}

// ---------------------------------------------------------------------------
// preconditioner apply (precond.cpp:38-48): t = Vt^T r / sig^2, w = Vt t.
// Vt is held column-major (Vcol) and row-major (Vrow) so both passes are
// warp-per-vector coalesced dot products over an L2-resident n x n matrix.
// ---------------------------------------------------------------------------
template <int B>
__global__ void __launch_bounds__(128) dots_kernel(const double* __restrict__ M, int64_t n,
                                                   const double* __restrict__ X, const double* __restrict__ sig,
                                                   double* __restrict__ out, DevState* st, int iter,
                                                   int check_finite) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * 4 + warp;
    if (c >= n) return;
    const double* mc = M + c * n;
    double acc[B];
#pragma unroll
    for (int j = 0; j < B; ++j) acc[j] = 0.0;
    constexpr int U = 16;  // the L2 loads of 16 steps in flight together
    for (int64_t base = 0; base < n; base += 32 * U) {
        double mv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + u * 32 + lane;
            mv[u] = i < n ? mc[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + u * 32 + lane;
            if (i < n)
#pragma unroll
                for (int j = 0; j < B; ++j) acc[j] = fma(mv[u], X[i + j * n], acc[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < B; ++j) acc[j] = warp_sum(acc[j]);
    if (lane == 0) {
        bool finite = true;
#pragma unroll
        for (int j = 0; j < B; ++j) {
            double v = acc[j];
            if (sig) {
                const double s = sig[c];
                v /= s * s;
            }
            out[c + j * n] = v;
            finite = finite && isfinite(v);
        }
        if (check_finite && !finite)
            if (atomicCAS(&st->err_code, 0, kErrNonfiniteW) == 0) st->err_iter = iter;
    }
}

__global__ void diag_scale_kernel(int kind, const double* R, const double* dinv, int64_t n, int b, double* W,
                                  DevState* st, int iter) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * b) return;
    const double v = kind == MSVD_PRECOND_DIAGONAL ? R[i] * dinv[i % n] : R[i];
    W[i] = v;
    if (!isfinite(v))
        if (atomicCAS(&st->err_code, 0, kErrNonfiniteW) == 0) st->err_iter = iter;
}

// ---------------------------------------------------------------------------
// BCGS2 (solver.cpp:213-261), single CTA.  Each pass projects against all
// basis columns and all earlier W columns at once (one multi-dot per pass);
// degenerate columns are replaced from the solver's SplitMix64 Gaussian
// stream, generated counter-style so every thread draws its own entries.
// ---------------------------------------------------------------------------
constexpr int kCgsT = 512;

__device__ double gauss_at(uint64_t s, int have_spare, double spare, int64_t e) {
    int64_t idx = e;
    if (have_spare) {
        if (e == 0) return spare;
        idx = e - 1;
    }
    const int64_t pr = idx / 2;
    const uint64_t d1 = sm_mix(s + kGolden * static_cast<uint64_t>(2 * pr + 1));
    const uint64_t d2 = sm_mix(s + kGolden * static_cast<uint64_t>(2 * pr + 2));
    const double u1 = static_cast<double>((d1 >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>((d2 >> 11) + 1) * 0x1.0p-53;
    const double rad = sqrt(-2.0 * log(u1));
    const double ang = 6.283185307179586476925286766559 * u2;
    return (idx & 1) ? rad * sin(ang) : rad * cos(ang);
}

// block-wide sums of cnt (<= 32) per-thread values; result in out[0..cnt)
__device__ void block_multi_sum(double (&v)[32], int cnt, double* red, double* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double t = warp_transpose_reduce32(v);
    red[warp * 32 + lane] = t;
    __syncthreads();
    if (threadIdx.x < cnt) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w * 32 + threadIdx.x];
        out[threadIdx.x] = s;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kCgsT) cgs2_kernel(double* W, int64_t n, int b, Cols basis, int nb,
                                                     DevState* st, int iter) {
    __shared__ double red[32 * 32];
    __shared__ double sums[32];
    __shared__ double scale_ref;
    // scale_ref = max column norm of the incoming W (solver.cpp:217)
    {
        double v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
            for (int j = 0; j < kMaxB; ++j)
                if (j < b) v[j] += W[i + j * n] * W[i + j * n];
        block_multi_sum(v, b, red, sums);
        if (threadIdx.x == 0) {
            double best = 0.0;
            for (int j = 0; j < b; ++j) best = fmax(best, sqrt(sums[j]));
            scale_ref = best;
        }
        __syncthreads();
    }
    const double drop = static_cast<double>(n) * kEps * scale_ref;
    for (int j = 0; j < b; ++j) {
        double* x = W + j * n;
        const int cnt = nb + j;
        bool replaced = false;
        for (int attempt = -1; attempt < 8; ++attempt) {
            if (attempt >= 0) {
                // x = fresh Gaussian draws (rng.hpp:40-52 stream continued)
                const uint64_t s0 = st->rng_state;
                const int hs = st->have_spare;
                const double sp = st->spare;
                for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = gauss_at(s0, hs, sp, i);
                __syncthreads();
                if (threadIdx.x == 0) {
                    const int64_t fresh = hs ? n - 1 : n;
                    const int64_t pairs = (fresh + 1) / 2;
                    if (fresh & 1) {
                        st->spare = gauss_at(s0, 0, 0.0, 2 * pairs - 1);
                        st->have_spare = 1;
                    } else {
                        st->have_spare = 0;
                    }
                    st->rng_state = s0 + kGolden * static_cast<uint64_t>(2 * pairs);
                }
            }
            for (int pass = 0; pass < 2; ++pass) {
                double v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = 0.0;
                for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
                    const double xi = x[i];
#pragma unroll
                    for (int l = 0; l < 2 * kMaxB + kMaxB; ++l) {
                        if (l < cnt) {
                            const double cl = l < nb ? basis.p[l][i] : W[i + (l - nb) * n];
                            v[l] = fma(cl, xi, v[l]);
                        }
                    }
                }
                block_multi_sum(v, cnt, red, sums);
                for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
                    double xi = x[i];
                    for (int l = 0; l < cnt; ++l) {
                        const double cl = l < nb ? basis.p[l][i] : W[i + (l - nb) * n];
                        xi -= sums[l] * cl;
                    }
                    x[i] = xi;
                }
                __syncthreads();
            }
            double v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.0;
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v[0] += x[i] * x[i];
            block_multi_sum(v, 1, red, sums);
            const double nrm = sqrt(sums[0]);
            const bool accept = attempt < 0 ? nrm > drop : nrm > 1e-3 * sqrt(static_cast<double>(n));
            if (accept) {
                const double inv = 1.0 / nrm;
                for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] *= inv;
                __syncthreads();
                if (attempt >= 0) replaced = true;
                break;
            }
            if (attempt == 7) {
                if (threadIdx.x == 0)
                    if (atomicCAS(&st->err_code, 0, kErrCgs2) == 0) st->err_iter = iter;
                return;
            }
        }
        if (replaced && threadIdx.x == 0) st->replacements += 1;
        __syncthreads();
    }
}

__global__ void state_init_kernel(DevState* st, uint64_t seed) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    st->stop = 0;
    st->err_code = 0;
    st->err_iter = -1;
    st->have_spare = 0;
    st->rng_state = sm_keyed_state(seed, 0x9e3779b97f4a7c15ULL);  // solver.cpp:342
    st->spare = 0.0;
    st->replacements = 0;
    st->t0_ns = now;
    st->max_drift = 0.0;
    st->worst_jacobi = 0.0;
    for (int j = 0; j < kMaxB; ++j) st->theta[j] = 0.0;
    st->snap_err_code = 0;
    st->snap_err_iter = -1;
    st->snap_replacements = 0;
}

__global__ void snapshot_kernel(DevState* st) {
    st->snap_err_code = st->err_code;
    st->snap_err_iter = st->err_iter;
    st->snap_replacements = st->replacements;
}

__global__ void drift_kernel(const double* fresh, const double* cached, int64_t count, DevState* st) {
    double v = 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v = fmax(v, fabs(fresh[i] - cached[i]));
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0) atomic_max_pos(&st->max_drift, v);
}

__global__ void drift_check_kernel(DevState* st, double limit, int iter) {
    if (st->max_drift > limit)
        if (atomicCAS(&st->err_code, 0, kErrDrift) == 0) st->err_iter = iter;
}

// column sums of squares of a row-major A: per-CTA partials then a fixed-order sum
__global__ void colsq_kernel(const double* A, int64_t m, int n, int64_t ld, double* part) {
    const int64_t r0 = (m * blockIdx.y) / gridDim.y, r1 = (m * (blockIdx.y + 1)) / gridDim.y;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    double s = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
        const double v = A[r * ld + c];
        s += v * v;
    }
    part[static_cast<int64_t>(blockIdx.y) * n + c] = s;
}
__global__ void colsq_finish_kernel(const double* part, int np, int n, double* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    double s = 0.0;
    for (int p = 0; p < np; ++p) s += part[static_cast<int64_t>(p) * n + c];
    out[c] = s;
}

__global__ void transpose_kernel(const double* A, int64_t m, int64_t n, int64_t ld, double* out) {
    __shared__ double tile[32][33];
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (r < m && c < n) ? A[r * ld + c] : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < m && c < n) out[c * m + r] = tile[threadIdx.x][i];
    }
}

__global__ void copy_cols_kernel(const double* src, int64_t ld, int64_t col0, int64_t rows, int64_t cols,
                                 double* dst) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows * cols) return;
    const int64_t r = i % rows, c = i / rows;
    dst[i] = src[r + (col0 + c) * ld];
}

template <int KM>
__global__ void __launch_bounds__(512) small_svd_kernel(const double* B, int k, double* sigma, double* Vout,
                                                         DevState* st) {
    __shared__ double Bm[KM * KM], V[KM * KM], Vs[KM * KM], sig[KM], worst[2];
    __shared__ int ord[KM];
    for (int i = threadIdx.x; i < KM * KM; i += blockDim.x) {
        const int r = i % KM, c = i / KM;
        Bm[i] = (r < k && c < k) ? B[r + c * k] : 0.0;
    }
    __syncthreads();
    const bool ok = jacobi_svd<KM>(Bm, V, k, sig, Vs, ord, worst);
    if (!ok && threadIdx.x == 0) st->err_code = kErrJacobi;
    if (threadIdx.x == 0) st->worst_jacobi = worst[1];
    if (threadIdx.x < k) sigma[threadIdx.x] = sig[threadIdx.x];
    for (int i = threadIdx.x; i < k * k; i += blockDim.x) Vout[i] = Vs[(i % k) + (i / k) * KM];
}

template <int KM>
size_t rr_smem() {
    return sizeof(double) * rr_base_words<KM>() + 64;
}

int km_for(int k) {
    if (k <= 4) return 4;
    if (k <= 8) return 8;
    if (k <= 16) return 16;
    if (k <= 24) return 24;
    fail(MSVD_ERR_DIMENSION, "msvd: trial width above 24 is not supported");
}

template <int KM>
void rr_launch(Ctx& c, const RRArgs& a) {
    size_t sm = rr_smem<KM>();
    const size_t stacked = sizeof(double) * (static_cast<size_t>(a.nparts) * a.k * (KM + 1) + 2 * 17 * (KM + 1));
    if (KM <= 8 && sm + stacked <= c.smem_optin) sm += stacked;  // room for the stacked-QR merge
    if (KM == 16) sm = c.smem_optin;                             // the stacked merge in groups of parts
    optin_smem(c, rr_kernel<KM>);
    rr_kernel<KM><<<1, 512, sm, c.stream>>>(a);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

}  // namespace

int tsqr_parts(const Ctx& c) { return c.num_sms; }

void launch_tsqr(Ctx& c, Cols T, int64_t m, int k, double* Rparts, DevState* st, int iter, const int* skip) {
    ProfScope prof(c, kProfTsqr);
    TsqrArgs a{T, m, k, Rparts, st, iter, skip};
    const int grid = tsqr_parts(c);
    auto smem_launch = [&](auto kernel, int km) {
        const size_t sm = sizeof(double) * 16 * (km * km + 32 * (km + 1));
        optin_smem(c, kernel);
        kernel<<<grid, 512, sm, c.stream>>>(a);
    };
    const bool stacked = !std::getenv("MSVD_TSQR_FOLD");
    switch (km_for(k)) {
        case 4:
            if (stacked) tsqr_stacked_kernel<4, 8><<<grid, 512, 0, c.stream>>>(a);
            else tsqr_kernel<4><<<grid, 256, 0, c.stream>>>(a);
            break;
        case 8:
            if (stacked) tsqr_stacked_kernel<8, 4><<<grid, 512, 0, c.stream>>>(a);
            else smem_launch(tsqr_smem_kernel<8>, 8);
            break;
        case 16: smem_launch(tsqr_smem_kernel<16>, 16); break;
        default: smem_launch(tsqr_smem_kernel<24>, 24); break;
    }
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    c.paths |= kPathTsqr;
}

template <int B>
static void tcombine_b(Ctx& c, Cols T, int k, const double* Cm, int q, OutCols out, int64_t m, unsigned grid) {
    if (k == 2 * B && q == 2 * B) tcombine_kernel<2 * B, 2 * B><<<grid, 256, 0, c.stream>>>(T, Cm, out, m);
    else if (k == 3 * B && q == 2 * B) tcombine_kernel<3 * B, 2 * B><<<grid, 256, 0, c.stream>>>(T, Cm, out, m);
    else if (k == B && q == B) tcombine_kernel<B, B><<<grid, 256, 0, c.stream>>>(T, Cm, out, m);
    else fail(MSVD_ERR_INVALID, "msvd: unsupported recurrence-product shape");
}

void launch_tcombine(Ctx& c, Cols T, int k, const double* Cm, int q, OutCols out, int64_t m) {
    if (m == 0) return;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(m, 256 * kTcRows), 16 * c.num_sms));
    const int b = q == k ? q : q / 2;  // (k, q) = (b, b), (2b, 2b) or (3b, 2b)
    switch (b) {
        case 1: tcombine_b<1>(c, T, k, Cm, q, out, m, grid); break;
        case 2: tcombine_b<2>(c, T, k, Cm, q, out, m, grid); break;
        case 3: tcombine_b<3>(c, T, k, Cm, q, out, m, grid); break;
        case 4: tcombine_b<4>(c, T, k, Cm, q, out, m, grid); break;
        case 5: tcombine_b<5>(c, T, k, Cm, q, out, m, grid); break;
        case 6: tcombine_b<6>(c, T, k, Cm, q, out, m, grid); break;
        case 7: tcombine_b<7>(c, T, k, Cm, q, out, m, grid); break;
        case 8: tcombine_b<8>(c, T, k, Cm, q, out, m, grid); break;
        default: fail(MSVD_ERR_INVALID, "msvd: unsupported recurrence-product shape");
    }
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_rr(Ctx& c, const RRArgs& a) {
    ProfScope prof(c, kProfRR);
    switch (km_for(a.k)) {
        case 4: rr_launch<4>(c, a); break;
        case 8: rr_launch<8>(c, a); break;
        case 16: rr_launch<16>(c, a); break;
        default: rr_launch<24>(c, a); break;
    }
}

void launch_small_svd(Ctx& c, const double* B, int k, double* sigma, double* V, DevState* st) {
    switch (km_for(k)) {
        case 4: small_svd_kernel<4><<<1, 512, 0, c.stream>>>(B, k, sigma, V, st); break;
        case 8: small_svd_kernel<8><<<1, 512, 0, c.stream>>>(B, k, sigma, V, st); break;
        case 16: small_svd_kernel<16><<<1, 512, 0, c.stream>>>(B, k, sigma, V, st); break;
        default: small_svd_kernel<24><<<1, 512, 0, c.stream>>>(B, k, sigma, V, st); break;
    }
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_reduce_g(Ctx& c, const double* Gpart, int nparts, int64_t n, int b, const double* V,
                     const DevState* st, int residual, double* Gout, double* nrm_part, int nblk,
                     const int* skip) {
    ProfScope prof(c, kProfReduce);
    dim3 grid(static_cast<unsigned>(nblk), static_cast<unsigned>(b));
    reduce_g_kernel<<<grid, kRedCols * kRedGroups, 0, c.stream>>>(Gpart, nparts, n, b, V, st, residual, Gout,
                                                                   nrm_part, skip);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_gate(Ctx& c, const double* nrm_part, int nblk, int b, DevState* st, double thresh) {
    ProfScope prof(c, kProfControl);
    gate_kernel<<<1, 32, 0, c.stream>>>(nrm_part, nblk, b, st, thresh);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_control(Ctx& c, const ControlArgs& a) {
    ProfScope prof(c, kProfControl);
    control_kernel<<<1, 256, 0, c.stream>>>(a);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

template <int B>
static void precond_b(Ctx& c, const double* Vcol, const double* Vrow, const double* sig, int64_t n,
                      const double* R, double* tmp, double* W, DevState* st, int iter) {
    const unsigned grid = static_cast<unsigned>(ceil_div(n, 4));
    dots_kernel<B><<<grid, 128, 0, c.stream>>>(Vcol, n, R, sig, tmp, st, iter, 0);
    dots_kernel<B><<<grid, 128, 0, c.stream>>>(Vrow, n, tmp, nullptr, W, st, iter, 1);
    MSVD_CUDA(cudaGetLastError());
    c.launches += 2;
}

void launch_precond(Ctx& c, int kind, const double* Vcol, const double* Vrow, const double* sig,
                    const double* dinv, int64_t n, const double* R, int b, double* tmp, double* W,
                    DevState* st, int iter) {
    ProfScope prof(c, kProfPrecond);
    if (kind != MSVD_PRECOND_RANDOMIZED) {
        const int64_t tot = n * b;
        diag_scale_kernel<<<static_cast<unsigned>(ceil_div(tot, 256)), 256, 0, c.stream>>>(kind, R, dinv, n, b, W,
                                                                                           st, iter);
        MSVD_CUDA(cudaGetLastError());
        ++c.launches;
        return;
    }
    switch (b) {
        case 1: precond_b<1>(c, Vcol, Vrow, sig, n, R, tmp, W, st, iter); break;
        case 2: precond_b<2>(c, Vcol, Vrow, sig, n, R, tmp, W, st, iter); break;
        case 3: precond_b<3>(c, Vcol, Vrow, sig, n, R, tmp, W, st, iter); break;
        case 4: precond_b<4>(c, Vcol, Vrow, sig, n, R, tmp, W, st, iter); break;
        case 5: precond_b<5>(c, Vcol, Vrow, sig, n, R, tmp, W, st, iter); break;
        case 6: precond_b<6>(c, Vcol, Vrow, sig, n, R, tmp, W, st, iter); break;
        case 7: precond_b<7>(c, Vcol, Vrow, sig, n, R, tmp, W, st, iter); break;
        default: precond_b<8>(c, Vcol, Vrow, sig, n, R, tmp, W, st, iter); break;
    }
}

void launch_cgs2(Ctx& c, double* W, int64_t n, int b, Cols basis, int nb, DevState* st, int iter) {
    ProfScope prof(c, kProfCgs2);
    cgs2_kernel<<<1, kCgsT, 0, c.stream>>>(W, n, b, basis, nb, st, iter);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_state_init(Ctx& c, DevState* st, uint64_t seed) {
    state_init_kernel<<<1, 1, 0, c.stream>>>(st, seed);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_stop_rule(Ctx& c, const double* rh, const double* th, int i, double sigma1, double tol, double factor,
                      int use_stag, int* flags) {
    stop_rule_kernel<<<1, 1, 0, c.stream>>>(rh, th, i, sigma1, tol, factor, use_stag, flags);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_snapshot(Ctx& c, DevState* st) {
    snapshot_kernel<<<1, 1, 0, c.stream>>>(st);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_drift(Ctx& c, const double* fresh, const double* cached, int64_t count, DevState* st, double limit,
                  int iter) {
    drift_kernel<<<c.num_sms * 2, 256, 0, c.stream>>>(fresh, cached, count, st);
    drift_check_kernel<<<1, 1, 0, c.stream>>>(st, limit, iter);
    MSVD_CUDA(cudaGetLastError());
    c.launches += 2;
}

void launch_colnorms(Ctx& c, const StreamGeom& g, double* part, double* out) {
    const int np = c.num_sms;
    dim3 grid(static_cast<unsigned>(ceil_div(g.n, 256)), static_cast<unsigned>(np));
    colsq_kernel<<<grid, 256, 0, c.stream>>>(g.A, g.m, g.n, g.ld, part);
    colsq_finish_kernel<<<static_cast<unsigned>(ceil_div(g.n, 256)), 256, 0, c.stream>>>(part, np, g.n, out);
    MSVD_CUDA(cudaGetLastError());
    c.launches += 2;
}

void launch_transpose_rm_to_cm(Ctx& c, const double* A, int64_t m, int64_t n, int64_t ld, double* out) {
    dim3 grid(static_cast<unsigned>(ceil_div(n, 32)), static_cast<unsigned>(ceil_div(m, 32)));
    transpose_kernel<<<grid, dim3(32, 8), 0, c.stream>>>(A, m, n, ld, out);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void launch_copy_cols(Ctx& c, const double* src, int64_t ld_src, int64_t col0, int64_t rows, int64_t cols,
                      double* dst) {
    const int64_t tot = rows * cols;
    if (tot == 0) return;
    copy_cols_kernel<<<static_cast<unsigned>(ceil_div(tot, 256)), 256, 0, c.stream>>>(src, ld_src, col0, rows, cols,
                                                                                      dst);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

}  // namespace msvd
