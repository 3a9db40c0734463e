// Cholesky QR2 of the m x k trial block [AV AX AW] (solver.cpp:412-417).
//
// The Rayleigh-Ritz step needs the R factor of the tall trial block
// (svd.cpp:21-55 Householder QR; then the Jacobi SVD of R).  For b >= 2 the
// separate Householder TSQR pass (a 48 MB block at C4, k = 12) ran at
// ~0.2 TB/s and its 148-part stacked merge took another ~0.2 ms per
// iteration.  Cholesky QR2 gives the same R (backward stable, positive
// diagonal -- the SVD's right vectors do not depend on R's row signs) while
// kappa(AT) < ~1e7: two streaming Gram passes over the block,
//   G1 = AT^T AT,              R1 = chol(G1)
//   G2 = (AT R1^-1)^T (AT R1^-1), R2 = chol(G2),   R = R2 R1,
// each a fixed-order per-CTA partial sum (deterministic), and two k x k
// Choleskys in one warp.  A device flag records whether both Choleskys
// succeeded with diag(R1) within 1e6 of each other; where not, the TSQR
// kernels (launched after, reading the flag) run and the RR step merges their
// parts as before -- no host round trip either way.
#include "common.cuh"
#include "msvd_internal.h"

namespace msvd {
namespace {

constexpr int kGramT = 128;    // threads per CTA (4 warps; static shared memory)
constexpr int kGramW = kGramT / 32;
constexpr int kGramRegT = 512;  // block_gram_reg_kernel: 16 warps, one CTA per SM -> num_sms parts
constexpr int kGramRegW = kGramRegT / 32;
constexpr int kMaxEnt = (kMaxK * (kMaxK + 1) / 2 + 31) / 32;  // Gram entries per lane (<= 10)
constexpr int kCholT = 512;    // chol_small_kernel threads

// Gpart[cta] (k x k, col-major, full) = sum over the CTA's rows of t t^T with
// t = the row of T (times Rinv, upper k x k, when given).  Each warp streams
// its own contiguous rows in 32-row tiles with no CTA barrier: lane = row for
// the loads (coalesced per column) and the R^-1 transform, then the tile goes
// through the warp's shared-memory slot and lane e sums the Gram entries e,
// e + 32, ... over the tile's rows; the 4 warp partials are added in warp
// order at the end (deterministic).  Four CTAs per SM.
__global__ void __launch_bounds__(kGramT) block_gram_kernel(Cols T, int64_t m, int k, const double* Rinv,
                                                           double* Gpart, const int* disabled) {
    if (*disabled) return;
    __shared__ double tile[kGramW][32][kMaxK + 1];
    __shared__ double ri[kMaxK * kMaxK];
    __shared__ double wsum[kGramW][kMaxK * (kMaxK + 1) / 2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (Rinv)
        for (int i = threadIdx.x; i < k * k; i += blockDim.x) ri[i] = Rinv[i];
    __syncthreads();
    const int64_t gw = static_cast<int64_t>(blockIdx.x) * kGramW + warp, nw = static_cast<int64_t>(gridDim.x) * kGramW;
    const int64_t r0 = (m * gw) / nw, r1 = (m * (gw + 1)) / nw;
    const int ne = k * (k + 1) / 2;
    int ep[kMaxEnt], eq[kMaxEnt];
#pragma unroll
    for (int s = 0; s < kMaxEnt; ++s) {
        const int e = lane + 32 * s;
        int q = 0, base = 0;
        if (e < ne)
            while (base + q + 1 <= e) {  // column q holds entries base .. base + q
                base += q + 1;
                ++q;
            }
        ep[s] = e < ne ? e - base : 0;
        eq[s] = e < ne ? q : 0;
    }
    double acc[kMaxEnt];
#pragma unroll
    for (int s = 0; s < kMaxEnt; ++s) acc[s] = 0.0;
    double(*tl)[kMaxK + 1] = tile[warp];
    for (int64_t base = r0; base < r1; base += 32) {
        const int64_t r = base + lane;
        double t[kMaxK];
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) t[j] = (j < k && r < r1) ? T.p[j][r] : 0.0;
        if (Rinv) {
#pragma unroll
            for (int j = kMaxK - 1; j >= 0; --j) {  // t <- t R^-1 (upper): column j uses t[0..j]
                if (j >= k) continue;
                double sj = 0.0;
#pragma unroll
                for (int l = 0; l <= j; ++l) sj += t[l] * ri[l + j * k];
                t[j] = sj;
            }
        }
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
            if (j < k) tl[lane][j] = t[j];
        __syncwarp();
#pragma unroll
        for (int s = 0; s < kMaxEnt; ++s) {
            if (lane + 32 * s >= ne) break;
            double a = acc[s];
            for (int rr = 0; rr < 32; ++rr) a += tl[rr][ep[s]] * tl[rr][eq[s]];
            acc[s] = a;
        }
        __syncwarp();
    }
#pragma unroll
    for (int s = 0; s < kMaxEnt; ++s)
        if (lane + 32 * s < ne) wsum[warp][lane + 32 * s] = acc[s];
    __syncthreads();
    double* G = Gpart + static_cast<size_t>(blockIdx.x) * k * k;
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
        double v = wsum[0][e];
        for (int w = 1; w < kGramW; ++w) v += wsum[w][e];
        int q = 0, base = 0;
        while (base + q + 1 <= e) {
            base += q + 1;
            ++q;
        }
        const int p0 = e - base;
        G[p0 + q * k] = v;
        G[q + p0 * k] = v;
    }
}

// Register form of the block Gram for k <= 12 (b <= 4): lane = row; the row's k values are
// transformed by R^-1 in registers and its outer product t t^T goes into k (k + 1) / 2
// per-thread accumulators -- no shared-memory tile, no per-entry row loops (the kernel
// above spends two shared loads per multiply-add and ran at ~1 TB/s).  The lanes' sums are
// reduced once at the end: a fixed butterfly per entry, the 4 warps in order (deterministic).
// K > 8: the k (k + 1) / 2 accumulators do not fit one thread (78 doubles at k = 12), so the
// warp takes 16 rows at a time and its two half-warps own the entries of columns
// [0, KH) and [KH, K) of the same rows (both halves load and transform the same 16 rows:
// the same addresses, one transaction).
template <int K>
__global__ void __launch_bounds__(kGramRegT) block_gram_reg_kernel(Cols T, int64_t m, const double* Rinv, double* Gpart,
                                                               const int* disabled) {
    if (*disabled) return;
    constexpr int NE = K * (K + 1) / 2;
    constexpr bool kHalves = K > 8;
    constexpr int KH = kHalves ? (K * 7 + 9) / 10 : K;     // columns [0, KH) hold about half the entries
    constexpr int NE0 = KH * (KH + 1) / 2;                  // entries of the first half
    constexpr int NA = kHalves ? (NE0 > NE - NE0 ? NE0 : NE - NE0) : NE;  // accumulators per thread
    constexpr int ROWS = kHalves ? 16 : 32;
    __shared__ double ri[K * K];
    __shared__ double wsum[kGramRegW][NE];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (Rinv)
        for (int i = threadIdx.x; i < K * K; i += blockDim.x) ri[i] = Rinv[i];
    __syncthreads();
    const int64_t gw = static_cast<int64_t>(blockIdx.x) * kGramRegW + warp, nw = static_cast<int64_t>(gridDim.x) * kGramRegW;
    const int64_t r0 = (m * gw) / nw, r1 = (m * (gw + 1)) / nw;
    const bool upper = kHalves && lane >= 16;
    // (volatile: R^-1 is re-read from shared memory per tile; hoisted into registers its
    // k (k + 1) / 2 entries would crowd out the accumulators)
    const volatile double* riv = ri;
    double acc[NA];
#pragma unroll
    for (int e = 0; e < NA; ++e) acc[e] = 0.0;
#pragma unroll 1
    for (int64_t base = r0; base < r1; base += ROWS) {
        const int64_t r = base + (lane & (ROWS - 1));
        double t[K];
#pragma unroll
        for (int j = 0; j < K; ++j) t[j] = r < r1 ? T.p[j][r] : 0.0;
        if (Rinv) {
#pragma unroll
            for (int j = K - 1; j >= 0; --j) {  // t <- t R^-1 (upper): column j uses t[0..j]
                double sj = 0.0;
#pragma unroll
                for (int l = 0; l <= j; ++l) sj += t[l] * riv[l + j * K];
                t[j] = sj;
            }
        }
        if (!upper) {
#pragma unroll
            for (int q = 0; q < KH; ++q)
#pragma unroll
                for (int pp = 0; pp <= q; ++pp) acc[q * (q + 1) / 2 + pp] = fma(t[pp], t[q], acc[q * (q + 1) / 2 + pp]);
        } else {
#pragma unroll
            for (int q = KH; q < K; ++q)
#pragma unroll
                for (int pp = 0; pp <= q; ++pp)
                    acc[q * (q + 1) / 2 + pp - NE0] = fma(t[pp], t[q], acc[q * (q + 1) / 2 + pp - NE0]);
        }
    }
    // lanes' sums: a fixed butterfly within each 16- or 32-lane owner set
#pragma unroll
    for (int e = 0; e < NA; ++e) {
        double v = acc[e];
#pragma unroll
        for (int o = ROWS / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if (!kHalves) {
            if (lane == 0) wsum[warp][e] = v;
        } else {
            if (lane == 0 && e < NE0) wsum[warp][e] = v;
            if (lane == 16 && e < NE - NE0) wsum[warp][NE0 + e] = v;
        }
    }
    __syncthreads();
    double* G = Gpart + static_cast<size_t>(blockIdx.x) * K * K;
    for (int e = threadIdx.x; e < NE; e += blockDim.x) {
        double v = wsum[0][e];
        for (int w = 1; w < kGramRegW; ++w) v += wsum[w][e];
        int q = 0, base = 0;
        while (base + q + 1 <= e) {  // column q holds entries base .. base + q
            base += q + 1;
            ++q;
        }
        const int p0 = e - base;
        G[p0 + q * K] = v;
        G[q + p0 * K] = v;
    }
}

// R = chol(G) upper (warp 0, lane = column), Rinv = R^-1 (thread = column, back
// substitution through shared memory); pass 2 also R_final = R Rprev.  flag: pass 1
// writes success (pivots finite and positive, diag(R) within 1e6); pass 2 ands its own.
__device__ void chol_tail(double* G, double* R, double* X, int* ok_sp, int k, double* Rout, double* Rinv,
                          const double* Rprev, double* Rfinal, int* flag, int pass, int* disabled) {
    int& ok_s = *ok_sp;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        // lane l owns column l of R (rows 0..l)
        double col[kMaxK];
#pragma unroll
        for (int i = 0; i < kMaxK; ++i) col[i] = 0.0;
        bool ok = true;
        double dmax = 0.0, dmin = 1e300;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) {
            if (j >= k) break;
            double d = 0.0;
            if (lane == j) {
                double s = G[j + j * k];
#pragma unroll
                for (int i = 0; i < kMaxK; ++i)
                    if (i < j) s -= col[i] * col[i];
                d = s > 0.0 ? sqrt(s) : 0.0;
                col[j] = d;
            }
            d = __shfl_sync(0xffffffffu, d, j);
            if (!(d > 0.0) || !isfinite(d)) ok = false;
            dmax = fmax(dmax, d);
            dmin = fmin(dmin, d);
            // R(j, l) for l > j: (G(j, l) - sum_i<j R(i, j) R(i, l)) / d
            double s = (lane > j && lane < k) ? G[j + lane * k] : 0.0;
#pragma unroll
            for (int i = 0; i < kMaxK; ++i) {
                if (i >= j) break;
                const double rij = __shfl_sync(0xffffffffu, col[i], j);
                s -= rij * col[i];
            }
            if (lane > j && lane < k) col[j] = d > 0.0 ? s / d : 0.0;
        }
        if (dmin < 1e-6 * dmax) ok = false;
        if (lane < k)
#pragma unroll
            for (int i = 0; i < kMaxK; ++i)
                if (i < k) R[i + lane * k] = (ok ? (i <= lane ? col[i] : 0.0) : (i == lane ? 1.0 : 0.0));
        if (lane == 0) ok_s = ok ? 1 : 0;  // not ok: identity factors keep everything finite
    }
    __syncthreads();
    if (Rout)
        for (int e = threadIdx.x; e < k * k; e += blockDim.x) Rout[e] = R[e];
    // Rinv column c = threadIdx.x: back substitution R x = e_c, x kept in X (shared)
    if (threadIdx.x < k) {
        const int cidx = threadIdx.x;
        for (int i = k - 1; i >= 0; --i) {
            double s = (i == cidx) ? 1.0 : 0.0;
            if (i <= cidx)
                for (int l = i + 1; l <= cidx; ++l) s -= R[i + l * k] * X[l + cidx * k];
            X[i + cidx * k] = i <= cidx ? s / R[i + i * k] : 0.0;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) Rinv[e] = X[e];
    if (pass == 2)  // R_final = R Rprev (both upper)
        for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
            const int i = e % k, c = e / k;
            double s = 0.0;
            for (int l = i; l <= c; ++l) s += R[i + l * k] * Rprev[l + c * k];
            Rfinal[e] = i <= c ? s : 0.0;
        }
    if (threadIdx.x == 0) {
        *flag = pass == 1 ? ok_s : ((*flag && ok_s) ? 1 : 0);
        // sticky: once a trial block needs the TSQR, the later ones (whose
        // conditioning only grows as the iteration converges) skip straight to it
        if (pass == 2 && !*flag) *disabled = 1;
    }
}

// G = sum of the parts (fixed order, below), R = chol(G)
// upper (warp 0, lane = column), Rinv = R^-1 (lane = column, back
// substitution through shared memory); pass 2 also R_final = R Rprev.
// flag: pass 1 writes success (pivots finite and positive, diag(R) within
// 1e6); pass 2 ands its own.
__global__ void __launch_bounds__(kCholT) chol_small_kernel(const double* Gpart, int nparts, int k, double* Rout,
                                                            double* Rinv, const double* Rprev, double* Rfinal,
                                                            int* flag, int pass, int* disabled) {
    if (*disabled) {  // an earlier iteration's block was too ill-conditioned: TSQR from here on
        if (threadIdx.x == 0) *flag = 0;
        return;
    }
    __shared__ double G[kMaxK * kMaxK];
    __shared__ double R[kMaxK * kMaxK];
    __shared__ double X[kMaxK * kMaxK];
    __shared__ int ok_s;
    // G = sum of the parts (fixed order): entry e is summed by NG threads, thread g
    // taking parts g, g + NG, ... with eight independent loads in flight, then the NG
    // partial sums in order -- deterministic, and a few dependent load rounds instead of
    // nparts / 32 per entry (26 us of the kernel's 46 at 592 parts)
    {
        __shared__ double part[kCholT];
        const int ne = k * (k + 1) / 2;
        const size_t kk = static_cast<size_t>(k) * k;
        const int NG = max(1, static_cast<int>(blockDim.x) / ne);
        const int e = threadIdx.x / NG, g = threadIdx.x % NG;
        int pq0 = 0, pq1 = 0;
        double sum = 0.0;
        if (e < ne) {
            int q = 0, base = 0;
            while (base + q + 1 <= e) {  // column q holds entries base .. base + q
                base += q + 1;
                ++q;
            }
            pq0 = e - base;
            pq1 = q;
            const double* Ge = Gpart + pq0 + static_cast<size_t>(pq1) * k;
            double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            int p = g;
            for (; p + 7 * NG < nparts; p += 8 * NG) {
#pragma unroll
                for (int u = 0; u < 8; ++u) a[u] += Ge[static_cast<size_t>(p + u * NG) * kk];
            }
            for (; p < nparts; p += NG) a[0] += Ge[static_cast<size_t>(p) * kk];
            sum = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
        }
        part[threadIdx.x] = sum;
        __syncthreads();
        if (e < ne && g == 0) {
            double t = part[threadIdx.x];
            for (int u = 1; u < NG; ++u) t += part[threadIdx.x + u];
            G[pq0 + pq1 * k] = t;
            G[pq1 + pq0 * k] = t;
        }
    }
    chol_tail(G, R, X, &ok_s, k, Rout, Rinv, Rprev, Rfinal, flag, pass, disabled);
}

// Pass 1 without a pass over the block: in one-pass mode the solver carries the images
// Z = A^T A [V X W] next to S = [V X W], and T^T T = S^T (A^T A S) = S^T Z -- k (k + 1) / 2
// dot products of length n instead of a sweep of the m x k block.  The block's columns are
// recurrence products (AV' = T C next to V' = S C), so S^T Z equals T^T T to the
// recurrences' rounding; it only has to make T R1^-1 well conditioned: pass 2 measures
// (T R1^-1)^T (T R1^-1) from the block itself.  A warp per entry (i <= j): lanes stride the
// n entries, fixed butterfly -- deterministic.
__global__ void __launch_bounds__(kCholT) image_chol_kernel(Cols S, Cols Z, int64_t n, int k, double* Rout,
                                                            double* Rinv, int* flag, int* disabled) {
    if (*disabled) {
        if (threadIdx.x == 0) *flag = 0;
        return;
    }
    __shared__ double G[kMaxK * kMaxK];
    __shared__ double R[kMaxK * kMaxK];
    __shared__ double X[kMaxK * kMaxK];
    __shared__ int ok_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int ne = k * (k + 1) / 2;
    for (int e = warp; e < ne; e += nw) {
        int q = 0, base = 0;
        while (base + q + 1 <= e) {  // column q holds entries base .. base + q
            base += q + 1;
            ++q;
        }
        const int pi = e - base;
        const double* sp = S.p[pi];
        const double* zq = Z.p[q];
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // eight loads in flight per lane
        int64_t i = lane;
        for (; i + 96 < n; i += 128) {
            a0 = fma(sp[i], zq[i], a0);
            a1 = fma(sp[i + 32], zq[i + 32], a1);
            a2 = fma(sp[i + 64], zq[i + 64], a2);
            a3 = fma(sp[i + 96], zq[i + 96], a3);
        }
        for (; i < n; i += 32) a0 = fma(sp[i], zq[i], a0);
        const double t = warp_sum((a0 + a1) + (a2 + a3));
        if (lane == 0) {
            G[pi + q * k] = t;
            G[q + pi * k] = t;
        }
    }
    chol_tail(G, R, X, &ok_s, k, Rout, Rinv, nullptr, nullptr, flag, 1, disabled);
}

}  // namespace

void launch_trial_cholqr(Ctx& c, Cols T, int64_t m, int k, TrialQr& q, const Cols* S, const Cols* Z, int64_t n) {
    ProfScope prof(c, kProfTsqr);
    const unsigned grid = static_cast<unsigned>(c.num_sms) * 4;
    // the block's Gram (of T Rinv when given): register form for the trial widths of b <= 4
    const unsigned rgrid = static_cast<unsigned>(c.num_sms);
    const bool reg = k == 2 || k == 3 || k == 4 || k == 6 || k == 8 || k == 9 || k == 12;
    const int parts = static_cast<int>(reg ? rgrid : grid);
    auto gram = [&](const double* Rinv) {
        switch (k) {
            case 2: block_gram_reg_kernel<2><<<rgrid, kGramRegT, 0, c.stream>>>(T, m, Rinv, q.gpart, q.disabled); break;
            case 3: block_gram_reg_kernel<3><<<rgrid, kGramRegT, 0, c.stream>>>(T, m, Rinv, q.gpart, q.disabled); break;
            case 4: block_gram_reg_kernel<4><<<rgrid, kGramRegT, 0, c.stream>>>(T, m, Rinv, q.gpart, q.disabled); break;
            case 6: block_gram_reg_kernel<6><<<rgrid, kGramRegT, 0, c.stream>>>(T, m, Rinv, q.gpart, q.disabled); break;
            case 8: block_gram_reg_kernel<8><<<rgrid, kGramRegT, 0, c.stream>>>(T, m, Rinv, q.gpart, q.disabled); break;
            case 9: block_gram_reg_kernel<9><<<rgrid, kGramRegT, 0, c.stream>>>(T, m, Rinv, q.gpart, q.disabled); break;
            case 12: block_gram_reg_kernel<12><<<rgrid, kGramRegT, 0, c.stream>>>(T, m, Rinv, q.gpart, q.disabled); break;
            default: block_gram_kernel<<<grid, kGramT, 0, c.stream>>>(T, m, k, Rinv, q.gpart, q.disabled); break;
        }
    };
    if (S && Z) {
        image_chol_kernel<<<1, kCholT, 0, c.stream>>>(*S, *Z, n, k, q.R1, q.R1inv, q.flag, q.disabled);
        c.launches += 1;
    } else {
        gram(nullptr);
        chol_small_kernel<<<1, kCholT, 0, c.stream>>>(q.gpart, parts, k, q.R1, q.R1inv, nullptr,
                                                   nullptr, q.flag, 1, q.disabled);
        c.launches += 2;
    }
    gram(q.R1inv);
    chol_small_kernel<<<1, kCholT, 0, c.stream>>>(q.gpart, parts, k, nullptr, q.R2inv, q.R1, q.R,
                                               q.flag, 2, q.disabled);
    MSVD_CUDA(cudaGetLastError());
    c.launches += 2;
}

}  // namespace msvd
