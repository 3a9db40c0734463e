// Randomized preconditioner factorization (precond.cpp:11-36).
//
// dense_svd(SA) in the reference is Householder QR (d x n -> n x n R) then
// one-sided Jacobi on R (svd.cpp:99-150, :180-252).  The default here
// ("eigj") is the same one-sided Jacobi, run on SA itself (same Gram as R)
// and started from the eigenvectors of SA^T SA (cuSOLVER syevd): B = SA V0 has
// nearly orthogonal columns, so the Jacobi sweeps converge in one or two
// passes.  Those passes run as dense simultaneous rotations on the
// tensor cores (all pair tangents from the Gram B^T B, Q = exp(K), B <- B Q,
// V <- V Q), with the reference's stop rule read from the Gram; pairs with
// large rotations (near-degenerate or rank-deficient clusters) get exact
// pairwise Jacobi sweeps, and anything else falls back to exact block sweeps
// over all pairs.  MSVD_SVD = eigj | polar | gesvd | gesvdj | gesvdp selects
// (the others: geqrf to R, then cuSOLVER's SVD of R; polar = QDWH gesvdp + an
// inverse-iteration refinement of its tail).
// A small kernel then applies the reference's conventions: descending order,
// each right vector signed so its largest-magnitude entry is positive
// (svd.cpp:232-248), and the sqrt(n) u sigma_1 floor (precond.cpp:26-34).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"
#include "msvd_internal.h"

namespace msvd {

namespace cg = cooperative_groups;

namespace {

#define MSVD_SOLVER(x)                                                                        \
    do {                                                                                      \
        cusolverStatus_t st__ = (x);                                                          \
        if (st__ != CUSOLVER_STATUS_SUCCESS)                                                  \
            fail(MSVD_ERR_CUDA, std::string("cuSOLVER failure ") + std::to_string(st__) + " in " #x); \
    } while (0)

__global__ void upper_copy_kernel(const double* W, int64_t ldw, int64_t n, double* R) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * n) return;
    const int64_t r = i % n, c = i / n;
    R[i] = r <= c ? W[r + c * ldw] : 0.0;
}

// V given column-major (vt_layout 0) or as V^T column-major (1).  Produce
// sign-fixed Vcol (column-major) and Vrow (row-major) copies: each column
// signed so its largest-magnitude entry (first one on ties) is positive
// (svd.cpp:232-248).  One CTA per column.
__global__ void signfix_kernel(const double* Vin, int vt_layout, int64_t n, double* Vcol, double* Vrow) {
    const int64_t j = blockIdx.x;
    __shared__ double bv[32];
    __shared__ int64_t bi[32];
    auto at = [&](int64_t i) { return vt_layout ? Vin[j + i * n] : Vin[i + j * n]; };
    double amax = -1.0;
    int64_t imax = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double a = fabs(at(i));
        if (a > amax) {  // ascending i per thread: keeps the first maximum
            amax = a;
            imax = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, amax, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, imax, o);
        if (ov > amax || (ov == amax && oi < imax)) {
            amax = ov;
            imax = oi;
        }
    }
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        bv[warp] = amax;
        bi[warp] = imax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
            if (bv[w] > bv[0] || (bv[w] == bv[0] && bi[w] < bi[0])) {
                bv[0] = bv[w];
                bi[0] = bi[w];
            }
    }
    __syncthreads();
    const double s = at(bi[0]) < 0.0 ? -1.0 : 1.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = s * at(i);
        Vcol[i + j * n] = v;
        Vrow[j + i * n] = v;
    }
}

__global__ void floor_kernel(double* sig, int64_t n, double* out2, int* info_flag) {
    // single thread: n <= a few thousand, runs once per solve
    const double smax = sig[0];
    const double fl = sqrt(static_cast<double>(n)) * 2.220446049250313e-16 * smax;
    long long cnt = 0;
    for (int64_t j = 0; j < n; ++j)
        if (sig[j] < fl) {
            sig[j] = fl;
            ++cnt;
        }
    out2[0] = smax;
    out2[1] = static_cast<double>(cnt);
    out2[2] = static_cast<double>(*info_flag);
}

// defensive: enforce descending order (the SVDs return sorted values)
__global__ void check_sorted_kernel(const double* sig, int64_t n, int* flag) {
    for (int64_t j = 1 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (sig[j] > sig[j - 1]) atomicCAS(flag, 0, 1000 + static_cast<int>(j));
}

// Triangular solves for the tail refinement (single CTA, p <= 32 right-hand
// sides, axpy form so every update reads a contiguous column of M):
//   back = 1: U x = y with U = M upper (back substitution)
//   back = 0: L y = z with L = M lower, i.e. M = U^T stored column-major
// Diagonal entries below delta are raised to +-delta (inverse-iteration guard
// for a numerically singular R).
__global__ void __launch_bounds__(1024) trsm_tail_kernel(const double* M, int64_t n, double* X, int p, int back,
                                                         double delta) {
    __shared__ double xi[32];
    for (int64_t step = 0; step < n; ++step) {
        const int64_t i = back ? n - 1 - step : step;
        if (threadIdx.x < p) {
            double d = M[i + i * n];
            if (fabs(d) < delta) d = d < 0.0 ? -delta : delta;
            const double x = X[i + threadIdx.x * n] / d;
            X[i + threadIdx.x * n] = x;
            xi[threadIdx.x] = x;
        }
        __syncthreads();
        const int64_t k0 = back ? 0 : i + 1;
        const int64_t len = back ? i : n - i - 1;
        const double* mc = M + i * n;
        for (int64_t t = threadIdx.x; t < len * p; t += blockDim.x) {
            const int64_t k = k0 + t % len;
            const int j = static_cast<int>(t / len);
            X[k + j * n] -= mc[k] * xi[j];
        }
        __syncthreads();
    }
}

// out (n x p) = U Z with U upper triangular (column-major)
__global__ void upper_times_kernel(const double* U, int64_t n, const double* Z, int p, double* out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n * p) return;
    const int64_t i = t % n;
    const int j = static_cast<int>(t / n);
    double s = 0.0;
    for (int64_t k = i; k < n; ++k) s = fma(U[i + k * n], Z[k + j * n], s);
    out[i + j * n] = s;
}

// V[:, n-p+j] = sum_l Z[:, l] W[l, j]; sig[n-p+j] = sgs[j]
__global__ void tail_write_kernel(const double* Z, int64_t n, int p, const double* W, const double* sgs, double* V,
                                  double* sig) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < p) sig[n - p + t] = sgs[t];
    if (t >= n * p) return;
    const int64_t i = t % n;
    const int j = static_cast<int>(t / n);
    double s = 0.0;
    for (int l = 0; l < p; ++l) s = fma(Z[i + l * n], W[l + j * p], s);
    V[i + (n - p + j) * n] = s;
}

__global__ void transpose_sq_kernel(const double* A, int64_t n, double* out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n * n) return;
    const int64_t i = t % n, j = t / n;
    out[j + i * n] = A[i + j * n];
}

// stable descending sort of sig with the columns of V (single thread picks the
// order -- the input is sorted except possibly at the refined tail boundary)
__global__ void sort_cols_kernel(double* sig, int64_t n, int* ord, double* tmps) {
    for (int64_t j = 0; j < n; ++j) ord[j] = static_cast<int>(j);
    for (int64_t j = 1; j < n; ++j) {
        const int key = ord[j];
        int64_t i = j - 1;
        while (i >= 0 && sig[key] > sig[ord[i]]) {
            ord[i + 1] = ord[i];
            --i;
        }
        ord[i + 1] = key;
    }
    for (int64_t j = 0; j < n; ++j) tmps[j] = sig[ord[j]];
    for (int64_t j = 0; j < n; ++j) sig[j] = tmps[j];
}
__global__ void permute_cols_kernel(const double* V, int64_t n, const int* ord, double* out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n * n) return;
    const int64_t i = t % n, j = t / n;
    out[i + j * n] = V[i + static_cast<int64_t>(ord[j]) * n];
}


// ---- eig-started one-sided Jacobi ("eigj") --------------------------------
// One-sided Jacobi (svd.cpp:99-150: same rotation formulas, same 1e-15
// pair-cosine threshold, same 60-sweep limit) on B = R V0, where V0 are the
// eigenvectors of R^T R.  The eigen-solve is only a starting rotation: the
// columns of B are already nearly orthogonal, so the sweeps that restore the
// reference's Jacobi accuracy converge quadratically in a few passes instead
// of the ~10 a cold start needs.  One persistent cooperative grid: each round
// of the parallel round-robin ordering rotates n/2 disjoint column pairs (one
// CTA per pair, fixed-order block reductions -> deterministic), then the grid
// synchronises.  B and V (2 n^2 doubles) stay resident in L2.
struct JacobiGridArgs {
    double* B;       // rows x n column-major
    double* V;       // n x n column-major
    int rows;
    int n;
    double* worst;   // [kJacMaxSweeps] pair-cosine maxima, zeroed
    int* status;     // [0] sweeps used, [1] 0 ok / 1 no convergence
};
constexpr int kJacMaxSweeps = 60;
constexpr int kJacThreads = 256;

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(__double_as_longlong(v)));
}

__global__ void __launch_bounds__(kJacThreads) jacobi_grid_kernel(JacobiGridArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[3][kJacThreads / 32];
    __shared__ double rot[3];
    const int n = a.n, K2 = n + (n & 1), npairs = K2 / 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int sweep = 0;
    bool converged = n <= 1;
    for (; sweep < kJacMaxSweeps && !converged; ++sweep) {
        for (int r = 0; r < K2 - 1; ++r) {
            for (int pi = blockIdx.x; pi < npairs; pi += gridDim.x) {
                int p, q;
                if (pi == 0) {
                    p = r;
                    q = K2 - 1;
                } else {
                    p = (r + pi) % (K2 - 1);
                    q = (r - pi + (K2 - 1)) % (K2 - 1);
                }
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                if (q >= n) continue;  // odd n: the phantom column
                double* bp = a.B + static_cast<size_t>(p) * a.rows;
                double* bq = a.B + static_cast<size_t>(q) * a.rows;
                double spp = 0.0, sqq = 0.0, spq = 0.0;
                for (int i = threadIdx.x; i < a.rows; i += kJacThreads) {
                    const double x = bp[i], y = bq[i];
                    spp = fma(x, x, spp);
                    sqq = fma(y, y, sqq);
                    spq = fma(x, y, spq);
                }
                spp = warp_sum(spp);
                sqq = warp_sum(sqq);
                spq = warp_sum(spq);
                if (lane == 0) {
                    red[0][warp] = spp;
                    red[1][warp] = sqq;
                    red[2][warp] = spq;
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    double app = 0.0, aqq = 0.0, apq = 0.0;
                    for (int w = 0; w < kJacThreads / 32; ++w) {
                        app += red[0][w];
                        aqq += red[1][w];
                        apq += red[2][w];
                    }
                    double c = 1.0, sn = 0.0;
                    bool go = false;
                    if (!(app == 0.0 || aqq == 0.0 || apq == 0.0)) {
                        const double rel = fabs(apq) / sqrt(app * aqq);
                        atomic_max_nonneg(&a.worst[sweep], rel);
                        if (rel > 1e-15) {
                            const double tau = (aqq - app) / (2.0 * apq);
                            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                            c = 1.0 / sqrt(1.0 + t * t);
                            sn = c * t;
                            go = true;
                        }
                    }
                    rot[0] = c;
                    rot[1] = sn;
                    rot[2] = go ? 1.0 : 0.0;
                }
                __syncthreads();
                if (rot[2] != 0.0) {
                    const double c = rot[0], sn = rot[1];
                    double* vp = a.V + static_cast<size_t>(p) * n;
                    double* vq = a.V + static_cast<size_t>(q) * n;
                    for (int i = threadIdx.x; i < a.rows; i += kJacThreads) {
                        const double xp = bp[i], xq = bq[i];
                        bp[i] = c * xp - sn * xq;
                        bq[i] = sn * xp + c * xq;
                    }
                    for (int i = threadIdx.x; i < n; i += kJacThreads) {
                        const double yp = vp[i], yq = vq[i];
                        vp[i] = c * yp - sn * yq;
                        vq[i] = sn * yp + c * yq;
                    }
                }
                __syncthreads();
            }
            grid.sync();
        }
        converged = *reinterpret_cast<volatile double*>(&a.worst[sweep]) <= 1e-15;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.status[0] = sweep;
        a.status[1] = converged ? 0 : 1;
    }
}

constexpr double kStrongT = 1e-2;  // |tan| above which a pair goes to the exact cluster sweep
constexpr int kMaxCluster = 64;

// All pair rotations of one Jacobi sweep at once, from the Gram H = B^T B:
// K(p, q) = t_pq, K(q, p) = -t_pq with t the reference's rotation tangent
// (svd.cpp:118-131; pairs at or below the 1e-15 cosine are left alone, zero
// columns skipped).  Per-block partials: max pair cosine, max |t|, sum t^2.
__global__ void pair_rot_kernel(const double* H, int64_t n, double* K, double* part, int* strong) {
    __shared__ double red[4][8];
    double mrel = 0.0, mt = 0.0, st = 0.0, ns = 0.0;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < n * n;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx % n, j = idx / n;
        double kv = 0.0;
        if (i != j) {
            const int64_t p = i < j ? i : j, q = i < j ? j : i;
            const double app = H[p + p * n], aqq = H[q + q * n], apq = H[p + q * n];
            if (!(app == 0.0 || aqq == 0.0 || apq == 0.0)) {
                const double rel = fabs(apq) / sqrt(app * aqq);
                if (rel > 1e-15) {
                    const double tau = (aqq - app) / (2.0 * apq);
                    const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                    if (fabs(t) > kStrongT) {  // left to the exact cluster sweep
                        if (i < j) {
                            strong[p] = 1;
                            strong[q] = 1;
                            ns += 1.0;
                        }
                    } else {
                        kv = i < j ? t : -t;
                        if (i < j) {
                            mt = fmax(mt, fabs(t));
                            st = fma(t, t, st);
                        }
                    }
                }
                if (i < j) mrel = fmax(mrel, rel);
            }
        }
        K[idx] = kv;
    }
    for (int o = 16; o > 0; o >>= 1) {
        mrel = fmax(mrel, __shfl_xor_sync(0xffffffffu, mrel, o));
        mt = fmax(mt, __shfl_xor_sync(0xffffffffu, mt, o));
        st += __shfl_xor_sync(0xffffffffu, st, o);
        ns += __shfl_xor_sync(0xffffffffu, ns, o);
    }
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][warp] = mrel;
        red[1][warp] = mt;
        red[2][warp] = st;
        red[3][warp] = ns;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0, s2 = 0.0, s3 = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            a = fmax(a, red[0][w]);
            b = fmax(b, red[1][w]);
            s2 += red[2][w];
            s3 += red[3][w];
        }
        part[4 * blockIdx.x] = a;
        part[4 * blockIdx.x + 1] = b;
        part[4 * blockIdx.x + 2] = s2;
        part[4 * blockIdx.x + 3] = s3;
    }
}


// Exact one-sided Jacobi (svd.cpp:99-150) restricted to the few columns that
// take part in strong rotations (near-degenerate or rank-deficient clusters):
// one CTA, round-robin over the m <= 64 listed columns, a warp per pair,
// sweeps until every pair inside the cluster is at or below 1e-15.
__global__ void __launch_bounds__(1024) cluster_jacobi_kernel(double* B, double* V, int64_t rows, int64_t n, const int* cols,
                                                              int m, int* status) {
    __shared__ double worst;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int M2 = m + (m & 1);
    int sweep = 0;
    bool conv = m <= 1;
    for (; sweep < kJacMaxSweeps && !conv; ++sweep) {
        if (threadIdx.x == 0) worst = 0.0;
        __syncthreads();
        for (int r = 0; r < M2 - 1; ++r) {
            for (int pi = warp; pi < M2 / 2; pi += nw) {
                int a, b;
                if (pi == 0) {
                    a = r;
                    b = M2 - 1;
                } else {
                    a = (r + pi) % (M2 - 1);
                    b = (r - pi + (M2 - 1)) % (M2 - 1);
                }
                if (a >= m || b >= m) continue;
                const int p = min(cols[a], cols[b]), q = max(cols[a], cols[b]);
                double* bp = B + static_cast<size_t>(p) * rows;
                double* bq = B + static_cast<size_t>(q) * rows;
                double app = 0.0, aqq = 0.0, apq = 0.0;
                for (int64_t i = lane; i < rows; i += 32) {
                    const double x = bp[i], y = bq[i];
                    app = fma(x, x, app);
                    aqq = fma(y, y, aqq);
                    apq = fma(x, y, apq);
                }
                app = warp_sum(app);
                aqq = warp_sum(aqq);
                apq = warp_sum(apq);
                if (app == 0.0 || aqq == 0.0 || apq == 0.0) continue;
                const double rel = fabs(apq) / sqrt(app * aqq);
                if (lane == 0) atomic_max_nonneg(&worst, rel);
                if (rel <= 1e-15) continue;
                const double tau = (aqq - app) / (2.0 * apq);
                const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double sn = c * t;
                double* vp = V + static_cast<size_t>(p) * n;
                double* vq = V + static_cast<size_t>(q) * n;
                for (int64_t i = lane; i < rows; i += 32) {
                    const double xp = bp[i], xq = bq[i];
                    bp[i] = c * xp - sn * xq;
                    bq[i] = sn * xp + c * xq;
                }
                for (int64_t i = lane; i < n; i += 32) {
                    const double yp = vp[i], yq = vq[i];
                    vp[i] = c * yp - sn * yq;
                    vq[i] = sn * yp + c * yq;
                }
            }
            __syncthreads();
        }
        conv = worst <= 1e-15;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        status[0] = sweep;
        status[1] = conv ? 0 : 1;
    }
}

// T = I + alpha K
__global__ void ident_axpy_kernel(const double* K, double alpha, int64_t n, double* T) {
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < n * n;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x)
        T[idx] = (K ? alpha * K[idx] : 0.0) + ((idx % n) == (idx / n) ? 1.0 : 0.0);
}

// sig[j] = ||B(:, j)|| (warp per column, fixed-order sums)
__global__ void colnorm_kernel(const double* B, int64_t rows, int64_t n, double* sig) {
    const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (j >= n) return;
    double s = 0.0;
    for (int64_t i = lane; i < rows; i += 32) s = fma(B[i + j * rows], B[i + j * rows], s);
    s = warp_sum(s);
    if (lane == 0) sig[j] = sqrt(s);
}

// stable descending order by rank: rank(i) = #{sig_j > sig_i} + #{j < i : sig_j == sig_i}
__global__ void rank_sort_kernel(const double* sig, int64_t n, const double* V, double* sig_out, double* V_out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x);
    __shared__ int64_t rk;
    if (threadIdx.x == 0) rk = 0;
    __syncthreads();
    const double si = sig[i];
    int64_t cnt = 0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        const double sj = sig[j];
        cnt += (sj > si || (sj == si && j < i)) ? 1 : 0;
    }
    cnt = static_cast<int64_t>(warp_sum(static_cast<double>(cnt)));
    if ((threadIdx.x & 31) == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&rk), static_cast<unsigned long long>(cnt));
    __syncthreads();
    const int64_t r = rk;
    if (threadIdx.x == 0) sig_out[r] = si;
    for (int64_t t = threadIdx.x; t < n; t += blockDim.x) V_out[t + r * n] = V[t + i * n];
}
}  // namespace

// Polar SVD (cusolver gesvdp, QDWH) is fast but only backward stable to a few
// hundred ulps of sigma_1, so its smallest singular triplets -- the ones that
// set the preconditioner's dominant weights, the floor count and the start
// block V0 -- can be off by many orders of magnitude relative to the
// one-sided Jacobi of the reference (a floored nullspace comes out at 1e-11
// instead of 1e-15).  They are recomputed here the way inverse iteration
// would: two block inverse iterations with R (which suppress every larger
// singular direction by (sigma_tail / sigma)^2 per step), then Rayleigh-Ritz
// through an exact one-sided Jacobi SVD of R Z (svd.cpp:99-150 semantics).
template <class LW>
static void refine_tail(Ctx& c, const double* R, int64_t n, double* V, double* sig, int tail_hint, double err_sigma,
                        int* info, LW&& lwork_buf) {
    std::vector<double> hs(n);
    MSVD_CUDA(cudaMemcpyAsync(hs.data(), sig, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
    MSVD_CUDA(cudaStreamSynchronize(c.stream));
    // refine exactly the triplets the polar SVD cannot resolve: sigma below
    // 1e3 x its backward error (or the sqrt(n) u sigma_1 floor region).  A
    // block mixing those with well-resolved ones would be swamped by the
    // (sigma_max / sigma_min)^2 growth of inverse iteration.
    (void)tail_hint;
    const double tau = std::max(1e3 * err_sigma, 1e3 * std::sqrt(static_cast<double>(n)) * 2.220446049250313e-16 *
                                                     hs[0]);
    int p = 0;
    for (int64_t j = 0; j < n; ++j)
        if (hs[j] < tau) p = std::max<int>(p, static_cast<int>(n - j));
    p = static_cast<int>(std::min<int64_t>(std::min<int64_t>(p, n), 24));
    if (p == 0) return;
    const int64_t np = n * p;
    double* base = static_cast<double*>(c.ensure_scratch(sizeof(double) * (n * n + 3 * np + 3 * p * p + 4 * p + 64) +
                                                         sizeof(DevState) + 4096));
    double* Rt = base;
    double* Z = Rt + n * n;
    double* Bm = Z + np;
    double* tz = Bm + np;
    double* W = tz + np;
    double* sgs = W + p * p;
    double* Rs = sgs + p;
    DevState* st = reinterpret_cast<DevState*>(Rs + p * p + 64);
    MSVD_CUDA(cudaMemsetAsync(st, 0, sizeof(DevState), c.stream));
    const unsigned g2 = static_cast<unsigned>(ceil_div(n * n, 256));
    transpose_sq_kernel<<<g2, 256, 0, c.stream>>>(R, n, Rt);
    MSVD_CUDA(cudaMemcpyAsync(Z, V + (n - p) * n, sizeof(double) * np, cudaMemcpyDeviceToDevice, c.stream));
    const double delta = static_cast<double>(n) * 2.220446049250313e-16 * hs[0];
    const int in = static_cast<int>(n);
    int lq = 0, lo = 0;
    MSVD_SOLVER(cusolverDnDgeqrf_bufferSize(c.solver, in, p, Z, in, &lq));
    MSVD_SOLVER(cusolverDnDorgqr_bufferSize(c.solver, in, p, p, Z, in, tz, &lo));
    double* lw = lwork_buf(sizeof(double) * (std::max(lq, lo) + 1));
    for (int half = 0; half < 4; ++half) {  // (R^T R)^-2 in four orthonormalized half steps
        if (half % 2 == 0) trsm_tail_kernel<<<1, 1024, 0, c.stream>>>(Rt, n, Z, p, 0, delta);  // R^T y = z
        else trsm_tail_kernel<<<1, 1024, 0, c.stream>>>(R, n, Z, p, 1, delta);                 // R x = y
        MSVD_SOLVER(cusolverDnDgeqrf(c.solver, in, p, Z, in, tz, lw, std::max(lq, lo), info));
        MSVD_SOLVER(cusolverDnDorgqr(c.solver, in, p, p, Z, in, tz, lw, std::max(lq, lo), info));
    }
    upper_times_kernel<<<static_cast<unsigned>(ceil_div(np, 256)), 256, 0, c.stream>>>(R, n, Z, p, Bm);
    MSVD_SOLVER(cusolverDnDgeqrf(c.solver, in, p, Bm, in, tz, lw, std::max(lq, lo), info));
    upper_copy_kernel<<<static_cast<unsigned>(ceil_div(p * p, 256)), 256, 0, c.stream>>>(Bm, n, p, Rs);
    launch_small_svd(c, Rs, p, sgs, W, st);
    tail_write_kernel<<<static_cast<unsigned>(ceil_div(np, 256)), 256, 0, c.stream>>>(Z, n, p, W, sgs, V, sig);
    // restore global order (the refined tail can only move at its boundary)
    int* ord = reinterpret_cast<int*>(Bm);  // n ints fit in n*p doubles
    sort_cols_kernel<<<1, 1, 0, c.stream>>>(sig, n, ord, Z);
    permute_cols_kernel<<<g2, 256, 0, c.stream>>>(V, n, ord, Rt);
    MSVD_CUDA(cudaMemcpyAsync(V, Rt, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, c.stream));
    MSVD_CUDA(cudaGetLastError());
    c.launches += 10;
    DevState h;
    MSVD_CUDA(cudaMemcpyAsync(&h, st, sizeof(DevState), cudaMemcpyDeviceToHost, c.stream));
    MSVD_CUDA(cudaStreamSynchronize(c.stream));
    if (h.err_code) fail(MSVD_ERR_NUMERICAL, "build_preconditioner: tail refinement Jacobi did not converge");
}


// eig-started one-sided Jacobi SVD of the sketch SA (rows x n, column-major,
// leading dimension rows):  G = SA^T SA, V0 = eig(G) (cuSOLVER syevd),
// B = SA V0, then Jacobi passes on (B, V) to the reference's 1e-15 pair-cosine
// tolerance.  The reference runs its Jacobi on the R of a Householder QR of SA
// (svd.cpp:180-252); B^T B is the same Gram either way, and starting from SA
// skips the QR.  On return sig (descending) and V (n x n, column-major, same
// order).  work: >= rows*n doubles scratch; wv: >= n doubles.
template <class LW>
static void eig_jacobi(Ctx& c, const double* SA, int64_t rows, int64_t n, double* V, double* sig, double* work,
                       double* wv, int* info, LW&& lwork_buf) {
    if (!c.blas) {
        if (cublasCreate(&c.blas) != CUBLAS_STATUS_SUCCESS) fail(MSVD_ERR_CUDA, "cublasCreate failed");
        cublasSetPointerMode(c.blas, CUBLAS_POINTER_MODE_HOST);
    }
    if (cublasSetStream(c.blas, c.stream) != CUBLAS_STATUS_SUCCESS) fail(MSVD_ERR_CUDA, "cublasSetStream failed");
    const int in = static_cast<int>(n), ir = static_cast<int>(rows);
    // C (mm x nn) = alpha op(A) Bm + beta C, inner dimension kk
    auto gemm = [&](cublasOperation_t ta, int mm, int nn_, int kk, const double* A, int lda, const double* Bm, int ldb,
                    double alpha, double beta, double* C, int ldc, const char* what) {
        if (cublasDgemm(c.blas, ta, CUBLAS_OP_N, mm, nn_, kk, &alpha, A, lda, Bm, ldb, &beta, C, ldc) !=
            CUBLAS_STATUS_SUCCESS)
            fail(MSVD_ERR_CUDA, std::string("cublasDgemm failed: ") + what);
    };
    // G = SA^T SA into V (syevd reads the lower triangle)
    gemm(CUBLAS_OP_T, in, in, ir, SA, ir, SA, ir, 1.0, 0.0, V, in, "SA^T SA");
    int lwork = 0;
    MSVD_SOLVER(cusolverDnDsyevd_bufferSize(c.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, in, V, in, wv,
                                            &lwork));
    double* lw = lwork_buf(sizeof(double) * (lwork + 1));
    MSVD_SOLVER(cusolverDnDsyevd(c.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, in, V, in, wv, lw, lwork,
                                 info));
    // B = SA V0 into work
    gemm(CUBLAS_OP_N, ir, in, in, SA, ir, V, in, 1.0, 0.0, work, ir, "SA V0");
    c.launches += 3;

    // Simultaneous passes while every rotation is small: K holds the tangent
    // of every pair's Jacobi rotation (svd.cpp:118-131) computed from the
    // Gram B^T B, Q = exp(K) (scaling and squaring around a degree-5 Taylor in
    // Horner form, ||K / 2^s||_F <= 1e-3), B <- B Q, V <- V Q.  Each pass
    // squares the off-diagonal mass like a Jacobi sweep.  Pairs whose rotation
    // is large (near-degenerate or rank-deficient clusters, |t| > 1e-2) are
    // left out of K and rotated by exact pairwise sweeps over just their
    // columns; anything else falls through to exact sweeps over all pairs.
    const size_t nn = static_cast<size_t>(n) * n, rn = static_cast<size_t>(rows) * n;
    const int pgrid = static_cast<int>(std::min<int64_t>(ceil_div(static_cast<int64_t>(nn), 256), 4 * c.num_sms));
    double* pool = lwork_buf(sizeof(double) * (2 * nn + rn + 4 * pgrid + 8) + sizeof(int) * (2 * n + 8));
    double* K = pool;
    double* T2 = K + nn;
    double* T1 = T2 + nn;  // rows x n: the Gram, Taylor terms, then B Q
    double* part = T1 + rn;
    int* strong = reinterpret_cast<int*>(part + 4 * pgrid + 8);
    int* clist = strong + n;
    int* cstat = clist + n;
    double* B = work;
    double* Vp = V;
    std::vector<double> hp(4 * pgrid);
    std::vector<int> hflag(n), hcols;
    bool done = false;
    int steps = 0, csweeps = 0;
    const char* ms = std::getenv("MSVD_JACOBI_GEMM_STEPS");
    const int max_steps = ms ? std::atoi(ms) : 8;
    const bool dbg = std::getenv("MSVD_DEBUG_JACOBI") != nullptr;
    for (; steps < max_steps; ++steps) {
        gemm(CUBLAS_OP_T, in, in, ir, B, ir, B, ir, 1.0, 0.0, T1, in, "B^T B");
        MSVD_CUDA(cudaMemsetAsync(strong, 0, sizeof(int) * n, c.stream));
        pair_rot_kernel<<<pgrid, 256, 0, c.stream>>>(T1, n, K, part, strong);
        MSVD_CUDA(cudaMemcpyAsync(hp.data(), part, sizeof(double) * 4 * pgrid, cudaMemcpyDeviceToHost, c.stream));
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
        c.launches += 2;
        double mrel = 0.0, mt = 0.0, st = 0.0, ns = 0.0;
        for (int b = 0; b < pgrid; ++b) {
            mrel = std::max(mrel, hp[4 * b]);
            mt = std::max(mt, hp[4 * b + 1]);
            st += hp[4 * b + 2];
            ns += hp[4 * b + 3];
        }
        const double fro = std::sqrt(2.0 * st);
        if (dbg)
            std::fprintf(stderr, "eig_jacobi: step %d max cos %.3e max t %.3e ||K||_F %.3e strong pairs %.0f\n", steps,
                         mrel, mt, fro, ns);
        if (mrel <= 1e-15) {  // the reference's stop rule, svd.cpp:146
            done = true;
            break;
        }
        hcols.clear();
        if (ns > 0) {
            MSVD_CUDA(cudaMemcpyAsync(hflag.data(), strong, sizeof(int) * n, cudaMemcpyDeviceToHost, c.stream));
            MSVD_CUDA(cudaStreamSynchronize(c.stream));
            for (int64_t j = 0; j < n; ++j)
                if (hflag[j]) hcols.push_back(static_cast<int>(j));
        }
        if (fro > 4.0 || static_cast<int>(hcols.size()) > kMaxCluster) break;  // -> exact sweeps
        // the rotation that reaches the GEMM-cosine floor is the last one
        const bool last = mrel <= 1e-13 && hcols.empty();
        if (st > 0.0) {
            // exp(K) = exp(K / 2^sq)^(2^sq), with ||K / 2^sq||_F <= 1e-3, and a
            // Taylor degree just high enough that the first dropped term
            // x^(d+1) / (d+1)! is below 1e-17 (x = ||K / 2^sq||_F): near
            // convergence Q = I + K needs no GEMM at all
            int sq = 0;
            while (fro / std::ldexp(1.0, sq) > 1e-3) ++sq;
            const double sc = std::ldexp(1.0, -sq);
            const double x = fro * sc;
            int deg = 1;
            double term = x * x / 2.0;
            while (deg < 5 && term > 1e-17) {
                ++deg;
                term *= x / (deg + 1);
            }
            ident_axpy_kernel<<<pgrid, 256, 0, c.stream>>>(K, sc / deg, n, T2);
            double* Ta = T1;
            double* Tb = T2;
            for (int dd = deg - 1; dd >= 1; --dd) {  // Horner: I + K/dd (...)
                ident_axpy_kernel<<<pgrid, 256, 0, c.stream>>>(nullptr, 0.0, n, Ta);
                gemm(CUBLAS_OP_N, in, in, in, K, in, Tb, in, sc / dd, 1.0, Ta, in, "Taylor");
                std::swap(Ta, Tb);
            }
            for (int k = 0; k < sq; ++k) {
                gemm(CUBLAS_OP_N, in, in, in, Tb, in, Tb, in, 1.0, 0.0, Ta, in, "square");
                std::swap(Ta, Tb);
            }
            if (Tb != T2) {
                MSVD_CUDA(cudaMemcpyAsync(T2, Tb, sizeof(double) * nn, cudaMemcpyDeviceToDevice, c.stream));
                Tb = T2;
            }
            c.launches += sq;
            // Q = exp(K) in Tb == T2.  After the last rotation only V is
            // needed: sigma = column norms of B Q = those of B to O(||K||^2)
            // relative (below 1e-26 here), so B is not rotated again
            if (!last) {
                gemm(CUBLAS_OP_N, ir, in, in, B, ir, Tb, in, 1.0, 0.0, T1, ir, "B Q");
                std::swap(B, T1);
            }
            gemm(CUBLAS_OP_N, in, in, in, Vp, in, Tb, in, 1.0, 0.0, K, in, "V Q");
            std::swap(Vp, K);
            c.launches += 2 * deg + 1;
        }
        if (!hcols.empty()) {
            MSVD_CUDA(cudaMemcpyAsync(clist, hcols.data(), sizeof(int) * hcols.size(), cudaMemcpyHostToDevice,
                                      c.stream));
            cluster_jacobi_kernel<<<1, 1024, 0, c.stream>>>(B, Vp, rows, n, clist, static_cast<int>(hcols.size()),
                                                            cstat);
            int h2[2];
            MSVD_CUDA(cudaMemcpyAsync(h2, cstat, sizeof(h2), cudaMemcpyDeviceToHost, c.stream));
            MSVD_CUDA(cudaStreamSynchronize(c.stream));
            ++c.launches;
            csweeps += h2[0];
            if (h2[1]) fail(MSVD_ERR_NUMERICAL, "one_sided_jacobi: no convergence after 60 sweeps (cluster)");
        }
        // GEMM cosines carry a ~sqrt(rows) u roundoff floor right at the 1e-15
        // threshold: once every computed cosine is at that floor (<= 1e-13),
        // the rotation just applied leaves the true cosines at O(max^2).
        if (mrel <= 1e-13) {
            done = true;
            ++steps;
            break;
        }
    }
    int hs[2] = {0, 0};
    if (!done) {
        // exact pairwise sweeps over all pairs: worst[60] | status[2]
        double* worst = static_cast<double*>(c.ensure_scratch(sizeof(double) * (kJacMaxSweeps + 2)));
        int* status = reinterpret_cast<int*>(worst + kJacMaxSweeps);
        MSVD_CUDA(cudaMemsetAsync(worst, 0, sizeof(double) * (kJacMaxSweeps + 2), c.stream));
        JacobiGridArgs ja{B, Vp, ir, in, worst, status};
        void* kargs[] = {&ja};
        int per_sm = 0;
        MSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_grid_kernel, kJacThreads, 0));
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((n + (n & 1)) / 2, int64_t(per_sm) * c.num_sms));
        MSVD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(jacobi_grid_kernel),
                                              dim3(static_cast<unsigned>(grid)), dim3(kJacThreads), kargs, 0,
                                              c.stream));
        MSVD_CUDA(cudaMemcpyAsync(hs, status, sizeof(hs), cudaMemcpyDeviceToHost, c.stream));
        ++c.launches;
    }
    colnorm_kernel<<<static_cast<unsigned>(ceil_div(n * 32, 256)), 256, 0, c.stream>>>(B, rows, n, wv);
    // sorted copies into B's buffer (free after the norms), then into V
    rank_sort_kernel<<<static_cast<unsigned>(n), 256, 0, c.stream>>>(wv, n, Vp, sig, B);
    MSVD_CUDA(cudaMemcpyAsync(V, B, sizeof(double) * nn, cudaMemcpyDeviceToDevice, c.stream));
    MSVD_CUDA(cudaGetLastError());
    c.launches += 2;
    MSVD_CUDA(cudaStreamSynchronize(c.stream));
    if (dbg)
        std::fprintf(stderr, "eig_jacobi: n=%lld rows=%lld gemm steps=%d cluster sweeps=%d exact sweeps=%d\n",
                     static_cast<long long>(n), static_cast<long long>(rows), steps, csweeps, hs[0]);
    if (hs[1]) fail(MSVD_ERR_NUMERICAL, "one_sided_jacobi: no convergence after 60 sweeps");
}

void precond_build_dev(Ctx& c, const double* SA, int64_t rows, int64_t n, double* Vcol, double* Vrow, double* sig,
                       double* sigma_max, int64_t* nfloor, int tail_hint) {
    if (n < 1) fail(MSVD_ERR_DIMENSION, "build_preconditioner: empty sketch");
    if (rows < n) fail(MSVD_ERR_DIMENSION, "build_preconditioner: sketch has fewer rows than columns");
    ProfScope prof(c, kProfSvd);
    if (!c.solver) {
        MSVD_SOLVER(cusolverDnCreate(&c.solver));
    }
    MSVD_SOLVER(cusolverDnSetStream(c.solver, c.stream));
    const char* algo_env = std::getenv("MSVD_SVD");
    const std::string algo = algo_env ? algo_env : "eigj";
    const int in = static_cast<int>(n), ir = static_cast<int>(rows);

    // ctx-owned workspace (grown on demand, reused across solves):
    // work (rows x n) | R (n x n) | V (n x n) | tau (n) | out2 (4) | info (4 ints)
    const size_t wbytes = sizeof(double) * static_cast<size_t>(rows) * n;
    const size_t nn = sizeof(double) * static_cast<size_t>(n) * n;
    const size_t need = wbytes + 3 * nn + sizeof(double) * (n + 8) + 64;
    if (need > c.svd_ws_bytes) {
        if (c.svd_ws) MSVD_CUDA(cudaFree(c.svd_ws));
        c.svd_ws = nullptr;
        MSVD_CUDA(cudaMalloc(&c.svd_ws, need));
        c.svd_ws_bytes = need;
    }
    double* work = static_cast<double*>(c.svd_ws);
    double* R = work + static_cast<size_t>(rows) * n;
    double* V = R + static_cast<size_t>(n) * n;
    double* Rk = V + static_cast<size_t>(n) * n;  // R kept for the tail refinement
    double* tau = Rk + static_cast<size_t>(n) * n;
    double* out2 = tau + n;
    int* info = reinterpret_cast<int*>(out2 + 4);
    double* lw = nullptr;
    auto lwork_buf = [&](size_t bytes) -> double* {
        if (bytes > c.svd_lw_bytes) {
            if (c.svd_lw) MSVD_CUDA(cudaFree(c.svd_lw));
            c.svd_lw = nullptr;
            MSVD_CUDA(cudaMalloc(&c.svd_lw, bytes));
            c.svd_lw_bytes = bytes;
        }
        return static_cast<double*>(c.svd_lw);
    };
    MSVD_CUDA(cudaMemsetAsync(info, 0, sizeof(int) * 4, c.stream));
    int vt_layout = 0;
    try {
        if (algo == "eigj") {
            eig_jacobi(c, SA, rows, n, V, sig, work, tau, info + 1, lwork_buf);
        } else {
        MSVD_CUDA(cudaMemcpyAsync(work, SA, wbytes, cudaMemcpyDeviceToDevice, c.stream));
        if (rows > n) {
            int lwork = 0;
            MSVD_SOLVER(cusolverDnDgeqrf_bufferSize(c.solver, ir, in, work, ir, &lwork));
            lw = lwork_buf(sizeof(double) * (lwork + 1));
            MSVD_SOLVER(cusolverDnDgeqrf(c.solver, ir, in, work, ir, tau, lw, lwork, info));
            upper_copy_kernel<<<static_cast<unsigned>(ceil_div(n * n, 256)), 256, 0, c.stream>>>(work, rows, n, R);
        } else {
            MSVD_CUDA(cudaMemcpyAsync(R, work, nn, cudaMemcpyDeviceToDevice, c.stream));
        }
        if (algo == "gesvd") {
            int lwork = 0;
            MSVD_SOLVER(cusolverDnDgesvd_bufferSize(c.solver, in, in, &lwork));
            lw = lwork_buf(sizeof(double) * (lwork + 1));
            double* rwork = work;  // reuse (>= n doubles)
            MSVD_SOLVER(cusolverDnDgesvd(c.solver, 'N', 'A', in, in, R, in, sig, nullptr, 1, V, in, lw, lwork,
                                         rwork, info + 1));
            vt_layout = 1;
        } else if (algo == "gesvdp" || algo == "polar") {
            if (algo == "polar") MSVD_CUDA(cudaMemcpyAsync(Rk, R, nn, cudaMemcpyDeviceToDevice, c.stream));
            cusolverDnParams_t params;
            MSVD_SOLVER(cusolverDnCreateParams(&params));
            size_t dws = 0, hws = 0;
            double* U = work;  // n x n fits in rows x n
            MSVD_SOLVER(cusolverDnXgesvdp_bufferSize(c.solver, params, CUSOLVER_EIG_MODE_VECTOR, 0, n, n, CUDA_R_64F, R,
                                                     n, CUDA_R_64F, sig, CUDA_R_64F, U, n, CUDA_R_64F, V, n,
                                                     CUDA_R_64F, &dws, &hws));
            lw = lwork_buf(dws + 64);
            std::vector<char> hbuf(hws + 64);
            double err_sigma = 0.0;
            MSVD_SOLVER(cusolverDnXgesvdp(c.solver, params, CUSOLVER_EIG_MODE_VECTOR, 0, n, n, CUDA_R_64F, R, n,
                                          CUDA_R_64F, sig, CUDA_R_64F, U, n, CUDA_R_64F, V, n, CUDA_R_64F, lw, dws,
                                          hbuf.data(), hws, info + 1, &err_sigma));
            MSVD_SOLVER(cusolverDnDestroyParams(params));
            vt_layout = 0;
            if (algo == "polar") refine_tail(c, Rk, n, V, sig, tail_hint, err_sigma, info + 3, lwork_buf);
        } else {
            gesvdjInfo_t params;
            MSVD_SOLVER(cusolverDnCreateGesvdjInfo(&params));
            MSVD_SOLVER(cusolverDnXgesvdjSetTolerance(params, 2.220446049250313e-16));
            MSVD_SOLVER(cusolverDnXgesvdjSetMaxSweeps(params, 100));
            int lwork = 0;
            double* U = work;
            MSVD_SOLVER(cusolverDnDgesvdj_bufferSize(c.solver, CUSOLVER_EIG_MODE_VECTOR, 0, in, in, R, in, sig, U, in,
                                                     V, in, &lwork, params));
            lw = lwork_buf(sizeof(double) * (lwork + 1));
            MSVD_SOLVER(cusolverDnDgesvdj(c.solver, CUSOLVER_EIG_MODE_VECTOR, 0, in, in, R, in, sig, U, in, V, in, lw,
                                          lwork, info + 1, params));
            MSVD_SOLVER(cusolverDnDestroyGesvdjInfo(params));
            vt_layout = 0;
        }
        }  // R-based algorithms
        check_sorted_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c.stream>>>(sig, n, info + 2);
        signfix_kernel<<<static_cast<unsigned>(n), 256, 0, c.stream>>>(V, vt_layout, n, Vcol, Vrow);
        floor_kernel<<<1, 1, 0, c.stream>>>(sig, n, out2, info + 1);
        MSVD_CUDA(cudaGetLastError());
        c.launches += 4;
        double h[3];
        int hinfo[3];
        MSVD_CUDA(cudaMemcpyAsync(h, out2, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
        MSVD_CUDA(cudaMemcpyAsync(hinfo, info, sizeof(hinfo), cudaMemcpyDeviceToHost, c.stream));
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
        if (hinfo[0] != 0) fail(MSVD_ERR_NUMERICAL, "build_preconditioner: geqrf info " + std::to_string(hinfo[0]));
        if (hinfo[1] != 0)
            fail(MSVD_ERR_NUMERICAL, "build_preconditioner: " + algo + " did not converge (info " +
                                         std::to_string(hinfo[1]) + ")");
        if (hinfo[2] != 0) fail(MSVD_ERR_NUMERICAL, "build_preconditioner: singular values not sorted");
        *sigma_max = h[0];
        *nfloor = static_cast<int64_t>(h[1]);
    } catch (...) {
        throw;
    }
    if (*sigma_max == 0.0) fail(MSVD_ERR_NUMERICAL, "build_preconditioner: sketched matrix is exactly zero");
}

}  // namespace msvd
