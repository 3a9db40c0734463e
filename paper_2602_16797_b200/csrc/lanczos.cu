// Golub-Kahan-Lanczos baseline (baselines.cpp:51-166 lanczos_gk) on the device.
//
// The comparison method of the reference's `compare` client (cli.cpp:356-362)
// run over the same A passes as the solver: u = A v is the apply pass (K3,
// b = 1) and w = A^T u the Gram pass (K2, direct mode), each one streaming
// read of A.  Everything else is n- or m-side vector work on the device:
//
//  * two-pass reorthogonalization of w against the right basis V (n x j) and
//    of u against the left basis U (m_local x j).  The reference projects
//    modified-Gram-Schmidt style, one column at a time (baselines.cpp:19-31);
//    here each pass is classical (c = Q^T x, x -= Q c), two passes, which is
//    the same projector to rounding and turns j dependent reductions into two
//    coalesced sweeps over Q.
//  * the smallest singular triplet of the j x j upper-bidiagonal section
//    (baselines.cpp:33-40, :113-116).  The reference runs its dense Jacobi SVD
//    on the section; here one CTA bisects the Golub-Kahan tridiagonal
//    [[0 B^T];[B 0]] (zero diagonal, off-diagonal a1 b1 a2 b2 ... aj), whose
//    eigenvalues are +-sigma_i, with 256-way multisection on Sturm counts, then
//    runs inverse iteration (tridiagonal LU with partial pivoting) at the
//    converged shift; the right singular vector is the even half of the
//    eigenvector -- LAPACK dbdsvdx's route.  Sign fixed like dense_svd
//    (svd.cpp:232-248: largest |entry| positive).
//
// Control (the invariant-subspace tests and the record rows) reads a few
// scalars back per step; the run is A-pass bound (2 passes per step).
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "msvd_internal.h"

namespace msvd {
namespace {

constexpr double kEpsL = 2.220446049250313e-16;
constexpr int kBisT = 256;   // multisection width
constexpr int kRowsPerCta = 4096;

// ---------------------------------------------------------------- reductions
// parts[blockIdx.x] = sum of squares of x over the block's rows (fixed order)
__global__ void __launch_bounds__(256) sumsq_parts_kernel(const double* __restrict__ x, int64_t len, double* parts) {
    __shared__ double red[8];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kRowsPerCta;
    const int64_t r1 = r0 + kRowsPerCta < len ? r0 + kRowsPerCta : len;
    double s = 0.0;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += 256) s += x[r] * x[r];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        parts[blockIdx.x] = t;
    }
}
// out[0] = sum of parts (fixed order)
__global__ void sum_parts_kernel(const double* parts, int np, double* out) {
    __shared__ double red[8];
    double s = 0.0;
    for (int p = threadIdx.x; p < np; p += 256) s += parts[p];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        out[0] = t;
    }
}
// norm = sqrt(sumsq); dst = src * (1 / norm) (baselines.cpp scale(x, 1/norm))
__global__ void scale_by_norm_kernel(const double* __restrict__ src, int64_t len, const double* sumsq,
                                     double* norm_out, double* __restrict__ dst) {
    const double nr = sqrt(sumsq[0]);
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i == 0 && norm_out) norm_out[0] = nr;
    if (i < len) dst[i] = src[i] * (1.0 / nr);
}
// y += (-coef[0]) x  (axpy(-coef, x, y))
__global__ void axpy_neg_kernel(const double* __restrict__ x, int64_t len, const double* coef, double* __restrict__ y) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < len) y[i] += -coef[0] * x[i];
}

// ------------------------------------------------ projections c = Q^T x
// Q column-major (len x cols, ld); CTA b covers rows [b*4096, ...); warp w
// takes columns w, w+8, ...; part[b][l] = the CTA's partial dot.
__global__ void __launch_bounds__(256) proj_parts_kernel(const double* __restrict__ Q, int64_t ld, int64_t len,
                                                         int cols, const double* __restrict__ x, double* part) {
    __shared__ double xs[kRowsPerCta];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kRowsPerCta;
    const int rows = static_cast<int>(r0 + kRowsPerCta < len ? kRowsPerCta : len - r0);
    for (int i = threadIdx.x; i < rows; i += 256) xs[i] = x[r0 + i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int l = warp; l < cols; l += 8) {
        const double* q = Q + static_cast<int64_t>(l) * ld + r0;
        double s = 0.0;
        for (int i = lane; i < rows; i += 32) s += q[i] * xs[i];
        s = warp_sum(s);
        if (lane == 0) part[static_cast<int64_t>(blockIdx.x) * cols + l] = s;
    }
}
__global__ void proj_sum_kernel(const double* part, int np, int cols, double* c) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= cols) return;
    double s = 0.0;
    for (int p = 0; p < np; ++p) s += part[static_cast<int64_t>(p) * cols + l];
    c[l] = s;
}
// x -= Q c (classical Gram-Schmidt update); also y = Q c when `form` (the
// Ritz vector v_est = V y of baselines.cpp:117-119, sum in column order)
__global__ void __launch_bounds__(256) qc_kernel(const double* __restrict__ Q, int64_t ld, int64_t len, int cols,
                                                 const double* __restrict__ c, double* __restrict__ x, int form) {
    __shared__ double cs[1024];
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double s = 0.0;
    for (int l0 = 0; l0 < cols; l0 += 1024) {
        const int nl = cols - l0 < 1024 ? cols - l0 : 1024;
        __syncthreads();
        for (int t = threadIdx.x; t < nl; t += blockDim.x) cs[t] = c[l0 + t];
        __syncthreads();
        if (i < len)
            for (int l = 0; l < nl; ++l) s += cs[l] * Q[static_cast<int64_t>(l0 + l) * ld + i];
    }
    if (i >= len) return;
    if (form) x[i] = s;
    else x[i] -= s;
}

// ------------------------------------------- smallest triplet of a section
struct BidiagArgs {
    const double* alpha;   // a_0 .. a_{j-1}
    const double* beta;    // b_0 .. b_{j-2}
    int j;
    double* work;          // 6 * 2j doubles + 2j ints
    double* y;             // out: j, unit, sign-fixed
    double* theta;         // out
};

// Sturm count of T_GK - x I: eigenvalues of the zero-diagonal tridiagonal
// with off-diagonal squares e2[0..N-2] below x
__device__ int gk_count(const double* e2, int N, double x, double pivmin) {
    double q = -x;
    if (fabs(q) < pivmin) q = -pivmin;
    int cnt = q < 0.0;
    for (int k = 1; k < N; ++k) {
        q = -x - e2[k - 1] / q;
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

__global__ void __launch_bounds__(kBisT) bidiag_min_kernel(BidiagArgs a) {
    extern __shared__ double sh[];
    const int j = a.j, N = 2 * j;
    double* e = sh;          // N - 1 off-diagonals
    double* e2 = sh + N;     // squares
    __shared__ double s_lo, s_hi, s_pivmin, s_norm;
    __shared__ int s_best;
    for (int k = threadIdx.x; k < N - 1; k += blockDim.x) {
        const double v = (k & 1) ? a.beta[k >> 1] : a.alpha[k >> 1];
        e[k] = v;
        e2[k] = v * v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double emax = 0.0, cmin = INFINITY;
        for (int k = 0; k < N - 1; ++k) emax = fmax(emax, fabs(e[k]));
        // sigma_min <= the smallest column norm of B: column i = (b_{i-1}, a_i)
        for (int i = 0; i < j; ++i) {
            const double ai = a.alpha[i], bi = i > 0 ? a.beta[i - 1] : 0.0;
            cmin = fmin(cmin, sqrt(ai * ai + bi * bi));
        }
        s_norm = emax;
        s_pivmin = 2.2250738585072014e-308 * fmax(1.0, emax * emax);
        s_lo = 0.0;
        s_hi = cmin * (1.0 + 8.0 * kEpsL) + s_pivmin;
    }
    __syncthreads();
    // 256-way multisection: find the smallest x with count(x) > j
    for (int round = 0; round < 48; ++round) {
        const double lo = s_lo, hi = s_hi;
        if (!(hi - lo > 2.0 * kEpsL * hi) || hi <= 1e-300) break;
        const double x = lo + (hi - lo) * (static_cast<double>(threadIdx.x + 1) / (kBisT + 1));
        const bool above = gk_count(e2, N, x, s_pivmin) > j;
        if (threadIdx.x == 0) s_best = kBisT;
        __syncthreads();
        if (above) atomicMin(&s_best, static_cast<int>(threadIdx.x));
        __syncthreads();
        if (threadIdx.x == 0) {
            const int t = s_best;
            const double nlo = t == 0 ? lo : lo + (hi - lo) * (static_cast<double>(t) / (kBisT + 1));
            const double nhi = t == kBisT ? hi : lo + (hi - lo) * (static_cast<double>(t + 1) / (kBisT + 1));
            s_lo = nlo;
            s_hi = nhi;
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    const double theta = 0.5 * (s_lo + s_hi);
    // inverse iteration on T_GK - theta I: LU with partial pivoting (dgttrf)
    double* dl = a.work;          // N
    double* dd = a.work + N;      // N
    double* du = a.work + 2 * N;  // N
    double* du2 = a.work + 3 * N; // N
    double* z = a.work + 4 * N;   // N
    int* ip = reinterpret_cast<int*>(a.work + 5 * N);
    for (int k = 0; k < N; ++k) {
        dd[k] = -theta;
        dl[k] = k < N - 1 ? e[k] : 0.0;
        du[k] = k < N - 1 ? e[k] : 0.0;
        du2[k] = 0.0;
        ip[k] = 0;
    }
    const double tiny = fmax(kEpsL * s_norm, 1e-300);
    for (int i = 0; i < N - 1; ++i) {
        if (fabs(dd[i]) >= fabs(dl[i])) {
            if (dd[i] == 0.0) dd[i] = tiny;
            const double l = dl[i] / dd[i];
            dl[i] = l;
            dd[i + 1] -= l * du[i];
        } else {
            const double l = dd[i] / dl[i];
            dd[i] = dl[i];
            dl[i] = l;
            const double t = du[i];
            du[i] = dd[i + 1];
            dd[i + 1] = t - l * dd[i + 1];
            if (i < N - 2) {
                du2[i] = du[i + 1];
                du[i + 1] = -l * du[i + 1];
            }
            ip[i] = 1;
        }
    }
    if (dd[N - 1] == 0.0) dd[N - 1] = tiny;
    for (int k = 0; k < N; ++k) z[k] = 1.0;
    for (int it = 0; it < 3; ++it) {
        for (int i = 0; i < N - 1; ++i) {  // forward: P L
            if (ip[i]) {
                const double t = z[i];
                z[i] = z[i + 1];
                z[i + 1] = t - dl[i] * z[i];
            } else {
                z[i + 1] -= dl[i] * z[i];
            }
        }
        z[N - 1] /= dd[N - 1];  // backward: U with two superdiagonals
        if (N > 1) z[N - 2] = (z[N - 2] - du[N - 2] * z[N - 1]) / dd[N - 2];
        for (int i = N - 3; i >= 0; --i) z[i] = (z[i] - du[i] * z[i + 1] - du2[i] * z[i + 2]) / dd[i];
        double mx = 0.0;
        for (int k = 0; k < N; ++k) mx = fmax(mx, fabs(z[k]));
        if (!(mx > 0.0) || !isfinite(mx)) {
            for (int k = 0; k < N; ++k) z[k] = 1.0;
            break;
        }
        for (int k = 0; k < N; ++k) z[k] /= mx;
    }
    // right singular vector = even components, unit norm, largest |entry| > 0
    double nrm = 0.0;
    for (int i = 0; i < j; ++i) nrm += z[2 * i] * z[2 * i];
    nrm = sqrt(nrm);
    int imax = 0;
    double amax = -1.0;
    for (int i = 0; i < j; ++i)
        if (fabs(z[2 * i]) > amax) {
            amax = fabs(z[2 * i]);
            imax = i;
        }
    const double sgn = z[2 * imax] < 0.0 ? -1.0 : 1.0;
    for (int i = 0; i < j; ++i) a.y[i] = sgn * z[2 * i] / nrm;
    a.theta[0] = theta;
}

// per-step telemetry: out = {v_est . v_true (truth), |y_{j-1}|, alpha_{j-1}}
__global__ void __launch_bounds__(256) step_stats_kernel(const double* vest, const double* tv, int64_t n,
                                                         const double* y, const double* alpha, int j, double* out) {
    __shared__ double red[8];
    double s = 0.0;
    if (tv)
        for (int64_t i = threadIdx.x; i < n; i += 256) s += vest[i] * tv[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        out[0] = t;
        out[1] = fabs(y[j - 1]);
        out[2] = alpha[j - 1];
    }
}
__global__ void sqrt_store_kernel(const double* sumsq, double* dst) { dst[0] = sqrt(sumsq[0]); }

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

}  // namespace

void lanczos_run(Ctx& c, const msvd_matrix& M, int iters, const double* v0h, const msvd_truth* truth, bool timing,
                 msvd_lanczos_result* res) {
    const int64_t n = M.n, ml = M.m_local, m = M.m_global;
    Comm& comm = *c.comm;
    // baselines.cpp:53-61, in order
    if (m < n) fail(MSVD_ERR_DIMENSION, "lanczos_gk: matrix must be tall");
    if (iters < 1 || iters > n) fail(MSVD_ERR_DIMENSION, "lanczos_gk: step count must lie in [1, cols]");
    double v0n = 0.0;
    for (int64_t i = 0; i < n; ++i) v0n += v0h[i] * v0h[i];
    v0n = std::sqrt(v0n);
    if (v0n == 0.0) fail(MSVD_ERR_NUMERICAL, "lanczos_gk: starting vector is zero");
    if (truth && !truth->v_min) fail(MSVD_ERR_DIMENSION, "lanczos_gk: ground-truth vector length mismatch");
    if (n > kMaxCols) fail(MSVD_ERR_DIMENSION, "msvd: more than 2^20 columns is not supported by this build");
    const auto t_start = std::chrono::steady_clock::now();
    auto elapsed_ms = [&] {
        return timing ? std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count()
                      : 0.0;
    };

    const int gparts = op_parts(c, M);
    const int nblk = static_cast<int>(ceil_div(n, 64));  // reduce_g column blocks
    const int pm = static_cast<int>(ceil_div(ml > 0 ? ml : 1, kRowsPerCta));  // m-side row blocks
    const int pn = static_cast<int>(ceil_div(n, kRowsPerCta));
    const int N2 = 2 * iters;
    // device layout (doubles)
    const size_t szV = static_cast<size_t>(n) * (iters + 1), szU = static_cast<size_t>(ml) * iters;
    const size_t szG = static_cast<size_t>(gparts) * n + nblk;
    const size_t szPart = static_cast<size_t>(pm > pn ? pm : pn) * iters + pm;
    const size_t total = szV + szU + 2 * static_cast<size_t>(ml) + 4 * static_cast<size_t>(n) + szG + szPart +
                         3 * static_cast<size_t>(iters) + 6 * static_cast<size_t>(N2) + 16 + iters;
    DevBuf buf;
    MSVD_CUDA(cudaMalloc(&buf.p, sizeof(double) * total));
    double* base = static_cast<double*>(buf.p);
    double* Vb = base;
    double* Ub = Vb + szV;
    double* u = Ub + szU;          // m-side work vector
    double* w = u + 2 * ml;
    double* vest = w + n;
    double* tv = vest + n;
    double* cvec = tv + n;         // n >= iters: projection coefficients
    double* gpart = cvec + n;
    double* nrm = gpart + static_cast<size_t>(gparts) * n;
    double* part = gpart + szG;
    double* alpha = part + szPart;
    double* beta = alpha + iters;
    double* y = beta + iters;
    double* work = y + iters;
    double* sc = work + 6 * static_cast<size_t>(N2);  // [0] sumsq [2] theta [3] dot [4] |y_last| [5] alpha_{j-1}
    cudaStream_t s = c.stream;

    auto sumsq = [&](const double* x, int64_t len, bool sharded) {  // -> sc[0]
        const int np = static_cast<int>(ceil_div(len > 0 ? len : 1, kRowsPerCta));
        if (len > 0) {
            sumsq_parts_kernel<<<np, 256, 0, s>>>(x, len, part);
        } else {
            MSVD_CUDA(cudaMemsetAsync(part, 0, sizeof(double), s));
        }
        sum_parts_kernel<<<1, 256, 0, s>>>(part, len > 0 ? np : 1, sc);
        c.launches += 2;
        if (sharded) comm.allreduce_sum(sc, 1, s);
    };
    auto scale_norm = [&](const double* src, int64_t len, double* norm_out, double* dst) {
        scale_by_norm_kernel<<<static_cast<unsigned>(ceil_div(len > 0 ? len : 1, 256)), 256, 0, s>>>(src, len, sc,
                                                                                                     norm_out, dst);
        ++c.launches;
    };
    // two classical passes of x -= Q (Q^T x) against the first `cols` columns
    auto reorth = [&](const double* Q, int64_t ld, int64_t len, int cols, double* x, bool sharded) {
        if (cols <= 0) return;
        const int np = static_cast<int>(ceil_div(len > 0 ? len : 1, kRowsPerCta));
        for (int pass = 0; pass < 2; ++pass) {
            if (len > 0) {
                proj_parts_kernel<<<np, 256, 0, s>>>(Q, ld, len, cols, x, part);
                proj_sum_kernel<<<static_cast<unsigned>(ceil_div(cols, 256)), 256, 0, s>>>(part, np, cols, cvec);
                c.launches += 2;
            } else {
                MSVD_CUDA(cudaMemsetAsync(cvec, 0, sizeof(double) * cols, s));
            }
            if (sharded) comm.allreduce_sum(cvec, static_cast<size_t>(cols), s);
            if (len > 0) {
                qc_kernel<<<static_cast<unsigned>(ceil_div(len, 256)), 256, 0, s>>>(Q, ld, len, cols, cvec, x, 0);
                ++c.launches;
            }
        }
    };
    auto read = [&](double* h, const double* d, int cnt) {
        MSVD_CUDA(cudaMemcpyAsync(h, d, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s));
        MSVD_CUDA(cudaStreamSynchronize(s));
    };
    const bool sharded = comm.nranks() > 1;

    // v = v0 / ||v0|| (host norm above is validation only; the device scales)
    MSVD_CUDA(cudaMemcpyAsync(w, v0h, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    if (truth) MSVD_CUDA(cudaMemcpyAsync(tv, truth->v_min, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    sumsq(w, n, false);
    scale_norm(w, n, nullptr, Vb);

    OutCols out{};
    out.p[0] = u;
    op_apply(c, M, Vb, 1, out);  // u = A v
    long mva = 1, mvat = 0;
    sumsq(u, ml, sharded);
    double h[8];
    read(h, sc, 1);
    const double a1 = std::sqrt(h[0]);
    res->rows_count = 0;
    res->steps = 0;
    res->status = MSVD_LANCZOS_COMPLETED;
    auto finish = [&] {
        if (res->steps > 0) MSVD_CUDA(cudaMemcpyAsync(res->v, vest, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        if (res->v_basis && res->steps > 0)
            MSVD_CUDA(cudaMemcpyAsync(res->v_basis, Vb, sizeof(double) * n * res->steps, cudaMemcpyDeviceToHost, s));
        if (res->u_basis && res->steps > 0 && ml > 0)
            MSVD_CUDA(cudaMemcpyAsync(res->u_basis, Ub, sizeof(double) * ml * res->steps, cudaMemcpyDeviceToHost, s));
        MSVD_CUDA(cudaStreamSynchronize(s));
    };
    if (a1 == 0.0) {  // v0 is an exact null vector of A
        res->sigma_min = 0.0;
        MSVD_CUDA(cudaMemcpyAsync(res->v, Vb, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        res->status = MSVD_LANCZOS_INVARIANT_SUBSPACE;
        finish();
        return;
    }
    scale_norm(u, ml, alpha, Ub);  // alpha[0] = ||u||, U(:,0) = u / alpha
    double coeff = a1;

    const size_t bis_smem = sizeof(double) * 2 * static_cast<size_t>(N2);
    if (bis_smem > 48 * 1024) optin_smem(c, bidiag_min_kernel);
    for (int j = 1; j <= iters; ++j) {
        // w = A^T u_{j-1} - alpha_{j-1} v_{j-1}, reorthogonalized against V
        Cols T{};
        T.p[0] = Ub + static_cast<int64_t>(j - 1) * ml;
        const int np = op_adjoint(c, M, T, 1, gpart);
        launch_reduce_g(c, gpart, np, n, 1, nullptr, nullptr, 0, w, nrm, nblk);
        if (sharded) comm.allreduce_sum(w, static_cast<size_t>(n), s);
        ++mvat;
        axpy_neg_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, s>>>(Vb + (j - 1) * n, n, alpha + (j - 1), w);
        ++c.launches;
        reorth(Vb, n, n, j, w, false);
        sumsq(w, n, false);
        read(h, sc, 1);
        const double bj = std::sqrt(h[0]);
        coeff = std::max(coeff, bj);
        sqrt_store_kernel<<<1, 1, 0, s>>>(sc, beta + (j - 1));

        // smallest triplet of the j x j section, Ritz vector, telemetry
        BidiagArgs ba{alpha, beta, j, work, y, sc + 2};
        bidiag_min_kernel<<<1, kBisT, sizeof(double) * 2 * 2 * j, s>>>(ba);
        qc_kernel<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, s>>>(Vb, n, n, j, y, vest, 1);
        step_stats_kernel<<<1, 256, 0, s>>>(vest, truth ? tv : nullptr, n, y, alpha, j, sc + 3);
        c.launches += 4;
        read(h, sc, 6);
        const double theta = h[2];
        const double alpha_prev = h[5];
        msvd_record_row row{};
        row.iter = j;
        row.matvecs_a = mva;
        row.matvecs_at = mvat;
        row.wall_ms = elapsed_ms();
        row.theta = theta;
        row.resid = alpha_prev * bj * h[4];
        row.relerr = -1.0;
        row.sin_angle = -1.0;
        if (truth) {
            const double sn = truth->sigma_min;
            row.relerr = sn > 0.0 ? std::fabs(theta - sn) / sn : std::fabs(theta);
            const double cc = std::min(1.0, std::max(-1.0, h[3]));
            row.sin_angle = std::sqrt(std::max(0.0, 1.0 - cc * cc));
        }
        if (res->rows_count < res->rows_capacity && res->rows) res->rows[res->rows_count] = row;
        res->rows_count++;
        res->sigma_min = theta;
        res->steps = j;

        if (bj <= 64.0 * kEpsL * coeff) {
            res->status = MSVD_LANCZOS_INVARIANT_SUBSPACE;
            break;
        }
        if (j == iters) break;

        // v_j = w / beta; u = A v_j - beta u_{j-1}, reorthogonalized against U
        scale_norm(w, n, nullptr, Vb + static_cast<int64_t>(j) * n);  // sc[0] still holds ||w||^2
        op_apply(c, M, Vb + static_cast<int64_t>(j) * n, 1, out);
        ++mva;
        if (ml > 0) {
            axpy_neg_kernel<<<static_cast<unsigned>(ceil_div(ml, 256)), 256, 0, s>>>(Ub + (j - 1) * ml, ml,
                                                                                   beta + (j - 1), u);
            ++c.launches;
        }
        reorth(Ub, ml, ml, j, u, sharded);
        sumsq(u, ml, sharded);
        read(h, sc, 1);
        const double aj = std::sqrt(h[0]);
        coeff = std::max(coeff, aj);
        if (aj <= 64.0 * kEpsL * coeff) {
            res->status = MSVD_LANCZOS_INVARIANT_SUBSPACE;
            break;
        }
        scale_norm(u, ml, alpha + j, Ub + static_cast<int64_t>(j) * ml);
    }
    finish();
}

}  // namespace msvd
