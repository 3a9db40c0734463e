// Randomized preconditioner factorization (precond.cpp:11-36).
//
// dense_svd(SA) in the reference is Householder QR (d x n -> n x n R) then
// one-sided Jacobi on R.  Here the n-scale factorization runs on the device
// with cuSOLVER (allowed by the north star): geqrf reduces the tall sketch,
// then an SVD of R.  Default ("polar"): cuSOLVER's QDWH polar SVD (gesvdp,
// the fastest on B200) followed by a Jacobi-accurate refinement of the
// singular triplets it cannot resolve (refine_tail below).  MSVD_SVD =
// gesvd | gesvdj | gesvdp | polar selects.
// A small kernel then applies the reference's conventions: descending order,
// each right vector signed so its largest-magnitude entry is positive
// (svd.cpp:232-248), and the sqrt(n) u sigma_1 floor (precond.cpp:26-34).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "msvd_internal.h"

namespace msvd {

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
// sign-fixed Vcol (column-major) and Vrow (row-major) copies.
__global__ void signfix_kernel(const double* Vin, int vt_layout, int64_t n, double* Vcol, double* Vrow) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    auto at = [&](int64_t i) { return vt_layout ? Vin[j + i * n] : Vin[i + j * n]; };
    int64_t imax = 0;
    double amax = -1.0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = fabs(at(i));
        if (a > amax) {
            amax = a;
            imax = i;
        }
    }
    const double s = at(imax) < 0.0 ? -1.0 : 1.0;
    for (int64_t i = 0; i < n; ++i) {
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

// defensive: enforce descending order (cuSOLVER returns sorted values; ties keep order)
__global__ void check_sorted_kernel(const double* sig, int64_t n, int* flag) {
    for (int64_t j = 1; j < n; ++j)
        if (sig[j] > sig[j - 1]) {
            *flag = 1000 + static_cast<int>(j);
            return;
        }
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
    const std::string algo = algo_env ? algo_env : "polar";
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
    MSVD_CUDA(cudaMemcpyAsync(work, SA, wbytes, cudaMemcpyDeviceToDevice, c.stream));
    int vt_layout = 0;
    try {
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
        check_sorted_kernel<<<1, 1, 0, c.stream>>>(sig, n, info + 2);
        signfix_kernel<<<static_cast<unsigned>(ceil_div(n, 128)), 128, 0, c.stream>>>(V, vt_layout, n, Vcol, Vrow);
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
