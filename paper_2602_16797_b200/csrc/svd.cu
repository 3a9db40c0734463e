// Randomized preconditioner factorization (precond.cpp:11-36).
//
// dense_svd(SA) in the reference is Householder QR (d x n -> n x n R) then
// one-sided Jacobi on R.  Here the n-scale factorization runs on the device
// with cuSOLVER (allowed by the north star): geqrf reduces the tall sketch,
// then an SVD of R (gesvdp, the polar-decomposition SVD, by default; MSVD_SVD=gesvd|gesvdj|gesvdp selects).
// A small kernel then applies the reference's conventions: descending order,
// each right vector signed so its largest-magnitude entry is positive
// (svd.cpp:232-248), and the sqrt(n) u sigma_1 floor (precond.cpp:26-34).
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

}  // namespace

void precond_build_dev(Ctx& c, const double* SA, int64_t rows, int64_t n, double* Vcol, double* Vrow, double* sig,
                       double* sigma_max, int64_t* nfloor) {
    if (n < 1) fail(MSVD_ERR_DIMENSION, "build_preconditioner: empty sketch");
    if (rows < n) fail(MSVD_ERR_DIMENSION, "build_preconditioner: sketch has fewer rows than columns");
    ProfScope prof(c, kProfSvd);
    if (!c.solver) {
        MSVD_SOLVER(cusolverDnCreate(&c.solver));
    }
    MSVD_SOLVER(cusolverDnSetStream(c.solver, c.stream));
    const char* algo_env = std::getenv("MSVD_SVD");
    const std::string algo = algo_env ? algo_env : "gesvd";
    const int in = static_cast<int>(n), ir = static_cast<int>(rows);

    // ctx-owned workspace (grown on demand, reused across solves):
    // work (rows x n) | R (n x n) | V (n x n) | tau (n) | out2 (4) | info (4 ints)
    const size_t wbytes = sizeof(double) * static_cast<size_t>(rows) * n;
    const size_t nn = sizeof(double) * static_cast<size_t>(n) * n;
    const size_t need = wbytes + 2 * nn + sizeof(double) * (n + 8) + 64;
    if (need > c.svd_ws_bytes) {
        if (c.svd_ws) MSVD_CUDA(cudaFree(c.svd_ws));
        c.svd_ws = nullptr;
        MSVD_CUDA(cudaMalloc(&c.svd_ws, need));
        c.svd_ws_bytes = need;
    }
    double* work = static_cast<double*>(c.svd_ws);
    double* R = work + static_cast<size_t>(rows) * n;
    double* V = R + static_cast<size_t>(n) * n;
    double* tau = V + static_cast<size_t>(n) * n;
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
        } else if (algo == "gesvdp") {
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
