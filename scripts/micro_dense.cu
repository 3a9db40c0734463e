// Micro-benchmark of the dense n-scale library calls the Cholesky-QR
// preconditioner route makes (csrc/precond_chol.cu), at the C2 sketch shape
// (d = 4000, n = 1000): which cuBLAS / cuSOLVER entry point is fastest for
// each step.  Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a
//   scripts/micro_dense.cu -lcublas -lcusolver -o build/micro_dense
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                         \
    do {                                                              \
        auto e__ = (x);                                               \
        if (e__ != 0) {                                               \
            std::printf("error %d at %s:%d\n", (int)e__, __FILE__, __LINE__); \
            std::exit(1);                                             \
        }                                                             \
    } while (0)

__global__ void fill(double* p, long n, unsigned seed) {
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (i < n) {
        unsigned x = (unsigned)i * 2654435761u + seed;
        x ^= x >> 13;
        x *= 0x5bd1e995u;
        x ^= x >> 15;
        p[i] = (x & 0xffff) / 65536.0 - 0.5;
    }
}

int main(int argc, char** argv) {
    const int d = argc > 1 ? atoi(argv[1]) : 4000, n = argc > 2 ? atoi(argv[2]) : 1000;
    double *SA, *G, *G2, *R, *Q, *W;
    CK(cudaMalloc(&SA, sizeof(double) * d * n));
    CK(cudaMalloc(&Q, sizeof(double) * d * n));
    CK(cudaMalloc(&G, sizeof(double) * n * n));
    CK(cudaMalloc(&G2, sizeof(double) * n * n));
    CK(cudaMalloc(&R, sizeof(double) * n * n));
    fill<<<(d * n + 255) / 256, 256>>>(SA, (long)d * n, 1);
    cublasHandle_t h;
    cusolverDnHandle_t s;
    CK(cublasCreate(&h));
    CK(cusolverDnCreate(&s));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    CK(cublasSetStream(h, st));
    CK(cusolverDnSetStream(s, st));
    int lw = 0;
    CK(cusolverDnDpotrf_bufferSize(s, CUBLAS_FILL_MODE_UPPER, n, G, n, &lw));
    CK(cudaMalloc(&W, sizeof(double) * (lw + 16)));
    int* info;
    CK(cudaMalloc(&info, sizeof(int)));
    cusolverDnParams_t prm;
    CK(cusolverDnCreateParams(&prm));
    size_t dws = 0, hws = 0;
    CK(cusolverDnXpotrf_bufferSize(s, prm, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, G, n, CUDA_R_64F, &dws, &hws));
    void* dw;
    CK(cudaMalloc(&dw, dws + 16));
    std::vector<char> hw(hws + 16);
    const double one = 1.0, zero = 0.0;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto fn) {
        for (int w = 0; w < 3; ++w) fn();
        cudaStreamSynchronize(st);
        cudaEventRecord(a, st);
        const int reps = 10;
        for (int r = 0; r < reps; ++r) fn();
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        std::printf("%-40s %8.3f ms\n", name, ms / reps);
    };
    timeit("dsyrk  G = SA^T SA", [&] {
        CK(cublasDsyrk(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, n, d, &one, SA, d, &zero, G, n));
    });
    timeit("dgemm  G = SA^T SA", [&] {
        CK(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, n, n, d, &one, SA, d, SA, d, &zero, G, n));
    });
    CK(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, n, n, d, &one, SA, d, SA, d, &zero, G, n));
    timeit("dpotrf (copy + factor)", [&] {
        CK(cudaMemcpyAsync(R, G, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
        CK(cusolverDnDpotrf(s, CUBLAS_FILL_MODE_UPPER, n, R, n, W, lw, info));
    });
    timeit("Xpotrf (copy + factor)", [&] {
        CK(cudaMemcpyAsync(R, G, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
        CK(cusolverDnXpotrf(s, prm, CUBLAS_FILL_MODE_UPPER, n, CUDA_R_64F, R, n, CUDA_R_64F, dw, dws, hw.data(), hws,
                            info));
    });
    timeit("copy n x n only", [&] {
        CK(cudaMemcpyAsync(R, G, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
    });
    timeit("dtrsm  Q = SA R^-1 (right)", [&] {
        CK(cublasDtrsm(h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, d, n, &one, R,
                       n, Q, d));
    });
    timeit("dtrmm  Q = SA R (right, out of place)", [&] {
        CK(cublasDtrmm(h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, d, n, &one, R,
                       n, SA, d, Q, d));
    });
    timeit("dgemm  Q = SA R (d x n x n)", [&] {
        CK(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, d, n, n, &one, SA, d, R, n, &zero, Q, d));
    });
    timeit("dtrsm  R^-1 (left, B = n x n)", [&] {
        CK(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n, &one, R, n,
                       G2, n));
    });
    size_t tdws = 0, thws = 0;
    CK(cusolverDnXtrtri_bufferSize(s, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, G2, n, &tdws,
                                   &thws));
    void* tdw;
    CK(cudaMalloc(&tdw, tdws + 16));
    std::vector<char> thw(thws + 16);
    timeit("Xtrtri R^-1 (copy + invert)", [&] {
        CK(cudaMemcpyAsync(G2, R, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
        CK(cusolverDnXtrtri(s, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, G2, n, tdw, tdws,
                            thw.data(), thws, info));
    });
    timeit("dgemm  n x n x n", [&] {
        CK(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, G, n, R, n, &zero, G2, n));
    });
    timeit("dgemm  n x 24 x n", [&] {
        CK(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, 24, n, &one, G, n, R, n, &zero, G2, n));
    });
    timeit("dgeqrf+dorgqr n x 24", [&] {
        int lq = 0;
        CK(cusolverDnDgeqrf_bufferSize(s, n, 24, G2, n, &lq));
        CK(cusolverDnDgeqrf(s, n, 24, G2, n, R, W, lw, info));
        CK(cusolverDnDorgqr(s, n, 24, 24, G2, n, R, W, lw, info));
    });
    std::printf("done\n");
    return 0;
}
