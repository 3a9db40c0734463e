// CSR operator on the device (csr.hpp / csr.cpp,
// operator.hpp:58-74 CsrOperator, sketch.cpp:97-118).
//
// The same solver passes as the dense path, over a borrowed device CSR
// (row offsets int64, column indices int32 or int64, values f64):
//
//  * attach validates the structure exactly as CsrMatrix::validate does
//    (csr.cpp:9-31: endpoints, nondecreasing offsets, column range, strictly
//    increasing columns, finiteness; first failing row reported) and builds
//    the transpose (CSC) once, by a stable radix sort of the nonzeros on their
//    column, so that A^T y is a deterministic gather instead of the
//    reference's scatter (csr.cpp:46-57) -- operator.hpp:10-14 requires the
//    same output bits for the same input.
//  * A W (b <= 8 columns): G lanes per row (G from the mean row length),
//    W gathered through L1/L2, one pass over the nonzeros for all b columns.
//  * A^T Y: one warp per (column, segment) of the CSC, per-segment partials
//    [S][b][n] summed in fixed order by the solver's reduce kernel.
//  * S A: bit-identical to sketch_apply(S, CsrMatrix).  The (sketch row,
//    source row) lists are the dense path's (radix-sorted, source rows
//    ascending); one warp per sketch row keeps the n running sums in shared
//    memory and adds each source row's nonzeros in order (distinct columns
//    within a row, so lanes never collide), unfused multiply/add.
//  * column norms in the reference's accumulation order (per column,
//    ascending rows: operator.cpp:98-104).
//
// Algorithmic bytes per pass: 8 (value) + 4 or 8 (index) per nonzero, plus
// 8 (b = 1) per row for the offsets; the solver's skinny vectors are extra.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "msvd_internal.h"

namespace msvd {
namespace {

constexpr int kT = 256;

template <typename Idx>
__device__ __forceinline__ int64_t ld_idx(const Idx* p, int64_t k) {
    return static_cast<int64_t>(__ldg(p + k));
}

// ---------------------------------------------------------------- validate
// per row: the first structural defect, as a key ordered like the reference's
// row-by-row scan: ((row << 32 | where) << 1 | kind); where 0 = the offsets
// check, k - start + 1 = entry k.  kind 0 = range / offsets, 1 = ordering.
template <typename Idx>
__global__ void csr_validate_kernel(const int64_t* rp, const Idx* ci, const double* v, int64_t m, int64_t n,
                                    int64_t nnz, unsigned long long* first_bad, int* nonfinite) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t s = rp[i], e = rp[i + 1];
    unsigned long long key = ~0ull;
    if (s > e) {
        key = (static_cast<unsigned long long>(i) << 33) | 0ull;  // not nondecreasing
    } else {
        for (int64_t k = s; k < e && k < nnz; ++k) {
            const int64_t j = ld_idx(ci, k);
            const unsigned long long where = static_cast<unsigned long long>(k - s + 1);
            if (j < 0 || j >= n) {
                key = ((static_cast<unsigned long long>(i) << 32 | where) << 1) | 0ull;
                break;
            }
            if (k > s && ld_idx(ci, k - 1) >= j) {
                key = ((static_cast<unsigned long long>(i) << 32 | where) << 1) | 1ull;
                break;
            }
        }
        for (int64_t k = s; k < e && k < nnz; ++k)
            if (!isfinite(v[k])) {
                atomicOr(nonfinite, 1);
                break;
            }
    }
    if (key != ~0ull) atomicMin(first_bad, key);
}

// ------------------------------------------------------------ transpose
template <typename Idx>
__global__ void csc_keys_kernel(const Idx* ci, int64_t nnz, uint32_t* keys, uint32_t* perm) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    keys[k] = static_cast<uint32_t>(ld_idx(ci, k));
    perm[k] = static_cast<uint32_t>(k);
}
__global__ void row_of_kernel(const int64_t* rp, int64_t m, uint32_t* rowof) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) rowof[k] = static_cast<uint32_t>(i);
}
__global__ void csc_fill_kernel(const uint32_t* perm, const uint32_t* rowof, const double* v, int64_t nnz,
                                uint32_t* ri, double* cv) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    const uint32_t p = perm[q];
    ri[q] = rowof[p];
    cv[q] = v[p];
}
__global__ void csc_ptr_kernel(const uint32_t* keys, int64_t nnz, int64_t n, int64_t* cp) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j > n) return;
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (static_cast<int64_t>(keys[mid]) < j) lo = mid + 1;
        else hi = mid;
    }
    cp[j] = lo;
}

// ------------------------------------------------------------- Y = A W
template <int G, int B, typename Idx>
__global__ void __launch_bounds__(kT) csr_spmm_kernel(const int64_t* __restrict__ rp, const Idx* __restrict__ ci,
                                                      const double* __restrict__ v, int64_t m,
                                                      const double* __restrict__ W, int64_t n, OutCols out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t row = t / G;
    const int sub = static_cast<int>(t % G);
    double acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) acc[c] = 0.0;
    if (row < m) {
        const int64_t e = rp[row + 1];
        for (int64_t k = rp[row] + sub; k < e; k += G) {
            const double a = __ldg(v + k);
            const int64_t j = ld_idx(ci, k);
#pragma unroll
            for (int c = 0; c < B; ++c) acc[c] += a * __ldg(W + j + c * n);
        }
    }
#pragma unroll
    for (int c = 0; c < B; ++c)
#pragma unroll
        for (int o = G / 2; o >= 1; o >>= 1) acc[c] += __shfl_xor_sync(kFull, acc[c], o);
    if (row < m && sub == 0)
#pragma unroll
        for (int c = 0; c < B; ++c) out.p[c][row] = acc[c];
}

// ------------------------------------------------------------ G = A^T Y
// Gpart[(s * b + c) * n + j] = sum over segment s of column j of the CSC
template <int B>
__global__ void __launch_bounds__(kT) csc_gather_kernel(const int64_t* __restrict__ cp,
                                                        const uint32_t* __restrict__ ri,
                                                        const double* __restrict__ cv, int64_t n, Cols Y,
                                                        int S, double* Gpart) {
    constexpr int b = B;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j = static_cast<int64_t>(blockIdx.x) * (kT / 32) + warp;
    const int s = blockIdx.y;
    if (j >= n) return;
    const int64_t c0 = cp[j], len = cp[j + 1] - c0;
    const int64_t q0 = c0 + (len * s) / S, q1 = c0 + (len * (s + 1)) / S;
    double acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) acc[c] = 0.0;
    constexpr int U = 4;  // four entries per lane in flight: the row-index -> Y loads overlap
    int64_t q = q0 + lane;
    for (; q + 32 * (U - 1) < q1; q += 32 * U) {
        double a[U];
        uint32_t r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a[u] = __ldg(cv + q + 32 * u);
            r[u] = __ldg(ri + q + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < B; ++c) acc[c] += a[u] * __ldg(Y.p[c] + r[u]);
    }
    for (; q < q1; q += 32) {
        const double a = __ldg(cv + q);
        const uint32_t r = __ldg(ri + q);
#pragma unroll
        for (int c = 0; c < B; ++c) acc[c] += a * __ldg(Y.p[c] + r);
    }
#pragma unroll
    for (int c = 0; c < B; ++c) {
        const double t = warp_sum(acc[c]);
        if (lane == 0) Gpart[(static_cast<int64_t>(s) * b + c) * n + j] = t;
    }
}

// column sums of squares in the reference's order (ascending rows)
__global__ void csc_colsq_kernel(const int64_t* cp, const double* cv, int64_t n, double* out) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int64_t q = cp[j]; q < cp[j + 1]; ++q) s = __dadd_rn(s, __dmul_rn(cv[q], cv[q]));
    out[j] = s;
}

// --------------------------------------------------------------- S A
// one warp per sketch row; running sums of its n columns in shared memory,
// or (GLOBAL: rows wider than shared memory holds) in the sketch row itself
// (SA zeroed by the caller; stride d) -- the same per-column order either way
template <typename Idx, bool GLOBAL>
__global__ void __launch_bounds__(kT) csr_sketch_kernel(const int64_t* __restrict__ rp, const Idx* __restrict__ ci,
                                                        const double* __restrict__ v, int64_t n, int64_t d,
                                                        const int64_t* offs, const uint32_t* vals, double val,
                                                        double* SA) {
    extern __shared__ double acc_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t s = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
    if (s >= d) return;
    double* acc = GLOBAL ? SA + s : acc_all + static_cast<int64_t>(warp) * n;
    const int64_t as = GLOBAL ? d : 1;
    if (!GLOBAL)
        for (int64_t j = lane; j < n; j += 32) acc[j] = 0.0;
    __syncwarp();
    const int64_t e0 = offs[s], e1 = offs[s + 1];
    for (int64_t e = e0; e < e1; ++e) {
        const uint32_t w = vals[e];
        const int64_t r = static_cast<int64_t>(w & 0x7fffffffu);
        const double svv = (w >> 31) ? -val : val;
        const int64_t k1 = rp[r + 1];
        for (int64_t k = rp[r] + lane; k < k1; k += 32) {
            const int64_t j = ld_idx(ci, k) * as;
            acc[j] = __dadd_rn(acc[j], __dmul_rn(svv, v[k]));
        }
        __syncwarp();
    }
    if (!GLOBAL)
        for (int64_t j = lane; j < n; j += 32) SA[s + j * d] = acc[j];
}

// dense row-major rows [row0, row0 + m) of an (m_global x n) zero matrix
template <typename Idx>
__global__ void csr_scatter_kernel(const int64_t* rp, const Idx* ci, const double* v, int64_t m, int64_t n,
                                   double* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) out[i * n + ld_idx(ci, k)] = v[k];
}

unsigned grid_for(int64_t threads) { return static_cast<unsigned>(ceil_div(threads > 0 ? threads : 1, kT)); }

template <typename F>
void with_idx(const msvd_matrix& M, F&& f) {
    if (M.csr_idx64) f(static_cast<const int64_t*>(M.csr_ci));
    else f(static_cast<const int32_t*>(M.csr_ci));
}

}  // namespace

void csr_prepare(Ctx& c, msvd_matrix& M) {
    const int64_t m = M.m_local, n = M.n, nnz = M.csr_nnz;
    cudaStream_t s = c.stream;
    // csr.cpp:9-31, in order: dimensions, endpoints, per-row structure, values
    if (m < 0 || n < 0) fail(MSVD_ERR_DIMENSION, "CsrMatrix: negative dimension");
    if (nnz < 0) fail(MSVD_ERR_DIMENSION, "CsrMatrix: col_indices and values length mismatch");
    if (nnz >= (1LL << 32) - 1 || m >= (1LL << 31))
        fail(MSVD_ERR_DIMENSION, "msvd: CSR operator limited to < 2^31 rows and < 2^32 nonzeros per rank");
    int64_t ends[2] = {0, 0};
    MSVD_CUDA(cudaMemcpyAsync(&ends[0], M.csr_rp, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MSVD_CUDA(cudaMemcpyAsync(&ends[1], M.csr_rp + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MSVD_CUDA(cudaStreamSynchronize(s));
    if (ends[0] != 0 || ends[1] != nnz)
        fail(MSVD_ERR_DIMENSION, "CsrMatrix: row_offsets endpoints inconsistent with nnz");
    // owned: [first_bad u64 | nonfinite int | pad] [cp (n+1)] [ri nnz] [cv nnz]
    const size_t head = 256;
    const size_t cpb = ((sizeof(int64_t) * (n + 1) + 255) / 256) * 256;
    const size_t rib = ((sizeof(uint32_t) * (nnz > 0 ? nnz : 1) + 255) / 256) * 256;
    const size_t cvb = ((sizeof(double) * (nnz > 0 ? nnz : 1) + 255) / 256) * 256;
    MSVD_CUDA(cudaMalloc(&M.csr_owned, head + cpb + rib + cvb));
    unsigned char* base = static_cast<unsigned char*>(M.csr_owned);
    auto* first_bad = reinterpret_cast<unsigned long long*>(base);
    int* nonfinite = reinterpret_cast<int*>(base + 8);
    M.csc_cp = reinterpret_cast<int64_t*>(base + head);
    M.csc_ri = reinterpret_cast<uint32_t*>(base + head + cpb);
    M.csc_cv = reinterpret_cast<double*>(base + head + cpb + rib);
    MSVD_CUDA(cudaMemsetAsync(first_bad, 0xff, 8, s));
    MSVD_CUDA(cudaMemsetAsync(nonfinite, 0, 4, s));
    if (m > 0)
        with_idx(M, [&](auto* ci) {
            csr_validate_kernel<<<grid_for(m), kT, 0, s>>>(M.csr_rp, ci, M.csr_v, m, n, nnz, first_bad, nonfinite);
        });
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    unsigned long long hb = 0;
    int hn = 0;
    MSVD_CUDA(cudaMemcpyAsync(&hb, first_bad, 8, cudaMemcpyDeviceToHost, s));
    MSVD_CUDA(cudaMemcpyAsync(&hn, nonfinite, 4, cudaMemcpyDeviceToHost, s));
    MSVD_CUDA(cudaStreamSynchronize(s));
    if (hb != ~0ull) {
        const int64_t row = static_cast<int64_t>(hb >> 33);
        const unsigned long long where = (hb >> 1) & 0xffffffffull;
        const std::string r = std::to_string(row);
        if (where == 0) fail(MSVD_ERR_DIMENSION, "CsrMatrix: row_offsets not nondecreasing at row " + r);
        if ((hb & 1ull) == 0) fail(MSVD_ERR_DIMENSION, "CsrMatrix: column index out of range in row " + r);
        fail(MSVD_ERR_DIMENSION, "CsrMatrix: column indices not strictly increasing in row " + r);
    }
    if (hn) fail(MSVD_ERR_NUMERICAL, "CsrMatrix: non-finite value");

    // transpose: stable sort of the nonzeros on their column
    if (nnz > 0) {
        int bits = 1;
        while ((1LL << bits) < n) ++bits;
        size_t temp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<uint32_t*>(nullptr),
                                        static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                        static_cast<uint32_t*>(nullptr), static_cast<int>(nnz), 0, bits, s);
        const size_t arr = ((sizeof(uint32_t) * nnz + 255) / 256) * 256;
        unsigned char* t = static_cast<unsigned char*>(c.ensure_scratch(5 * arr + temp + 256));
        uint32_t* k_in = reinterpret_cast<uint32_t*>(t);
        uint32_t* p_in = reinterpret_cast<uint32_t*>(t + arr);
        uint32_t* k_out = reinterpret_cast<uint32_t*>(t + 2 * arr);
        uint32_t* p_out = reinterpret_cast<uint32_t*>(t + 3 * arr);
        uint32_t* rowof = reinterpret_cast<uint32_t*>(t + 4 * arr);
        with_idx(M, [&](auto* ci) { csc_keys_kernel<<<grid_for(nnz), kT, 0, s>>>(ci, nnz, k_in, p_in); });
        MSVD_CUDA(cub::DeviceRadixSort::SortPairs(t + 5 * arr, temp, k_in, k_out, p_in, p_out, static_cast<int>(nnz),
                                                  0, bits, s));
        row_of_kernel<<<grid_for(m), kT, 0, s>>>(M.csr_rp, m, rowof);
        csc_fill_kernel<<<grid_for(nnz), kT, 0, s>>>(p_out, rowof, M.csr_v, nnz, M.csc_ri, M.csc_cv);
        csc_ptr_kernel<<<grid_for(n + 1), kT, 0, s>>>(k_out, nnz, n, M.csc_cp);
        MSVD_CUDA(cudaGetLastError());
        c.launches += 5;
    } else {
        MSVD_CUDA(cudaMemsetAsync(M.csc_cp, 0, sizeof(int64_t) * (n + 1), s));
    }
    // lanes per row from the mean row length
    const double mean = m > 0 ? static_cast<double>(nnz) / static_cast<double>(m) : 0.0;
    // ~4 or more nonzeros per lane (measured at 10 per row: 2 lanes 4.6 TB/s,
    // 4 lanes 3.4, 16 lanes 1.2)
    int g = 1;
    while (g < 32 && 4 * (2 * g) <= mean) g <<= 1;
    if (const char* e = std::getenv("MSVD_CSR_LANES")) g = std::max(1, std::min(32, std::atoi(e)));
    M.csr_lanes = g;
    MSVD_CUDA(cudaStreamSynchronize(s));
}

void csr_release(msvd_matrix& M) {
    if (M.csr_owned) cudaFree(M.csr_owned);
    M.csr_owned = nullptr;
}

void csr_apply(Ctx& c, const msvd_matrix& M, const double* W, int b, OutCols out) {
    ProfScope prof(c, kProfApply);
    const int64_t m = M.m_local;
    if (m == 0) return;
    const int g = M.csr_lanes;
    const unsigned grid = grid_for(m * g);
    with_idx(M, [&](auto* ci) {
        using Idx = std::remove_const_t<std::remove_pointer_t<decltype(ci)>>;
        auto go = [&](auto gtag) {
            constexpr int G = decltype(gtag)::value;
            switch (b) {
                case 1: csr_spmm_kernel<G, 1, Idx><<<grid, kT, 0, c.stream>>>(M.csr_rp, ci, M.csr_v, m, W, M.n, out); break;
                case 2: csr_spmm_kernel<G, 2, Idx><<<grid, kT, 0, c.stream>>>(M.csr_rp, ci, M.csr_v, m, W, M.n, out); break;
                case 3: csr_spmm_kernel<G, 3, Idx><<<grid, kT, 0, c.stream>>>(M.csr_rp, ci, M.csr_v, m, W, M.n, out); break;
                case 4: csr_spmm_kernel<G, 4, Idx><<<grid, kT, 0, c.stream>>>(M.csr_rp, ci, M.csr_v, m, W, M.n, out); break;
                case 5: csr_spmm_kernel<G, 5, Idx><<<grid, kT, 0, c.stream>>>(M.csr_rp, ci, M.csr_v, m, W, M.n, out); break;
                case 6: csr_spmm_kernel<G, 6, Idx><<<grid, kT, 0, c.stream>>>(M.csr_rp, ci, M.csr_v, m, W, M.n, out); break;
                case 7: csr_spmm_kernel<G, 7, Idx><<<grid, kT, 0, c.stream>>>(M.csr_rp, ci, M.csr_v, m, W, M.n, out); break;
                default: csr_spmm_kernel<G, 8, Idx><<<grid, kT, 0, c.stream>>>(M.csr_rp, ci, M.csr_v, m, W, M.n, out); break;
            }
        };
        switch (g) {
            case 1: go(std::integral_constant<int, 1>{}); break;
            case 2: go(std::integral_constant<int, 2>{}); break;
            case 4: go(std::integral_constant<int, 4>{}); break;
            case 8: go(std::integral_constant<int, 8>{}); break;
            case 16: go(std::integral_constant<int, 16>{}); break;
            default: go(std::integral_constant<int, 32>{}); break;
        }
    });
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

int csr_parts(const Ctx& c, const msvd_matrix& M) {
    const int64_t n = M.n > 0 ? M.n : 1;
    const int64_t target = static_cast<int64_t>(c.num_sms) * 256;  // 4 waves of resident warps: gathers in flight
    int64_t S = ceil_div(target, n);
    const int64_t mean = M.csr_nnz / n;
    S = std::min<int64_t>(S, std::max<int64_t>(1, mean / 128));
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(S, 64)));
}

int csr_adjoint_parts(Ctx& c, const msvd_matrix& M, Cols Y, int b, double* Gpart) {
    ProfScope prof(c, kProfGram);
    const int S = csr_parts(c, M);
    dim3 grid(static_cast<unsigned>(ceil_div(M.n, kT / 32)), static_cast<unsigned>(S));
    switch (b) {
        case 1: csc_gather_kernel<1><<<grid, kT, 0, c.stream>>>(M.csc_cp, M.csc_ri, M.csc_cv, M.n, Y, S, Gpart); break;
        case 2: csc_gather_kernel<2><<<grid, kT, 0, c.stream>>>(M.csc_cp, M.csc_ri, M.csc_cv, M.n, Y, S, Gpart); break;
        case 3: csc_gather_kernel<3><<<grid, kT, 0, c.stream>>>(M.csc_cp, M.csc_ri, M.csc_cv, M.n, Y, S, Gpart); break;
        case 4: csc_gather_kernel<4><<<grid, kT, 0, c.stream>>>(M.csc_cp, M.csc_ri, M.csc_cv, M.n, Y, S, Gpart); break;
        case 5: csc_gather_kernel<5><<<grid, kT, 0, c.stream>>>(M.csc_cp, M.csc_ri, M.csc_cv, M.n, Y, S, Gpart); break;
        case 6: csc_gather_kernel<6><<<grid, kT, 0, c.stream>>>(M.csc_cp, M.csc_ri, M.csc_cv, M.n, Y, S, Gpart); break;
        case 7: csc_gather_kernel<7><<<grid, kT, 0, c.stream>>>(M.csc_cp, M.csc_ri, M.csc_cv, M.n, Y, S, Gpart); break;
        default: csc_gather_kernel<8><<<grid, kT, 0, c.stream>>>(M.csc_cp, M.csc_ri, M.csc_cv, M.n, Y, S, Gpart); break;
    }
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    return S;
}

void csr_colsq(Ctx& c, const msvd_matrix& M, double* out) {
    csc_colsq_kernel<<<grid_for(M.n), kT, 0, c.stream>>>(M.csc_cp, M.csc_cv, M.n, out);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void csr_sketch(Ctx& c, const msvd_matrix& M, int64_t d, int zeta, uint64_t seed, double* SA) {
    ProfScope prof(c, kProfSketch);
    const int64_t n = M.n;
    if (M.m_local == 0) {
        MSVD_CUDA(cudaMemsetAsync(SA, 0, sizeof(double) * d * n, c.stream));
        return;
    }
    const SketchLists L = sketch_prepare(c, M.m_local, M.row0, d, zeta, seed, M.m_local);
    int warps = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, 65536 / (8 * n))));
    const size_t smem = sizeof(double) * n * warps;
    const bool global = smem + 1024 > c.smem_optin;  // a row wider than shared memory: sums in SA
    if (global) {
        warps = 8;
        MSVD_CUDA(cudaMemsetAsync(SA, 0, sizeof(double) * d * n, c.stream));
    }
    with_idx(M, [&](auto* ci) {
        using Idx = std::remove_const_t<std::remove_pointer_t<decltype(ci)>>;
        if (global) {
            csr_sketch_kernel<Idx, true><<<static_cast<unsigned>(ceil_div(d, warps)), 32 * warps, 0, c.stream>>>(
                M.csr_rp, ci, M.csr_v, n, d, L.offs, L.vals, L.val, SA);
            return;
        }
        auto kern = csr_sketch_kernel<Idx, false>;
        if (smem > 48 * 1024) optin_smem(c, kern);
        kern<<<static_cast<unsigned>(ceil_div(d, warps)), 32 * warps, smem, c.stream>>>(M.csr_rp, ci, M.csr_v, n, d,
                                                                                        L.offs, L.vals, L.val, SA);
    });
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

void csr_scatter_dense(Ctx& c, const msvd_matrix& M, double* out_rows) {
    if (M.m_local == 0) return;
    with_idx(M, [&](auto* ci) {
        csr_scatter_kernel<<<grid_for(M.m_local), kT, 0, c.stream>>>(M.csr_rp, ci, M.csr_v, M.m_local, M.n, out_rows);
    });
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

}  // namespace msvd
