// SparseStack sketch S A (SURVEY 2.3 K1; sketch.cpp:36-60, :75-95).
//
// S is never stored: each row r of A regenerates its zeta (position, sign)
// pairs from SplitMix64(seed, row0 + r), exactly as build_sparsestack keys a
// column of S.  The scatter  SA[blk*k + pos] += sign * zeta^-1/2 * A[r, :]  is
// turned into a deterministic gather: the (sketch row, source row) pairs are
// radix-sorted by sketch row (stable, so source rows stay ascending), and one
// CTA per sketch row sums its source rows in that order with unfused
// multiply/add -- the reference's accumulation order, so on one rank SA is
// bit-identical to sketch_apply(S, A).
#include <cstdlib>

#include <cub/cub.cuh>

#include "common.cuh"
#include "msvd_internal.h"

namespace msvd {

namespace {

// next_below without modulo bias (rng.hpp:27-32)
__device__ __forceinline__ uint64_t below(uint64_t& s, uint64_t bound) {
    const uint64_t lim = UINT64_MAX - UINT64_MAX % bound;
    uint64_t x;
    do {
        s += kGolden;
        x = sm_mix(s);
    } while (x >= lim);
    return x % bound;
}

// one thread per local row: zeta (sketch row, signed source row) pairs
__global__ void keys_kernel(int64_t m, int64_t row0, int64_t d, int zeta, uint64_t seed, uint32_t* keys,
                            uint32_t* vals, uint32_t* pos_out, int8_t* sgn_out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= m) return;
    uint64_t s = sm_keyed_state(seed, static_cast<uint64_t>(row0 + r));
    const uint64_t blk = static_cast<uint64_t>(d / zeta);
    for (int k = 0; k < zeta; ++k) {
        const uint32_t pos = static_cast<uint32_t>(below(s, blk));
        s += kGolden;
        const bool neg = (sm_mix(s) >> 63) != 0;
        const int64_t at = r * zeta + k;
        if (keys) {
            keys[at] = static_cast<uint32_t>(k * blk + pos);
            vals[at] = static_cast<uint32_t>(r) | (neg ? 0x80000000u : 0u);
        }
        if (pos_out) {
            pos_out[at] = pos;
            sgn_out[at] = neg ? -1 : 1;
        }
    }
}

// offs[s] = first index with key >= s (binary search), s in [0, d]
__global__ void offsets_kernel(const uint32_t* keys, int64_t cnt, int64_t d, int64_t* offs) {
    const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s > d) return;
    int64_t lo = 0, hi = cnt;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (static_cast<int64_t>(keys[mid]) < s) lo = mid + 1;
        else hi = mid;
    }
    offs[s] = lo;
}

constexpr int kGatherT = 256;
constexpr int kGatherUnroll = 4;

// bounds[c * (d+1) + s] = first entry of sketch row s whose source row is
// >= c * step (binary search; rows ascend within a segment); c in [0, nch]
__global__ void bounds_kernel(const int64_t* offs, const uint32_t* vals, int64_t d, int64_t step, int64_t nch,
                              int64_t* bounds) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= (nch + 1) * d) return;
    const int64_t c = i / d, s = i - c * d;
    int64_t lo = offs[s], hi = offs[s + 1];
    const int64_t bound = c * step;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (static_cast<int64_t>(vals[mid] & 0x7fffffffu) < bound) lo = mid + 1;
        else hi = mid;
    }
    bounds[c * (d + 1) + s] = lo;
}

// Row-chunked gather: adds the contributions of source rows [r_lo, r_hi) of
// sketch row s to SAr[s, :] (ROW-major d x n, so the read-modify-write of the
// running sums is coalesced), continuing each sum in source-row order.
// Launched chunk by chunk in row order, so the sum is the reference's
// sequential one bit for bit, while each chunk of A (~48 MB) is fetched from
// HBM once and its zeta re-reads hit L2.
__global__ void __launch_bounds__(kGatherT) gather_chunk_kernel(const double* A, int64_t ld, int n, int64_t d,
                                                                const int64_t* bounds, const uint32_t* vals,
                                                                double val, double* SA, DevState* st, int vec,
                                                                int64_t chunk) {
    const int64_t s = blockIdx.x;
    const int64_t e0 = bounds[chunk * (d + 1) + s], e1 = bounds[(chunk + 1) * (d + 1) + s];
    if (e0 == e1) return;
    const int npairs = (n + 1) >> 1;
    bool finite = true;
    for (int pi = threadIdx.x; pi < npairs; pi += kGatherT) {
        const int c0 = 2 * pi;
        const bool has1 = c0 + 1 < n;
        double* o0 = SA + s * n + c0;
        double acc0 = *o0;
        double acc1 = has1 ? o0[1] : 0.0;
        int64_t e = e0;
        for (; e + kGatherUnroll <= e1; e += kGatherUnroll) {
            double x0[kGatherUnroll], x1[kGatherUnroll], sv[kGatherUnroll];
#pragma unroll
            for (int u = 0; u < kGatherUnroll; ++u) {
                const uint32_t v = __ldg(vals + e + u);
                const int64_t r = v & 0x7fffffffu;
                sv[u] = (v >> 31) ? -val : val;
                const double* row = A + r * ld + c0;
                if (vec && has1) {
                    const double2 x = __ldg(reinterpret_cast<const double2*>(row));
                    x0[u] = x.x;
                    x1[u] = x.y;
                } else {
                    x0[u] = __ldg(row);
                    x1[u] = has1 ? __ldg(row + 1) : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < kGatherUnroll; ++u) {
                acc0 = __dadd_rn(acc0, __dmul_rn(sv[u], x0[u]));
                acc1 = __dadd_rn(acc1, __dmul_rn(sv[u], x1[u]));
                finite = finite && isfinite(x0[u]) && isfinite(x1[u]);
            }
        }
        for (; e < e1; ++e) {
            const uint32_t v = __ldg(vals + e);
            const int64_t r = v & 0x7fffffffu;
            const double svv = (v >> 31) ? -val : val;
            const double* row = A + r * ld + c0;
            const double x0 = __ldg(row);
            const double x1 = has1 ? __ldg(row + 1) : 0.0;
            acc0 = __dadd_rn(acc0, __dmul_rn(svv, x0));
            acc1 = __dadd_rn(acc1, __dmul_rn(svv, x1));
            finite = finite && isfinite(x0) && isfinite(x1);
        }
        *o0 = acc0;
        if (has1) o0[1] = acc1;
    }
    if (!finite && st) atomicCAS(&st->err_code, 0, kErrNonfiniteA);
}

// one CTA per sketch row; threads own column pairs; rows summed in source order
__global__ void __launch_bounds__(kGatherT) gather_kernel(const double* A, int64_t ld, int n, int64_t d,
                                                          const int64_t* offs, const uint32_t* vals, double val,
                                                          double* SA, DevState* st, int vec) {
    const int64_t s = blockIdx.x;
    const int64_t e0 = offs[s], e1 = offs[s + 1];
    const int npairs = (n + 1) >> 1;
    bool finite = true;
    for (int pi = threadIdx.x; pi < npairs; pi += kGatherT) {
        const int c0 = 2 * pi;
        const bool has1 = c0 + 1 < n;
        double acc0 = 0.0, acc1 = 0.0;
        int64_t e = e0;
        for (; e + kGatherUnroll <= e1; e += kGatherUnroll) {
            double x0[kGatherUnroll], x1[kGatherUnroll], sv[kGatherUnroll];
#pragma unroll
            for (int u = 0; u < kGatherUnroll; ++u) {
                const uint32_t v = __ldg(vals + e + u);
                const int64_t r = v & 0x7fffffffu;
                sv[u] = (v >> 31) ? -val : val;
                const double* row = A + r * ld + c0;
                if (vec && has1) {
                    const double2 x = __ldg(reinterpret_cast<const double2*>(row));
                    x0[u] = x.x;
                    x1[u] = x.y;
                } else {
                    x0[u] = __ldg(row);
                    x1[u] = has1 ? __ldg(row + 1) : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < kGatherUnroll; ++u) {
                acc0 = __dadd_rn(acc0, __dmul_rn(sv[u], x0[u]));
                acc1 = __dadd_rn(acc1, __dmul_rn(sv[u], x1[u]));
                finite = finite && isfinite(x0[u]) && isfinite(x1[u]);
            }
        }
        for (; e < e1; ++e) {
            const uint32_t v = __ldg(vals + e);
            const int64_t r = v & 0x7fffffffu;
            const double svv = (v >> 31) ? -val : val;
            const double* row = A + r * ld + c0;
            const double x0 = __ldg(row);
            const double x1 = has1 ? __ldg(row + 1) : 0.0;
            acc0 = __dadd_rn(acc0, __dmul_rn(svv, x0));
            acc1 = __dadd_rn(acc1, __dmul_rn(svv, x1));
            finite = finite && isfinite(x0) && isfinite(x1);
        }
        SA[s + static_cast<int64_t>(c0) * d] = acc0;
        if (has1) SA[s + static_cast<int64_t>(c0 + 1) * d] = acc1;
    }
    if (!finite && st) atomicCAS(&st->err_code, 0, kErrNonfiniteA);
}


// Column-slice form of the one-shot gather: A is read in slices of 32*CPL
// columns, one launch per slice, one warp per sketch row.  All d warps of a
// slice are resident together and walk their (ascending) source lists at the
// same pace, so the zeta readers of each A row-slice meet it in L2 within a
// short window: A comes from HBM once instead of zeta times.  Same per-column
// sequential __dmul_rn/__dadd_rn sums as gather_kernel -> the same bits.
template <int kSliceCPL, int kSliceU>
__global__ void __launch_bounds__(256, 4) gather_slice_kernel(const double* __restrict__ A, int64_t ld, int n,
                                                           int64_t d, const int64_t* __restrict__ offs,
                                                           const uint32_t* __restrict__ vals, double val,
                                                           double* __restrict__ SA, DevState* st, int c0) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t s = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    if (s >= d) return;
    const int64_t e0 = offs[s], e1 = offs[s + 1];
    int col[kSliceCPL];
    bool in[kSliceCPL];
#pragma unroll
    for (int q = 0; q < kSliceCPL; ++q) {
        col[q] = c0 + lane + 32 * q;
        in[q] = col[q] < n;
        if (!in[q]) col[q] = n - 1;  // clamped load, result dropped
    }
    double acc[kSliceCPL];
#pragma unroll
    for (int q = 0; q < kSliceCPL; ++q) acc[q] = 0.0;
    bool finite = true;
    int64_t e = e0;
    for (; e + kSliceU <= e1; e += kSliceU) {
        // lane u < U fetches entry e+u; the row indices are then broadcast
        const uint32_t mine = lane < kSliceU ? vals[e + lane] : 0u;
        double x[kSliceU][kSliceCPL];
        double sv[kSliceU];
#pragma unroll
        for (int u = 0; u < kSliceU; ++u) {
            const uint32_t v = __shfl_sync(0xffffffffu, mine, u);
            const int64_t r = v & 0x7fffffffu;
            sv[u] = (v >> 31) ? -val : val;
            const double* row = A + r * ld;
#pragma unroll
            for (int q = 0; q < kSliceCPL; ++q) x[u][q] = row[col[q]];
        }
#pragma unroll
        for (int u = 0; u < kSliceU; ++u)
#pragma unroll
            for (int q = 0; q < kSliceCPL; ++q) {
                acc[q] = __dadd_rn(acc[q], __dmul_rn(sv[u], x[u][q]));
                finite = finite && isfinite(x[u][q]);
            }
    }
    for (; e < e1; ++e) {
        const uint32_t v = vals[e];
        const int64_t r = v & 0x7fffffffu;
        const double svv = (v >> 31) ? -val : val;
        const double* row = A + r * ld;
#pragma unroll
        for (int q = 0; q < kSliceCPL; ++q) {
            const double xv = row[col[q]];
            acc[q] = __dadd_rn(acc[q], __dmul_rn(svv, xv));
            finite = finite && isfinite(xv);
        }
    }
#pragma unroll
    for (int q = 0; q < kSliceCPL; ++q)
        if (in[q]) SA[s + static_cast<int64_t>(col[q]) * d] = acc[q];
    if (!__all_sync(0xffffffffu, finite) && lane == 0 && st) atomicCAS(&st->err_code, 0, kErrNonfiniteA);
}

}  // namespace

void build_sparsestack_dev(Ctx& c, int64_t d, int64_t m, int zeta, uint64_t seed, uint32_t* pos, int8_t* sgn) {
    if (m == 0) return;
    keys_kernel<<<static_cast<unsigned>(ceil_div(m, 256)), 256, 0, c.stream>>>(m, 0, d, zeta, seed, nullptr,
                                                                              nullptr, pos, sgn);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

SketchLists sketch_prepare(Ctx& c, int64_t m, int64_t row0, int64_t d, int zeta, uint64_t seed, int64_t step) {
    if (m > 0x7fffffffLL) fail(MSVD_ERR_DIMENSION, "msvd: more than 2^31-1 local rows in one sketch");
    SketchLists L{};
    L.d = d;
    L.m = m;
    L.val = 1.0 / sqrt(static_cast<double>(zeta));  // sketch.cpp:12-14
    if (m == 0) return L;
    const int64_t cnt = m * zeta;
    int bits = 1;
    while ((1LL << bits) < d) ++bits;
    size_t temp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, static_cast<uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), cnt, 0, bits, c.stream);
    const size_t arr = ((sizeof(uint32_t) * cnt + 255) / 256) * 256;
    const size_t offb = ((sizeof(int64_t) * (d + 1) + 255) / 256) * 256;
    const int64_t nch = ceil_div(m, step);
    const size_t bnd = ((sizeof(int64_t) * (nch + 1) * (d + 1) + 255) / 256) * 256;
    unsigned char* base =
        static_cast<unsigned char*>(c.ensure_scratch(4 * arr + offb + bnd + temp_bytes + 256));
    uint32_t* k_in = reinterpret_cast<uint32_t*>(base);
    uint32_t* v_in = reinterpret_cast<uint32_t*>(base + arr);
    uint32_t* k_out = reinterpret_cast<uint32_t*>(base + 2 * arr);
    uint32_t* v_out = reinterpret_cast<uint32_t*>(base + 3 * arr);
    int64_t* offs = reinterpret_cast<int64_t*>(base + 4 * arr);
    int64_t* bounds = reinterpret_cast<int64_t*>(base + 4 * arr + offb);
    void* temp = base + 4 * arr + offb + bnd;
    keys_kernel<<<static_cast<unsigned>(ceil_div(m, 256)), 256, 0, c.stream>>>(m, row0, d, zeta, seed, k_in, v_in,
                                                                              nullptr, nullptr);
    MSVD_CUDA(cudaGetLastError());
    MSVD_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k_in, k_out, v_in, v_out, cnt, 0, bits, c.stream));
    offsets_kernel<<<static_cast<unsigned>(ceil_div(d + 1, 256)), 256, 0, c.stream>>>(k_out, cnt, d, offs);
    bounds_kernel<<<static_cast<unsigned>(ceil_div((nch + 1) * d, 256)), 256, 0, c.stream>>>(offs, v_out, d, step,
                                                                                            nch, bounds);
    MSVD_CUDA(cudaGetLastError());
    c.launches += 4;  // keys, radix sort (counted once), offsets, bounds
    L.offs = offs;
    L.vals = v_out;
    L.bounds = bounds;
    L.step = step;
    return L;
}

void sketch_rows(Ctx& c, const SketchLists& L, const double* A, int64_t ld, int n, int vec, int64_t chunk,
                 double* SA, DevState* st) {
    if (L.m == 0) return;
    gather_chunk_kernel<<<static_cast<unsigned>(L.d), kGatherT, 0, c.stream>>>(A, ld, n, L.d, L.bounds, L.vals,
                                                                               L.val, SA, st, vec, chunk);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
}

int64_t sketch_chunk_rows(int64_t ld) {
    const char* e = std::getenv("MSVD_SKETCH_CHUNK_MB");
    const int64_t mb = e ? std::atoll(e) : 48;
    const int64_t rows = (mb << 20) / (8 * ld);  // ~48 MB of A per chunk: re-reads hit L2
    return rows < 1 ? 1 : rows;
}

double* sketch_begin(Ctx& c, int64_t d, int64_t n) {
    double* SAr = static_cast<double*>(c.ensure_sar(sizeof(double) * d * n));
    MSVD_CUDA(cudaMemsetAsync(SAr, 0, sizeof(double) * d * n, c.stream));
    return SAr;
}

void sketch_finish(Ctx& c, const double* SAr, int64_t d, int64_t n, double* SA) {
    launch_transpose_rm_to_cm(c, SAr, d, n, n, SA);  // row-major running sums -> column-major SA
}

// A resident in HBM: column slices, one warp per sketch row (gather_slice_kernel;
// MSVD_SKETCH_GATHER = 1 selects the one-launch gather that reads A zeta
// times).  The chunked form above is used when A arrives from the host, where
// it hides under the H2D copy.
void sketch_dev(Ctx& c, const StreamGeom& g, int64_t row0, int64_t d, int zeta, uint64_t seed, double* SA,
                DevState* st) {
    ProfScope prof(c, kProfSketch);
    if (g.m == 0) {
        MSVD_CUDA(cudaMemsetAsync(SA, 0, sizeof(double) * d * g.n, c.stream));
        return;
    }
    const SketchLists L = sketch_prepare(c, g.m, row0, d, zeta, seed, g.m);  // one chunk
    if (std::getenv("MSVD_SKETCH_GATHER")) {  // one launch, A read zeta times
        gather_kernel<<<static_cast<unsigned>(d), kGatherT, 0, c.stream>>>(g.A, g.ld, g.n, d, L.offs, L.vals, L.val,
                                                                           SA, st, g.tma);
        MSVD_CUDA(cudaGetLastError());
        ++c.launches;
        return;
    }
    // measured (C2): 32 * 2 columns x 8 entries in flight per warp (the 1-, 4-
    // and 8-pair variants were slower and spilled; a cp.async form landing the
    // rows in a per-warp shared-memory ring, 6 x 8 entries ahead, took 8.0 ms
    // instead of 3.9: removed)
    const int slice = 64;
    const unsigned grid = static_cast<unsigned>(ceil_div(d, 8));
    for (int c0 = 0; c0 < g.n; c0 += slice) {
        gather_slice_kernel<2, 8><<<grid, 256, 0, c.stream>>>(g.A, g.ld, g.n, d, L.offs, L.vals, L.val, SA, st, c0);
        MSVD_CUDA(cudaGetLastError());
        ++c.launches;
    }
}

}  // namespace msvd
