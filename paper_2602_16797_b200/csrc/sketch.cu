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
constexpr int kIdxCap = 1024;  // list entries staged per warp (4 KB)

// Per entry and lane the inner loop is: the row index from a broadcast
// shared-memory read (four entries per 16-byte read), one IMAD.WIDE per column
// for the address (ld * 8 < 2^32, checked by the caller), the sign folded into
// the high word of val, two loads, two mul + add.  The compiler's 64-bit
// index arithmetic and shuffles had made it ~35 instructions per entry, and
// the kernel issue-bound (ncu: one issue every 1.9 cycles per scheduler).
template <int kU, int kMinB>
__global__ void __launch_bounds__(256, kMinB) gather_slice_kernel(const double* __restrict__ A, uint32_t ld8, int n,
                                                                 int64_t d, const int64_t* __restrict__ offs,
                                                                 const uint32_t* __restrict__ vals, double val,
                                                                 double* __restrict__ SA, DevState* st, int c0) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t s = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    c0 += 64 * static_cast<int>(blockIdx.y);  // several slices per launch (small d: fill the SMs)
    if (s >= d || c0 >= n) return;
    const int64_t e0 = offs[s], e1 = offs[s + 1];
    // the lane's two columns (clamped to n - 1: loaded, result dropped)
    const int colA = c0 + lane, colB = c0 + lane + 32;
    const bool inA = colA < n, inB = colB < n;
    const char* baseA = reinterpret_cast<const char*>(A + (inA ? colA : n - 1));
    const char* baseB = reinterpret_cast<const char*>(A + (inB ? colB : n - 1));
    const uint64_t vbits = static_cast<uint64_t>(__double_as_longlong(val));
    double accA = 0.0, accB = 0.0;
    // a non-finite entry of A makes its sums non-finite (sv = +-zeta^-1/2 is
    // never 0), so the operator's finite check (operator.cpp:33-35) looks at
    // the sums at the end and rescans elements only when one is not finite
    // the warp's (source row, sign) list is staged in shared memory a piece at
    // a time (one coalesced copy), so a batch's row indices come from shared
    // memory and only the A loads are on its critical path
    extern __shared__ __align__(16) uint32_t sidx_all[];  // [8 warps][kIdxCap]
    uint32_t* sidx = sidx_all + warp * kIdxCap;
    for (int64_t pb = e0; pb < e1; pb += kIdxCap) {
        const int cnt = static_cast<int>(min(static_cast<int64_t>(kIdxCap), e1 - pb));
        __syncwarp();
        for (int i = lane; i < cnt; i += 32) sidx[i] = vals[pb + i];
        __syncwarp();
        int e = 0;
        for (; e + kU <= cnt; e += kU) {
            uint32_t v[kU];
#pragma unroll
            for (int u = 0; u < kU; u += 4) {
                const uint4 q4 = *reinterpret_cast<const uint4*>(sidx + e + u);
                v[u] = q4.x;
                v[u + 1] = q4.y;
                v[u + 2] = q4.z;
                v[u + 3] = q4.w;
            }
            double xa[kU], xb[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint64_t off = static_cast<uint64_t>(v[u] & 0x7fffffffu) * ld8;
                xa[u] = __ldg(reinterpret_cast<const double*>(baseA + off));
                xb[u] = __ldg(reinterpret_cast<const double*>(baseB + off));
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const double sv = __longlong_as_double(
                    static_cast<long long>(vbits ^ (static_cast<uint64_t>(v[u] & 0x80000000u) << 32)));
                accA = __dadd_rn(accA, __dmul_rn(sv, xa[u]));
                accB = __dadd_rn(accB, __dmul_rn(sv, xb[u]));
            }
        }
        for (; e < cnt; ++e) {
            const uint32_t vv = sidx[e];
            const uint64_t off = static_cast<uint64_t>(vv & 0x7fffffffu) * ld8;
            const double sv =
                __longlong_as_double(static_cast<long long>(vbits ^ (static_cast<uint64_t>(vv & 0x80000000u) << 32)));
            accA = __dadd_rn(accA, __dmul_rn(sv, __ldg(reinterpret_cast<const double*>(baseA + off))));
            accB = __dadd_rn(accB, __dmul_rn(sv, __ldg(reinterpret_cast<const double*>(baseB + off))));
        }
    }
    if (inA) SA[s + static_cast<int64_t>(colA) * d] = accA;
    if (inB) SA[s + static_cast<int64_t>(colB) * d] = accB;
    if (__all_sync(0xffffffffu, isfinite(accA) && isfinite(accB))) return;
    // a non-finite sum: an element is non-finite, or finite ones overflowed
    // (not an error of A) -- rescan this warp's elements to tell which
    bool bad = false;
    for (int64_t e = e0; e < e1; ++e) {
        const uint64_t off = static_cast<uint64_t>(vals[e] & 0x7fffffffu) * ld8;
        bad = bad || !isfinite(*reinterpret_cast<const double*>(baseA + off)) ||
              !isfinite(*reinterpret_cast<const double*>(baseB + off));
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0 && st) atomicCAS(&st->err_code, 0, kErrNonfiniteA);
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
    // one launch, A read zeta times (also for a row stride of 2^29 or more
    // doubles, which the slice form's 32-bit byte offsets do not cover)
    if (std::getenv("MSVD_SKETCH_GATHER") || g.ld * 8 > static_cast<int64_t>(UINT32_MAX)) {
        gather_kernel<<<static_cast<unsigned>(d), kGatherT, 0, c.stream>>>(g.A, g.ld, g.n, d, L.offs, L.vals, L.val,
                                                                           SA, st, g.tma);
        MSVD_CUDA(cudaGetLastError());
        ++c.launches;
        return;
    }
    // measured (C2, 16 slices): 2.5 ms with 2 columns x 8 entries in flight
    // per lane and 4 CTAs per SM (every warp of a slice resident).  Slower,
    // and removed: 16 entries in flight or 3 CTAs per SM (a second wave;
    // 3.9 / 4.7 ms), L2 prefetch of the rows 16-32 entries ahead (3.7 ms), a
    // cp.async ring of rows in shared memory (8.0 ms), and pacing the warps so
    // the zeta readers of a row-slice meet in L2 (DRAM 1.77x -> 1.18x the
    // algorithmic bytes, but 2.5 -> 8.9 ms: the fast warps idle)
    const int slice = 64;
    const unsigned grid = static_cast<unsigned>(ceil_div(d, 8));
    // a small sketch (d / 8 CTAs of 4 * SMs slots) leaves the SMs half empty and each warp's
    // chain of load latencies exposed: as many slices per launch as fit resident
    const int per_launch = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, (4LL * c.num_sms) / grid)));
    for (int c0 = 0; c0 < g.n; c0 += slice * per_launch) {
        gather_slice_kernel<8, 4><<<dim3(grid, per_launch), 256, sizeof(uint32_t) * 8 * kIdxCap, c.stream>>>(
            g.A, static_cast<uint32_t>(g.ld * 8), g.n, d, L.offs, L.vals, L.val, SA, st, c0);
        MSVD_CUDA(cudaGetLastError());
        ++c.launches;
    }
}

}  // namespace msvd
