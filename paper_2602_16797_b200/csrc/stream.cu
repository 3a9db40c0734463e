// The two O(mn) passes over the tall row-major A.
//
// Both kernels are persistent (one CTA per SM, contiguous row range per CTA)
// and share one producer: warp 0 streams the CTA's rows HBM -> shared memory
// through a ring of `stages` buffers with 1-D TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx, L2 evict_first) or, when A's rows
// are not 16-byte aligned, with plain coalesced loads.  Consumer threads own
// fixed column pairs (16-byte shared loads, conflict free), so A is read from
// HBM exactly once per pass for all b right-hand sides.
//
//   apply_kernel  (K3)  Y = A W           -- operator.cpp:7-12 / dense.cpp:50-60
//   gram_kernel   (K2)  G = A^T (T C)     -- solver.cpp:357-369 residual_of with
//                        the recurrence products AV' = AT C, AX' = AT mix
//                        (solver.cpp:421, :462) formed in-tile by a Y warp.
#include <cstdlib>

#include "common.cuh"
#include "fold.cuh"
#include "msvd_internal.h"

namespace msvd {

namespace {

constexpr int kStageTarget = 32 * 1024;
constexpr int kStageBudget = 160 * 1024;

struct Pipe {
    uint64_t* full;
    uint64_t* empty;
    unsigned char* stage0;
    size_t stage_bytes;
};

__device__ __forceinline__ void cta_rows(int64_t m, int64_t& r0, int64_t& r1) {
    r0 = (m * blockIdx.x) / gridDim.x;
    r1 = (m * (blockIdx.x + 1)) / gridDim.x;
}

// Warp 0: fill stage c % S with rows [r_begin + c*rc, ...) of A.
__device__ void produce(const StreamGeom& g, const Pipe& p, int64_t r_begin, int64_t r_end) {
    const int lane = threadIdx.x & 31;
    const int64_t nrows = r_end - r_begin;
    const int64_t nchunks = ceil_div(nrows, g.rc);
    if (g.tma) {
        if (lane != 0) return;
        const uint64_t pol = l2_evict_first_policy();
        int s = 0;
        uint32_t ph = 1;  // parity of the empty phase to wait for (first lap: none)
        for (int64_t c = 0; c < nchunks; ++c) {
            if (c >= g.stages) mbar_wait(&p.empty[s], ph);
            const int64_t r0 = r_begin + c * g.rc;
            const int64_t rc = min(static_cast<int64_t>(g.rc), r_end - r0);
            const uint32_t bytes = static_cast<uint32_t>(rc * g.ld * 8);
            mbar_arrive_expect_tx(&p.full[s], bytes);
            bulk_g2s(p.stage0 + s * p.stage_bytes, g.A + r0 * g.ld, bytes, &p.full[s], pol);
            if (++s == g.stages) {
                s = 0;
                ph ^= 1;
            }
        }
    } else {
        int s = 0;
        uint32_t ph = 1;
        for (int64_t c = 0; c < nchunks; ++c) {
            if (c >= g.stages) mbar_wait(&p.empty[s], ph);
            const int64_t r0 = r_begin + c * g.rc;
            const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
            double* dst = reinterpret_cast<double*>(p.stage0 + s * p.stage_bytes);
            for (int r = 0; r < rc; ++r) {
                const double* src = g.A + (r0 + r) * g.ld;
                for (int e = lane; e < g.ld_s; e += 32) dst[r * g.ld_s + e] = e < g.n ? __ldg(src + e) : 0.0;
            }
            __syncwarp();
            mbar_arrive(&p.full[s]);  // all 32 lanes arrive (count includes them)
            if (++s == g.stages) {
                s = 0;
                ph ^= 1;
            }
        }
    }
}

// barrier area: full[stages] + empty[stages], 128-byte aligned
__host__ __device__ constexpr size_t bar_bytes(int stages) { return ((16 * static_cast<size_t>(stages) + 127) / 128) * 128; }

// shared-memory carve-up common to both kernels
__device__ __forceinline__ Pipe carve(unsigned char* smem, const StreamGeom& g, size_t extra_bytes,
                                      unsigned char** extra) {
    Pipe p;
    const size_t bars = bar_bytes(g.stages);
    p.full = reinterpret_cast<uint64_t*>(smem);
    p.empty = p.full + g.stages;
    *extra = smem + bars;
    p.stage0 = smem + bars + ((extra_bytes + 127) / 128) * 128;
    p.stage_bytes = g.stage_bytes;
    return p;
}

// TsqrFuse (msvd_internal.h): fused TSQR epilogue of the A*W pass (north-star
// item 3) -- the rows of the trial block [AV AX | AW] are folded into per-CTA
// Householder R factors while the pass streams, so the m x k block is never
// re-read.

struct ApplyArgs {
    StreamGeom g;
    const double* W;  // n x b col-major
    OutCols out;      // b columns of length m
    TsqrFuse ts;      // ts.Rparts == nullptr: no fused TSQR
    double* gpart;    // [grid][b][n] A_cta^T (A_cta W) partials (one-pass mode), or nullptr
    const double* ex; // pair kernel, EX: an m-vector e whose A_cta^T e fills column b of gpart
};

// K3: Y = A W.  Warps 1..8 consume.  Each warp reduces its threads'
// partial dots for a group of rows with a warp transpose-reduce and writes
// them to a per-stage slot; the last warp to finish a stage (shared-memory
// ticket) sums the 8 warp partials in fixed order and stores the rows -- no
// CTA-wide barrier on the streaming path, deterministic results.
constexpr int kRedSlots = 64;  // rows-per-chunk x B cap for the apply kernel

template <int B>
struct ApplyShape {
    static constexpr int NV = B == 1 ? 4 : (B == 2 ? 8 : 16);  // transpose slots
    static constexpr int GR = NV / B;                          // rows per group
};

template <int B>
__global__ void __launch_bounds__(32 + kConsumers, 1) apply_kernel(ApplyArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const StreamGeom& g = a.g;
    const int nslot = 2 * g.stages;  // reduction ring: a warp is at most `stages` chunks ahead
    unsigned char* extra;
    Pipe p = carve(smem, g, sizeof(double) * nslot * 8 * kRedSlots + 64 * sizeof(int), &extra);
    double* red = reinterpret_cast<double*>(extra);  // [nslot][8][kRedSlots]
    int* ticket = reinterpret_cast<int*>(red + nslot * 8 * kRedSlots);
    int64_t r_begin, r_end;
    cta_rows(g.m, r_begin, r_end);
    if (threadIdx.x == 0) {
        const uint32_t full_count = g.tma ? 1u : 32u;
        for (int s = 0; s < g.stages; ++s) {
            mbar_init(&p.full[s], full_count);
            mbar_init(&p.empty[s], kConsumers / 32);
        }
        for (int s = 0; s < nslot; ++s) ticket[s] = 0;
        mbar_fence_init();
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (warp == 0) {
        produce(g, p, r_begin, r_end);
        return;
    }
    const int ct = threadIdx.x - 32;
    const int cw = ct >> 5;
    const int n = g.n;
    const int npairs = (n + 1) >> 1;
    double w[kMaxPairs][2][B];
#pragma unroll
    for (int i = 0; i < kMaxPairs; ++i) {
        const int c0 = 2 * (ct + i * kConsumers);
#pragma unroll
        for (int j = 0; j < B; ++j) {
            w[i][0][j] = c0 < n ? a.W[c0 + static_cast<int64_t>(j) * n] : 0.0;
            w[i][1][j] = c0 + 1 < n ? a.W[c0 + 1 + static_cast<int64_t>(j) * n] : 0.0;
        }
    }
    constexpr int NV = ApplyShape<B>::NV;
    constexpr int GR = ApplyShape<B>::GR;
    const int64_t nchunks = ceil_div(r_end - r_begin, g.rc);
    int s = 0, slot = 0;
    uint32_t ph = 0;
    for (int64_t c = 0; c < nchunks; ++c) {
        mbar_wait(&p.full[s], ph);
        const double* As = reinterpret_cast<const double*>(p.stage0 + s * p.stage_bytes);
        const int64_t r0 = r_begin + c * g.rc;
        const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
        double* rs = red + (static_cast<size_t>(slot) * 8 + cw) * kRedSlots;
        for (int g0 = 0; g0 < rc; g0 += GR) {
            const int gn = min(GR, rc - g0);
            double v[NV];
#pragma unroll
            for (int i = 0; i < NV; ++i) v[i] = 0.0;
#pragma unroll
            for (int rr = 0; rr < GR; ++rr) {
                if (rr < gn) {
                    const double* row = As + static_cast<int64_t>(g0 + rr) * g.ld_s;
#pragma unroll
                    for (int i = 0; i < kMaxPairs; ++i) {
                        const int pi = ct + i * kConsumers;
                        if (pi < npairs) {
                            const double2 x = *reinterpret_cast<const double2*>(row + 2 * pi);
                            const double xy = (2 * pi + 1 < n) ? x.y : 0.0;
#pragma unroll
                            for (int j = 0; j < B; ++j) {
                                v[rr * B + j] = fma(x.x, w[i][0][j], v[rr * B + j]);
                                v[rr * B + j] = fma(xy, w[i][1][j], v[rr * B + j]);
                            }
                        }
                    }
                }
            }
            const double tot = warp_transpose_reduce<NV>(v);
            if (lane < gn * B) rs[g0 * B + lane] = tot;
        }
        // the stage's rows are in registers/partials now: hand it back to the
        // producer before the cross-warp finish, so the pipeline stays full
        __syncwarp();
        if (lane == 0) mbar_arrive(&p.empty[s]);
        if (++s == g.stages) {
            s = 0;
            ph ^= 1;
        }
        // ticket: the 8th warp through this chunk sums the warp partials
        int last = 0;
        if (lane == 0) {
            __threadfence_block();
            last = atomicAdd(&ticket[slot], 1) == 7;
        }
        last = __shfl_sync(kFull, last, 0);
        if (last) {
            __threadfence_block();
            const double* r8 = red + static_cast<size_t>(slot) * 8 * kRedSlots;
            for (int v = lane; v < rc * B; v += 32) {
                double sum = 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) sum += r8[q * kRedSlots + v];
                const int rr = v / B, j = v - (v / B) * B;
                a.out.p[j][r0 + rr] = sum;
            }
            __syncwarp();
            if (lane == 0) ticket[slot] = 0;
        }
        if (++slot == nslot) slot = 0;
    }
}

// K3, narrow-block variant (b small): every chunk is owned by ONE consumer
// warp (chunk c -> warp c mod 8), lanes own fixed column pairs and keep W in
// registers, and a row's b dot products are finished with warp butterflies.
// No cross-warp reduction at all; the ring is deep (many small stages), so
// the producer always has bytes in flight while each warp works on its chunk.
constexpr int kRowsFused = 4;  // rows per chunk supported by the fused TSQR prefetch

//
// GR: the same pass also accumulates A_cta^T (A_cta W) -- each lane re-reads
// its columns of the row from shared memory once the row's dot products are
// known -- so one sweep over A yields both A W and A^T A W (one-pass mode).
template <int B, int PL, int KM, bool GR>
__global__ void __launch_bounds__(32 + kConsumers, 1) apply_rows_kernel(ApplyArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const StreamGeom& g = a.g;
    // KM > 0: fused TSQR; per consumer warp an R factor and a 32-row tile
    constexpr size_t kTsqrBytes = KM > 0 ? sizeof(double) * 8 * (KM * KM + 32 * KM + 2 * kRowsFused * KM) : 0;
    // GR: W lives in shared memory (pairs, column-major, npad = n rounded up
    // to even) so the registers hold the A^T (A W) accumulators instead
    const int npad = (g.n + 1) & ~1;
    const size_t ws_bytes = GR ? sizeof(double) * npad * B : 0;
    unsigned char* extra;
    Pipe p = carve(smem, g, kTsqrBytes + ws_bytes, &extra);
    double* ws = reinterpret_cast<double*>(extra + kTsqrBytes);
    if constexpr (GR)
        for (int i = threadIdx.x; i < npad * B; i += blockDim.x) {
            const int cc = i % npad, j = i / npad;
            ws[i] = cc < g.n ? a.W[cc + static_cast<int64_t>(j) * g.n] : 0.0;
        }
    int64_t r_begin, r_end;
    cta_rows(g.m, r_begin, r_end);
    if (threadIdx.x == 0) {
        const uint32_t full_count = g.tma ? 1u : 32u;
        for (int s = 0; s < g.stages; ++s) {
            mbar_init(&p.full[s], full_count);
            mbar_init(&p.empty[s], 1);
        }
        mbar_fence_init();
    }
    if (KM > 0)
        for (size_t i = threadIdx.x; i < kTsqrBytes / sizeof(double); i += blockDim.x)
            reinterpret_cast<double*>(extra)[i] = 0.0;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (warp == 0) {
        produce(g, p, r_begin, r_end);
        return;
    }
    const int cw = warp - 1;
    double* Rw = KM > 0 ? reinterpret_cast<double*>(extra) + cw * KM * KM : nullptr;
    double* tile = KM > 0 ? reinterpret_cast<double*>(extra) + 8 * KM * KM + cw * 32 * KM : nullptr;
    // cached trial-column values of the next chunk, prefetched with cp.async
    double* tbuf = KM > 0 ? reinterpret_cast<double*>(extra) + 8 * (KM * KM + 32 * KM) + cw * 2 * kRowsFused * KM
                          : nullptr;
    const int kt = KM > 0 ? a.ts.k - B : 0;  // leading (cached) columns of the trial block
    int ntile = 0;
    bool finite = true;
    const int n = g.n;
    const int npairs = (n + 1) >> 1;
    double w[GR ? 1 : PL][2][B];
    double ga[GR ? PL : 1][2][B];
#pragma unroll
    for (int i = 0; i < (GR ? PL : 1); ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) ga[i][0][j] = ga[i][1][j] = 0.0;
#pragma unroll
    for (int i = 0; i < (GR ? 0 : PL); ++i) {
        const int c0 = 2 * (lane + 32 * i);
#pragma unroll
        for (int j = 0; j < B; ++j) {
            w[i][0][j] = c0 < n ? a.W[c0 + static_cast<int64_t>(j) * n] : 0.0;
            w[i][1][j] = c0 + 1 < n ? a.W[c0 + 1 + static_cast<int64_t>(j) * n] : 0.0;
        }
    }
    const int64_t nchunks = ceil_div(r_end - r_begin, g.rc);
    int s = cw;
    uint32_t ph = 0;
    while (s >= g.stages) {
        s -= g.stages;
        ph ^= 1;
    }
    auto prefetch = [&](int64_t cc, int buf) {
        if (KM > 0 && cc < nchunks && lane < kt) {
            const int64_t rr0 = r_begin + cc * g.rc;
            const int rcc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - rr0));
            const double* src = a.ts.T.p[lane];
            for (int r = 0; r < rcc; ++r) cp_async8(tbuf + (buf * kRowsFused + r) * KM + lane, src + rr0 + r);
        }
        cp_async_commit();
    };
    int tb = 0;
    if (KM > 0) prefetch(cw, 0);
    for (int64_t c = cw; c < nchunks; c += 8) {
        if (KM > 0) {
            prefetch(c + 8, tb ^ 1);  // next chunk of this warp, in flight while this one runs
            cp_async_wait<1>();       // this chunk's values have landed
            __syncwarp();
        }
        mbar_wait(&p.full[s], ph);
        const double* As = reinterpret_cast<const double*>(p.stage0 + s * p.stage_bytes);
        const int64_t r0 = r_begin + c * g.rc;
        const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
        for (int r = 0; r < rc; ++r) {
            double tv = 0.0;
            if (KM > 0 && lane < kt) tv = tbuf[(tb * kRowsFused + r) * KM + lane];
            const double* row = As + static_cast<int64_t>(r) * g.ld_s;
            double acc[B];
#pragma unroll
            for (int j = 0; j < B; ++j) acc[j] = 0.0;
#pragma unroll
            for (int i = 0; i < PL; ++i) {
                const int pi = lane + 32 * i;
                if (pi < npairs) {
                    const double2 x = *reinterpret_cast<const double2*>(row + 2 * pi);
                    const double xy = (2 * pi + 1 < n) ? x.y : 0.0;
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        double w0, w1;
                        if constexpr (GR) {
                            const double2 wv = *reinterpret_cast<const double2*>(ws + j * npad + 2 * pi);
                            w0 = wv.x;
                            w1 = wv.y;
                        } else {
                            w0 = w[i][0][j];
                            w1 = w[i][1][j];
                        }
                        acc[j] = fma(x.x, w0, acc[j]);
                        acc[j] = fma(xy, w1, acc[j]);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < B; ++j) acc[j] = warp_sum(acc[j]);
            if constexpr (GR) {
#pragma unroll
                for (int i = 0; i < PL; ++i) {
                    const int pi = lane + 32 * i;
                    if (pi < npairs) {
                        const double2 x = *reinterpret_cast<const double2*>(row + 2 * pi);
                        const double xy = (2 * pi + 1 < n) ? x.y : 0.0;
#pragma unroll
                        for (int j = 0; j < B; ++j) {
                            ga[i][0][j] = fma(x.x, acc[j], ga[i][0][j]);
                            ga[i][1][j] = fma(xy, acc[j], ga[i][1][j]);
                        }
                    }
                }
            }
            if (lane < B) {
                double v = acc[0];
#pragma unroll
                for (int j = 1; j < B; ++j)
                    if (lane == j) v = acc[j];
                a.out.p[lane][r0 + r] = v;
                if (KM > 0) tile[ntile * KM + kt + lane] = v;
            }
            if (KM > 0) {
                if (lane < kt) tile[ntile * KM + lane] = tv;
                if (++ntile == 32) {
                    __syncwarp();
                    double x[KM > 0 ? KM : 1];
#pragma unroll
                    for (int l = 0; l < (KM > 0 ? KM : 1); ++l) {
                        x[l] = l < a.ts.k ? tile[lane * KM + l] : 0.0;
                        finite = finite && isfinite(x[l]);
                    }
                    __syncwarp();
                    if constexpr (KM > 0) fold_rows<KM>(Rw, x, a.ts.k);
                    ntile = 0;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&p.empty[s]);
        s += 8;
        while (s >= g.stages) {
            s -= g.stages;
            ph ^= 1;
        }
        tb ^= 1;
    }
    if constexpr (KM > 0) {
        cp_async_wait<0>();
        // remaining rows of the warp's tile, then an 8 -> 1 tree over the CTA
        __syncwarp();
        if (ntile > 0) {
            double x[KM];
#pragma unroll
            for (int l = 0; l < KM; ++l) {
                x[l] = (lane < ntile && l < a.ts.k) ? tile[lane * KM + l] : 0.0;
                finite = finite && isfinite(x[l]);
            }
            __syncwarp();
            fold_rows<KM>(Rw, x, a.ts.k);
        }
        if (!__all_sync(kFull, finite) && lane == 0 && a.ts.st)
            if (atomicCAS(&a.ts.st->err_code, 0, kErrNonfiniteAT) == 0) a.ts.st->err_iter = a.ts.iter;
        named_sync(2, kConsumers);
        double* R0 = reinterpret_cast<double*>(extra);
#pragma unroll
        for (int st = 1; st < 8; st <<= 1) {
            if ((cw % (2 * st)) == 0) {
                double x[KM];
                rows_of<KM>(R0 + (cw + st) * KM * KM, a.ts.k, x);
                fold_rows<KM>(Rw, x, a.ts.k);
            }
            named_sync(3, kConsumers);
        }
        const int k = a.ts.k;
        double* out = a.ts.Rparts + static_cast<size_t>(blockIdx.x) * k * k;
        for (int i = threadIdx.x - 32; i < k * k; i += kConsumers) {
            const int r = i % k, cc = i / k;
            out[i] = r <= cc ? R0[r + cc * KM] : 0.0;
        }
    }
    if constexpr (GR) {
        // 8 warp partials -> one CTA partial, fixed order, through the (now
        // idle) stage ring: every chunk was consumed, so every bulk copy landed
        named_sync(4, kConsumers);
        double* red = reinterpret_cast<double*>(p.stage0);  // [8][B][n]
#pragma unroll
        for (int i = 0; i < PL; ++i) {
            const int c0 = 2 * (lane + 32 * i);
#pragma unroll
            for (int j = 0; j < B; ++j) {
                if (c0 < n) red[(static_cast<size_t>(cw) * B + j) * n + c0] = ga[i][0][j];
                if (c0 + 1 < n) red[(static_cast<size_t>(cw) * B + j) * n + c0 + 1] = ga[i][1][j];
            }
        }
        named_sync(5, kConsumers);
        double* gp = a.gpart + static_cast<size_t>(blockIdx.x) * B * n;
        for (int i = threadIdx.x - 32; i < B * n; i += kConsumers) {
            double sum = red[i];
#pragma unroll
            for (int q = 1; q < 8; ++q) sum += red[static_cast<size_t>(q) * B * n + i];
            gp[i] = sum;
        }
    }
}


// Self-fed form of the narrow kernel (TMA only): no producer warp.  Chunk c
// belongs to warp c % 8 and stage c % stages, and stages is a multiple of 8,
// so each warp owns its stages outright: it consumes a stage and immediately
// refills it with its own chunk c + stages.  Eight warps per CTA instead of
// nine lifts the register cap from 168 to 255 -- room for W and, in one-pass
// mode (GR), the A^T (A W) accumulators and the row values in registers.
// EX (b = 1, one-pass, fused TSQR): the pass also accumulates A^T e for e =
// the first trial column (A V' of the previous check iterate), whose rows the
// TSQR prefetch already brings in; gpart then holds [grid][2][n].  The row
// values are re-read from shared memory for the two accumulations instead of
// being held in registers.
template <int B, int PL, int KM, bool GR, bool EX = false>
__global__ void __launch_bounds__(256, 1) apply_self_kernel(ApplyArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const StreamGeom& g = a.g;
    constexpr size_t kTsqrBytes = KM > 0 ? sizeof(double) * 8 * (KM * KM + 32 * KM + 2 * kRowsFused * KM) : 0;
    unsigned char* extra;
    Pipe p = carve(smem, g, kTsqrBytes, &extra);
    int64_t r_begin, r_end;
    cta_rows(g.m, r_begin, r_end);
    if (threadIdx.x == 0) {
        for (int s = 0; s < g.stages; ++s) mbar_init(&p.full[s], 1);
        mbar_fence_init();
    }
    if (KM > 0)
        for (size_t i = threadIdx.x; i < kTsqrBytes / sizeof(double); i += blockDim.x)
            reinterpret_cast<double*>(extra)[i] = 0.0;
    __syncthreads();
    const int cw = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int per_warp = g.stages / 8;
    const int64_t nchunks = ceil_div(r_end - r_begin, g.rc);
    const uint64_t pol = l2_evict_first_policy();
    auto issue = [&](int64_t c, int s) {  // lane 0: chunk c into its stage s = c % stages
        const int64_t r0 = r_begin + c * g.rc;
        const int64_t rc = min(static_cast<int64_t>(g.rc), r_end - r0);
        const uint32_t bytes = static_cast<uint32_t>(rc * g.ld * 8);
        mbar_arrive_expect_tx(&p.full[s], bytes);
        bulk_g2s(p.stage0 + s * p.stage_bytes, g.A + r0 * g.ld, bytes, &p.full[s], pol);
    };
    if (lane == 0)
        for (int j = 0; j < per_warp; ++j) {
            const int64_t c = cw + 8 * static_cast<int64_t>(j);
            if (c < nchunks) issue(c, cw + 8 * j);
        }
    double* Rw = KM > 0 ? reinterpret_cast<double*>(extra) + cw * KM * KM : nullptr;
    double* tile = KM > 0 ? reinterpret_cast<double*>(extra) + 8 * KM * KM + cw * 32 * KM : nullptr;
    double* tbuf = KM > 0 ? reinterpret_cast<double*>(extra) + 8 * (KM * KM + 32 * KM) + cw * 2 * kRowsFused * KM
                          : nullptr;
    const int kt = KM > 0 ? a.ts.k - B : 0;
    int ntile = 0;
    bool finite = true;
    const int n = g.n;
    const int npairs = (n + 1) >> 1;
    static_assert(!EX || (GR && KM > 0 && B == 1), "EX: one-pass b = 1 with the fused TSQR");
    double w[PL][2][B];
    double ga[GR ? PL : 1][2][B];
    double ge[EX ? PL : 1][2];
#pragma unroll
    for (int i = 0; i < PL; ++i) {
        const int c0 = 2 * (lane + 32 * i);
#pragma unroll
        for (int j = 0; j < B; ++j) {
            w[i][0][j] = c0 < n ? a.W[c0 + static_cast<int64_t>(j) * n] : 0.0;
            w[i][1][j] = c0 + 1 < n ? a.W[c0 + 1 + static_cast<int64_t>(j) * n] : 0.0;
            if (GR) ga[GR ? i : 0][0][j] = ga[GR ? i : 0][1][j] = 0.0;
        }
        if (EX) ge[EX ? i : 0][0] = ge[EX ? i : 0][1] = 0.0;
    }
    auto prefetch = [&](int64_t cc, int buf) {
        if (KM > 0 && cc < nchunks && lane < kt) {
            const int64_t rr0 = r_begin + cc * g.rc;
            const int rcc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - rr0));
            const double* src = a.ts.T.p[lane];
            for (int r = 0; r < rcc; ++r) cp_async8(tbuf + (buf * kRowsFused + r) * KM + lane, src + rr0 + r);
        }
        cp_async_commit();
    };
    int tb = 0;
    if (KM > 0) prefetch(cw, 0);
    // column offsets clamped into the row: lanes past the last pair re-read
    // it (their W entries are zero, and their A^T A W sums are never stored),
    // so the row loop has no per-pair branches
    int off[PL];
    bool keepy[PL];
#pragma unroll
    for (int i = 0; i < PL; ++i) {
        const int pi = min(lane + 32 * i, npairs - 1);
        off[i] = 2 * pi;
        keepy[i] = 2 * pi + 1 < n;
    }
    int s = cw;
    uint32_t ph = 0;
    for (int64_t c = cw; c < nchunks; c += 8) {
        if (KM > 0) {
            prefetch(c + 8, tb ^ 1);
            cp_async_wait<1>();
            __syncwarp();
        }
        mbar_wait(&p.full[s], ph);
        const double* As = reinterpret_cast<const double*>(p.stage0 + s * p.stage_bytes);
        const int64_t r0 = r_begin + c * g.rc;
        const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
        for (int r = 0; r < rc; ++r) {
            double tv = 0.0;
            if (KM > 0 && lane < kt) tv = tbuf[(tb * kRowsFused + r) * KM + lane];
            const double* row = As + static_cast<int64_t>(r) * g.ld_s;
            // NA independent partial sums per right-hand side (pairs i mod NA),
            // combined in fixed order: a DFMA chain of 2 PL / NA, not 2 PL
            constexpr int NA = PL >= 8 ? 4 : (PL >= 4 ? 2 : 1);
            double part[NA][B];
#pragma unroll
            for (int q = 0; q < NA; ++q)
#pragma unroll
                for (int j = 0; j < B; ++j) part[q][j] = 0.0;
            double2 xr[GR && !EX ? PL : 1];
#pragma unroll
            for (int i = 0; i < PL; ++i) {
                double2 x = *reinterpret_cast<const double2*>(row + off[i]);
                x.y = keepy[i] ? x.y : 0.0;  // odd n: the pad column is not A
                if (GR && !EX) xr[GR && !EX ? i : 0] = x;
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    part[i % NA][j] = fma(x.x, w[i][0][j], part[i % NA][j]);
                    part[i % NA][j] = fma(x.y, w[i][1][j], part[i % NA][j]);
                }
            }
            double acc[B];
#pragma unroll
            for (int j = 0; j < B; ++j) {
                acc[j] = part[0][j];
#pragma unroll
                for (int q = 1; q < NA; ++q) acc[j] += part[q][j];
            }
#pragma unroll
            for (int j = 0; j < B; ++j) acc[j] = warp_sum(acc[j]);
            if constexpr (GR && !EX) {
#pragma unroll
                for (int i = 0; i < PL; ++i)
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        ga[i][0][j] = fma(xr[i].x, acc[j], ga[i][0][j]);
                        ga[i][1][j] = fma(xr[i].y, acc[j], ga[i][1][j]);
                    }
            }
            if constexpr (EX) {
                const double e = __shfl_sync(kFull, tv, 0);  // row r of the first trial column
#pragma unroll
                for (int i = 0; i < PL; ++i) {
                    double2 x = *reinterpret_cast<const double2*>(row + off[i]);
                    x.y = keepy[i] ? x.y : 0.0;
                    ga[i][0][0] = fma(x.x, acc[0], ga[i][0][0]);
                    ga[i][1][0] = fma(x.y, acc[0], ga[i][1][0]);
                    ge[i][0] = fma(x.x, e, ge[i][0]);
                    ge[i][1] = fma(x.y, e, ge[i][1]);
                }
            }
            if (lane < B) {
                double v = acc[0];
#pragma unroll
                for (int j = 1; j < B; ++j)
                    if (lane == j) v = acc[j];
                a.out.p[lane][r0 + r] = v;
                if (KM > 0) tile[ntile * KM + kt + lane] = v;
            }
            if (KM > 0) {
                if (lane < kt) tile[ntile * KM + lane] = tv;
                if (++ntile == 32) {
                    __syncwarp();
                    double x[KM > 0 ? KM : 1];
#pragma unroll
                    for (int l = 0; l < (KM > 0 ? KM : 1); ++l) {
                        x[l] = l < a.ts.k ? tile[lane * KM + l] : 0.0;
                        finite = finite && isfinite(x[l]);
                    }
                    __syncwarp();
                    if constexpr (KM > 0) fold_rows<KM>(Rw, x, a.ts.k);
                    ntile = 0;
                }
            }
        }
        __syncwarp();
        // refill the stage just consumed: every lane's reads of it have
        // retired (their values fed the warp reductions above)
        if (lane == 0 && c + g.stages < nchunks) issue(c + g.stages, s);
        tb ^= 1;
        s += 8;
        if (s >= g.stages) {
            s -= g.stages;
            ph ^= 1;
        }
    }
    if constexpr (KM > 0) {
        cp_async_wait<0>();
        __syncwarp();
        if (ntile > 0) {
            double x[KM];
#pragma unroll
            for (int l = 0; l < KM; ++l) {
                x[l] = (lane < ntile && l < a.ts.k) ? tile[lane * KM + l] : 0.0;
                finite = finite && isfinite(x[l]);
            }
            __syncwarp();
            fold_rows<KM>(Rw, x, a.ts.k);
        }
        if (!__all_sync(kFull, finite) && lane == 0 && a.ts.st)
            if (atomicCAS(&a.ts.st->err_code, 0, kErrNonfiniteAT) == 0) a.ts.st->err_iter = a.ts.iter;
        __syncthreads();
        double* R0 = reinterpret_cast<double*>(extra);
#pragma unroll
        for (int st = 1; st < 8; st <<= 1) {
            if ((cw % (2 * st)) == 0) {
                double x[KM];
                rows_of<KM>(R0 + (cw + st) * KM * KM, a.ts.k, x);
                fold_rows<KM>(Rw, x, a.ts.k);
            }
            __syncthreads();
        }
        const int k = a.ts.k;
        double* out = a.ts.Rparts + static_cast<size_t>(blockIdx.x) * k * k;
        for (int i = threadIdx.x; i < k * k; i += blockDim.x) {
            const int r = i % k, cc = i / k;
            out[i] = r <= cc ? R0[r + cc * KM] : 0.0;
        }
    }
    if constexpr (GR) {
        constexpr int BG = B + (EX ? 1 : 0);
        __syncthreads();  // every chunk consumed: the stage ring is free
        double* red = reinterpret_cast<double*>(p.stage0);  // [8][BG][n]
#pragma unroll
        for (int i = 0; i < PL; ++i) {
            const int c0 = 2 * (lane + 32 * i);
#pragma unroll
            for (int j = 0; j < BG; ++j) {
                const double v0 = j < B ? ga[i][0][j < B ? j : 0] : ge[EX ? i : 0][0];
                const double v1 = j < B ? ga[i][1][j < B ? j : 0] : ge[EX ? i : 0][1];
                if (c0 < n) red[(static_cast<size_t>(cw) * BG + j) * n + c0] = v0;
                if (c0 + 1 < n) red[(static_cast<size_t>(cw) * BG + j) * n + c0 + 1] = v1;
            }
        }
        __syncthreads();
        double* gp = a.gpart + static_cast<size_t>(blockIdx.x) * BG * n;
        for (int i = threadIdx.x; i < BG * n; i += blockDim.x) {
            double sum = red[i];
#pragma unroll
            for (int q = 1; q < 8; ++q) sum += red[static_cast<size_t>(q) * BG * n + i];
            gp[i] = sum;
        }
    }
}

// One-pass form for wider blocks: a row is split across a warp PAIR (warp
// 2q + h takes the column pairs [h * half, (h + 1) * half)), so W, the
// A^T (A W) accumulators and the row values of half a row fit in registers
// where a whole row does not (b = 2 up to n = 1024, b = 3, 4 up to n = 512,
// b = 1 up to n = 2048).  Chunk c belongs to pair c % 4 and stage c % stages
// (stages a multiple of 4), both warps wait on the stage's mbarrier, and
// the half-row dot products meet through shared memory behind a per-pair
// named barrier (the sum is formed in fixed order, the same bits in both
// warps).  No fused TSQR: the caller runs the separate TSQR pass.
template <int B, int PL, bool EX>
__global__ void __launch_bounds__(256, 1) apply_pair_kernel(ApplyArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const StreamGeom& g = a.g;
    unsigned char* extra;
    constexpr size_t kXBytes = sizeof(double) * 4 * 2 * 2 * B;  // [pair][buffer][half][B]
    Pipe p = carve(smem, g, kXBytes, &extra);
    double* xbuf = reinterpret_cast<double*>(extra);
    int64_t r_begin, r_end;
    cta_rows(g.m, r_begin, r_end);
    if (threadIdx.x == 0) {
        for (int s = 0; s < g.stages; ++s) mbar_init(&p.full[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const int cw = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pr = cw >> 1, h = cw & 1;
    const int bar = 1 + pr;  // named barrier of this pair (ids 1..4)
    const int per_pair = g.stages / 4;
    const int64_t nchunks = ceil_div(r_end - r_begin, g.rc);
    const uint64_t pol = l2_evict_first_policy();
    auto issue = [&](int64_t c, int s) {
        const int64_t r0 = r_begin + c * g.rc;
        const int64_t rc = min(static_cast<int64_t>(g.rc), r_end - r0);
        const uint32_t bytes = static_cast<uint32_t>(rc * g.ld * 8);
        mbar_arrive_expect_tx(&p.full[s], bytes);
        bulk_g2s(p.stage0 + s * p.stage_bytes, g.A + r0 * g.ld, bytes, &p.full[s], pol);
    };
    if (h == 0 && lane == 0)
        for (int j = 0; j < per_pair; ++j) {
            const int64_t c = pr + 4 * static_cast<int64_t>(j);
            if (c < nchunks) issue(c, pr + 4 * j);
        }
    const int n = g.n;
    const int npairs = (n + 1) >> 1;
    const int half = (npairs + 1) >> 1;
    const int p0 = h * half;
    const int pend = min(npairs, p0 + half);
    constexpr int BG = B + (EX ? 1 : 0);  // accumulated columns: A^T (A W) and, with EX, A^T e
    double w[PL][2][B], ga[PL][2][BG];
    int off[PL];
    bool keepy[PL], mine[PL];
#pragma unroll
    for (int i = 0; i < PL; ++i) {
        const int pi = p0 + lane + 32 * i;
        mine[i] = pi < pend;
        const int pc = mine[i] ? pi : max(0, min(npairs - 1, pend - 1));
        off[i] = 2 * pc;
        keepy[i] = 2 * pc + 1 < n;
#pragma unroll
        for (int j = 0; j < B; ++j) {
            w[i][0][j] = mine[i] ? a.W[2 * pc + static_cast<int64_t>(j) * n] : 0.0;
            w[i][1][j] = mine[i] && keepy[i] ? a.W[2 * pc + 1 + static_cast<int64_t>(j) * n] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < BG; ++j) ga[i][0][j] = ga[i][1][j] = 0.0;
    }
    // EX: the chunk's e values, lane l holding rows l and 32 + l, loaded one
    // chunk ahead so the row loop never waits on them
    double exc[2] = {0.0, 0.0}, exn[2] = {0.0, 0.0};
    auto ex_load = [&](int64_t cc, double (&dst)[2]) {
        if (!EX || cc >= nchunks) return;
        const int64_t rr0 = r_begin + cc * g.rc;
        const int rcc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - rr0));
        dst[0] = lane < rcc ? a.ex[rr0 + lane] : 0.0;
        dst[1] = 32 + lane < rcc ? a.ex[rr0 + 32 + lane] : 0.0;
    };
    ex_load(pr, exn);
    int s = pr, xb = 0;
    uint32_t ph = 0;
    for (int64_t c = pr; c < nchunks; c += 4) {
        if (EX) {
            exc[0] = exn[0];
            exc[1] = exn[1];
            ex_load(c + 4, exn);
        }
        mbar_wait(&p.full[s], ph);
        const double* As = reinterpret_cast<const double*>(p.stage0 + s * p.stage_bytes);
        const int64_t r0 = r_begin + c * g.rc;
        const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
        for (int r = 0; r < rc; ++r) {
            const double* row = As + static_cast<int64_t>(r) * g.ld_s;
            constexpr int NA = PL >= 8 ? 4 : (PL >= 4 ? 2 : 1);
            double part[NA][B];
#pragma unroll
            for (int q = 0; q < NA; ++q)
#pragma unroll
                for (int j = 0; j < B; ++j) part[q][j] = 0.0;
            double2 xr[PL];
#pragma unroll
            for (int i = 0; i < PL; ++i) {
                double2 x = *reinterpret_cast<const double2*>(row + off[i]);
                x.y = keepy[i] ? x.y : 0.0;  // odd n: the pad column is not A
                xr[i] = x;
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    part[i % NA][j] = fma(x.x, w[i][0][j], part[i % NA][j]);
                    part[i % NA][j] = fma(x.y, w[i][1][j], part[i % NA][j]);
                }
            }
            double acc[B];
#pragma unroll
            for (int j = 0; j < B; ++j) {
                acc[j] = part[0][j];
#pragma unroll
                for (int q = 1; q < NA; ++q) acc[j] += part[q][j];
                acc[j] = warp_sum(acc[j]);
            }
            double* xs = xbuf + (pr * 2 + xb) * 2 * B;
            if (lane == 0)
#pragma unroll
                for (int j = 0; j < B; ++j) xs[h * B + j] = acc[j];
            named_sync(bar, 64);
            double y[B];
#pragma unroll
            for (int j = 0; j < B; ++j) y[j] = xs[j] + xs[B + j];  // half 0 + half 1, both warps alike
            xb ^= 1;
            double e = 0.0;
            if (EX) e = __shfl_sync(kFull, r < 32 ? exc[0] : exc[1], r & 31);
#pragma unroll
            for (int i = 0; i < PL; ++i) {
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    ga[i][0][j] = fma(xr[i].x, y[j], ga[i][0][j]);
                    ga[i][1][j] = fma(xr[i].y, y[j], ga[i][1][j]);
                }
                if (EX) {
                    ga[i][0][BG - 1] = fma(xr[i].x, e, ga[i][0][BG - 1]);
                    ga[i][1][BG - 1] = fma(xr[i].y, e, ga[i][1][BG - 1]);
                }
            }
            if (h == 0 && lane < B) {
                double v = y[0];
#pragma unroll
                for (int j = 1; j < B; ++j)
                    if (lane == j) v = y[j];
                a.out.p[lane][r0 + r] = v;
            }
        }
        // both halves of every row of the stage are read: refill it
        named_sync(bar, 64);
        if (h == 0 && lane == 0 && c + g.stages < nchunks) issue(c + g.stages, s);
        s += 4;
        if (s >= g.stages) {
            s -= g.stages;
            ph ^= 1;
        }
    }
    __syncthreads();  // every chunk consumed: the stage ring is free
    double* red = reinterpret_cast<double*>(p.stage0);  // [4 pairs][BG][n]
#pragma unroll
    for (int i = 0; i < PL; ++i) {
        if (!mine[i]) continue;
        const int c0 = off[i];
#pragma unroll
        for (int j = 0; j < BG; ++j) {
            red[(static_cast<size_t>(pr) * BG + j) * n + c0] = ga[i][0][j];
            if (keepy[i]) red[(static_cast<size_t>(pr) * BG + j) * n + c0 + 1] = ga[i][1][j];
        }
    }
    __syncthreads();
    double* gp = a.gpart + static_cast<size_t>(blockIdx.x) * BG * n;
    for (int i = threadIdx.x; i < BG * n; i += blockDim.x) {
        double sum = red[i];
#pragma unroll
        for (int q = 1; q < 4; ++q) sum += red[static_cast<size_t>(q) * BG * n + i];
        gp[i] = sum;
    }
}

// The check-refresh pass for b >= 2: a row is split across a TEAM of T
// warps (T = 4: a quarter row each), so W, the accumulators of A^T (A W) and
// of A^T E (E = A V' of the previous check iterate, b columns) and the row
// values fit in registers.  Chunk c belongs to team c % (8 / T); the quarter
// dot products meet in shared memory behind a per-team named barrier and are
// summed in fixed order.  gpart holds [grid][2b][n].
constexpr int kTeamRows = 4;  // rows per team barrier (= rows per stage)

template <int B, int PL, int T>
__global__ void __launch_bounds__(256, 1) apply_team_ex_kernel(ApplyArgs a, Cols ex) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int TEAMS = 8 / T;
    constexpr int BG = 2 * B;
    const StreamGeom& g = a.g;
    unsigned char* extra;
    constexpr size_t kXBytes = sizeof(double) * TEAMS * 2 * T * kTeamRows * B;  // [team][buffer][member][row][B]
    Pipe p = carve(smem, g, kXBytes, &extra);
    double* xbuf = reinterpret_cast<double*>(extra);
    int64_t r_begin, r_end;
    cta_rows(g.m, r_begin, r_end);
    if (threadIdx.x == 0) {
        for (int s = 0; s < g.stages; ++s) mbar_init(&p.full[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const int cw = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tm = cw / T, h = cw % T;
    const int bar = 1 + tm;
    const int per_team = g.stages / TEAMS;
    const int64_t nchunks = ceil_div(r_end - r_begin, g.rc);
    const uint64_t pol = l2_evict_first_policy();
    auto issue = [&](int64_t c, int s) {
        const int64_t r0 = r_begin + c * g.rc;
        const int64_t rc = min(static_cast<int64_t>(g.rc), r_end - r0);
        const uint32_t bytes = static_cast<uint32_t>(rc * g.ld * 8);
        mbar_arrive_expect_tx(&p.full[s], bytes);
        bulk_g2s(p.stage0 + s * p.stage_bytes, g.A + r0 * g.ld, bytes, &p.full[s], pol);
    };
    if (h == 0 && lane == 0)
        for (int j = 0; j < per_team; ++j) {
            const int64_t c = tm + TEAMS * static_cast<int64_t>(j);
            if (c < nchunks) issue(c, tm + TEAMS * j);
        }
    const int n = g.n;
    const int npairs = (n + 1) >> 1;
    const int part = (npairs + T - 1) / T;
    const int p0 = h * part;
    const int pend = min(npairs, p0 + part);
    double w[PL][2][B], ga[PL][2][BG];
    int off[PL];
    bool keepy[PL], mine[PL];
#pragma unroll
    for (int i = 0; i < PL; ++i) {
        const int pi = p0 + lane + 32 * i;
        mine[i] = pi < pend;
        const int pc = mine[i] ? pi : max(0, min(npairs - 1, pend - 1));
        off[i] = 2 * pc;
        keepy[i] = 2 * pc + 1 < n;
#pragma unroll
        for (int j = 0; j < B; ++j) {
            w[i][0][j] = mine[i] ? a.W[2 * pc + static_cast<int64_t>(j) * n] : 0.0;
            w[i][1][j] = mine[i] && keepy[i] ? a.W[2 * pc + 1 + static_cast<int64_t>(j) * n] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < BG; ++j) ga[i][0][j] = ga[i][1][j] = 0.0;
    }
    // the chunk's E rows, lane l holding rows l and 32 + l, one chunk ahead
    double exc[2][B], exn[2][B];
    auto ex_load = [&](int64_t cc) {
        if (cc >= nchunks) return;
        const int64_t rr0 = r_begin + cc * g.rc;
        const int rcc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - rr0));
#pragma unroll
        for (int j = 0; j < B; ++j) {
            exn[0][j] = lane < rcc ? ex.p[j][rr0 + lane] : 0.0;
            exn[1][j] = 32 + lane < rcc ? ex.p[j][rr0 + 32 + lane] : 0.0;
        }
    };
#pragma unroll
    for (int j = 0; j < B; ++j) exn[0][j] = exn[1][j] = 0.0;
    ex_load(tm);
    static_assert(kTeamRows == 4, "the transpose-reduce below is written for 4 rows");
    int s = tm, xb = 0;
    uint32_t ph = 0;
    for (int64_t c = tm; c < nchunks; c += TEAMS) {
#pragma unroll
        for (int j = 0; j < B; ++j) {
            exc[0][j] = exn[0][j];
            exc[1][j] = exn[1][j];
        }
        ex_load(c + TEAMS);
        mbar_wait(&p.full[s], ph);
        const double* As = reinterpret_cast<const double*>(p.stage0 + s * p.stage_bytes);
        const int64_t r0 = r_begin + c * g.rc;
        const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
        for (int r = 0; r < rc; r += kTeamRows) {
            // sweep 1: this member's quarter-row dot products of kTeamRows rows, lane partials
            double v[B][kTeamRows];
#pragma unroll
            for (int q = 0; q < kTeamRows; ++q) {
#pragma unroll
                for (int j = 0; j < B; ++j) v[j][q] = 0.0;
                if (r + q < rc) {
                    const double* row = As + static_cast<int64_t>(r + q) * g.ld_s;
#pragma unroll
                    for (int i = 0; i < PL; ++i) {
                        double2 x = *reinterpret_cast<const double2*>(row + off[i]);
                        x.y = keepy[i] ? x.y : 0.0;  // odd n: the pad column is not A
#pragma unroll
                        for (int j = 0; j < B; ++j) {
                            v[j][q] = fma(x.x, w[i][0][j], v[j][q]);
                            v[j][q] = fma(x.y, w[i][1][j], v[j][q]);
                        }
                    }
                }
            }
            // transpose-reduce: row q = (lane >> 3) & 3 ends in lanes 8q .. 8q+7
            const bool b4 = lane & 16, b3 = lane & 8;
#pragma unroll
            for (int j = 0; j < B; ++j) {
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const double send = b4 ? v[j][t] : v[j][t + 2];
                    const double keep = b4 ? v[j][t + 2] : v[j][t];
                    v[j][t] = keep + __shfl_xor_sync(kFull, send, 16);
                }
                {
                    const double send = b3 ? v[j][0] : v[j][1];
                    const double keep = b3 ? v[j][1] : v[j][0];
                    v[j][0] = keep + __shfl_xor_sync(kFull, send, 8);
                }
                v[j][0] += __shfl_xor_sync(kFull, v[j][0], 4);
                v[j][0] += __shfl_xor_sync(kFull, v[j][0], 2);
                v[j][0] += __shfl_xor_sync(kFull, v[j][0], 1);
            }
            const int qm = (lane >> 3) & 3;
            double* xs = xbuf + (tm * 2 + xb) * T * kTeamRows * B;  // [member][row][B]
            if ((lane & 7) == 0)
#pragma unroll
                for (int j = 0; j < B; ++j) xs[(h * kTeamRows + qm) * B + j] = v[j][0];
            named_sync(bar, 32 * T);
            double ym[B];  // y of row qm: the members' quarters in order, the same bits in every warp
#pragma unroll
            for (int j = 0; j < B; ++j) {
                double t = xs[qm * B + j];
#pragma unroll
                for (int mm = 1; mm < T; ++mm) t += xs[(mm * kTeamRows + qm) * B + j];
                ym[j] = t;
            }
            xb ^= 1;
            if (h == 0 && (lane & 7) == 0 && r + qm < rc)
#pragma unroll
                for (int j = 0; j < B; ++j) a.out.p[j][r0 + r + qm] = ym[j];
            // sweep 2: the accumulators, the rows re-read from the stage
#pragma unroll
            for (int q = 0; q < kTeamRows; ++q) {
                if (r + q >= rc) break;
                const double* row = As + static_cast<int64_t>(r + q) * g.ld_s;
                const int rr = r + q;
                double y[B], e[B];
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    y[j] = __shfl_sync(kFull, ym[j], 8 * q);
                    e[j] = __shfl_sync(kFull, rr < 32 ? exc[0][j] : exc[1][j], rr & 31);
                }
#pragma unroll
                for (int i = 0; i < PL; ++i) {
                    double2 x = *reinterpret_cast<const double2*>(row + off[i]);
                    x.y = keepy[i] ? x.y : 0.0;
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        ga[i][0][j] = fma(x.x, y[j], ga[i][0][j]);
                        ga[i][1][j] = fma(x.y, y[j], ga[i][1][j]);
                        ga[i][0][B + j] = fma(x.x, e[j], ga[i][0][B + j]);
                        ga[i][1][B + j] = fma(x.y, e[j], ga[i][1][B + j]);
                    }
                }
            }
        }
        named_sync(bar, 32 * T);  // every member has read the stage: refill it
        if (h == 0 && lane == 0 && c + g.stages < nchunks) issue(c + g.stages, s);
        s += TEAMS;
        if (s >= g.stages) {
            s -= g.stages;
            ph ^= 1;
        }
    }
    __syncthreads();
    double* red = reinterpret_cast<double*>(p.stage0);  // [TEAMS][BG][n]
#pragma unroll
    for (int i = 0; i < PL; ++i) {
        if (!mine[i]) continue;
        const int c0 = off[i];
#pragma unroll
        for (int j = 0; j < BG; ++j) {
            red[(static_cast<size_t>(tm) * BG + j) * n + c0] = ga[i][0][j];
            if (keepy[i]) red[(static_cast<size_t>(tm) * BG + j) * n + c0 + 1] = ga[i][1][j];
        }
    }
    __syncthreads();
    double* gp = a.gpart + static_cast<size_t>(blockIdx.x) * BG * n;
    for (int i = threadIdx.x; i < BG * n; i += blockDim.x) {
        double sum = red[i];
#pragma unroll
        for (int q = 1; q < TEAMS; ++q) sum += red[static_cast<size_t>(q) * BG * n + i];
        gp[i] = sum;
    }
}

struct GramArgs {
    StreamGeom g;
    Cols T;            // k columns of length m
    int k;
    const double* Cm;  // k x q, ld k (gram mode)
    int q;             // Y columns produced (<= 2B); the first B feed G
    OutCols out;       // q output columns (gram mode)
    int direct;        // Y = T (k == B), no outputs
    double* Gpart;     // [grid][B][n]
    const int* skip;   // device flag: nonzero = the pass is not needed (one-pass check gate)
};

// K2: Gpart = A_cta^T Y_cta.  Warp 1 (the Y warp) forms Y rows for each
// stage from the skinny trial block and writes the new recurrence products;
// warps 2..9 stream the stage and accumulate in registers.
template <int B>
__global__ void __launch_bounds__(64 + kConsumers, 1) gram_kernel(GramArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (a.skip && *a.skip) return;
    const StreamGeom& g = a.g;
    const size_t cm_bytes = sizeof(double) * kMaxK * 2 * kMaxB;
    const size_t ys_bytes = sizeof(double) * g.stages * g.rc * B;
    unsigned char* extra;
    Pipe p = carve(smem, g, cm_bytes + ys_bytes, &extra);
    double* Cs = reinterpret_cast<double*>(extra);
    double* Ys = Cs + kMaxK * 2 * kMaxB;
    int64_t r_begin, r_end;
    cta_rows(g.m, r_begin, r_end);
    if (threadIdx.x == 0) {
        const uint32_t full_count = (g.tma ? 1u : 32u) + 32u;
        for (int s = 0; s < g.stages; ++s) {
            mbar_init(&p.full[s], full_count);
            mbar_init(&p.empty[s], kConsumers / 32);
        }
        mbar_fence_init();
    }
    if (!a.direct)
        for (int i = threadIdx.x; i < a.k * a.q; i += blockDim.x) Cs[i] = a.Cm[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nchunks = ceil_div(r_end - r_begin, g.rc);
    if (warp == 0) {
        produce(g, p, r_begin, r_end);
        return;
    }
    if (warp == 1) {
        // Y rows are formed 32 at a time (lane = row) so the skinny loads of a
        // whole window are in flight together, then handed to the stages that
        // cover them.  The window runs ahead of the A stream, never behind it.
        int64_t w0 = 0, w1 = 0;  // current window [w0, w1)
        double yv[2 * B];
#pragma unroll
        for (int j = 0; j < 2 * B; ++j) yv[j] = 0.0;
        int s = 0;
        uint32_t ph = 1;
        for (int64_t c = 0; c < nchunks; ++c) {
            const int64_t r0 = r_begin + c * g.rc;
            const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
            double* ys = Ys + static_cast<size_t>(s) * g.rc * B;
            bool waited = c < g.stages;
            for (int64_t sub = r0; sub < r0 + rc;) {
                if (sub >= w1) {
                    w0 = sub;
                    w1 = min(sub + 32, r_end);
                    const int64_t gr = w0 + lane;
                    if (gr < w1) {
                        if (a.direct) {
#pragma unroll
                            for (int j = 0; j < B; ++j) yv[j] = a.T.p[j][gr];
                        } else {
                            double t[kMaxK];
#pragma unroll
                            for (int l = 0; l < kMaxK; ++l) t[l] = l < a.k ? a.T.p[l][gr] : 0.0;
#pragma unroll
                            for (int j = 0; j < 2 * B; ++j) {
                                if (j < a.q) {
                                    double y = 0.0;
#pragma unroll
                                    for (int l = 0; l < kMaxK; ++l)
                                        if (l < a.k) y = fma(Cs[l + j * a.k], t[l], y);
                                    yv[j] = y;
                                    a.out.p[j][gr] = y;
                                }
                            }
                        }
                    }
                }
                if (!waited) {
                    mbar_wait(&p.empty[s], ph);
                    waited = true;
                }
                const int64_t end = min(w1, r0 + rc);
                const int64_t gr = w0 + lane;
                if (gr >= sub && gr < end) {
#pragma unroll
                    for (int j = 0; j < B; ++j) ys[(gr - r0) * B + j] = yv[j];
                }
                sub = end;
            }
            __syncwarp();
            mbar_arrive(&p.full[s]);
            if (++s == g.stages) {
                s = 0;
                ph ^= 1;
            }
        }
        return;
    }
    const int ct = threadIdx.x - 64;
    const int n = g.n;
    const int npairs = (n + 1) >> 1;
    double acc[kMaxPairs][2][B];
#pragma unroll
    for (int i = 0; i < kMaxPairs; ++i)
#pragma unroll
        for (int j = 0; j < B; ++j) acc[i][0][j] = acc[i][1][j] = 0.0;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t c = 0; c < nchunks; ++c) {
        mbar_wait(&p.full[s], ph);
        const double* As = reinterpret_cast<const double*>(p.stage0 + s * p.stage_bytes);
        const double* ys = Ys + static_cast<size_t>(s) * g.rc * B;
        const int64_t r0 = r_begin + c * g.rc;
        const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
#pragma unroll 2
        for (int r = 0; r < rc; ++r) {
            double y[B];
#pragma unroll
            for (int j = 0; j < B; ++j) y[j] = ys[r * B + j];
            const double* row = As + static_cast<int64_t>(r) * g.ld_s;
#pragma unroll
            for (int i = 0; i < kMaxPairs; ++i) {
                const int pi = ct + i * kConsumers;
                if (pi < npairs) {
                    const double2 x = *reinterpret_cast<const double2*>(row + 2 * pi);
                    const double xy = (2 * pi + 1 < n) ? x.y : 0.0;
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        acc[i][0][j] = fma(x.x, y[j], acc[i][0][j]);
                        acc[i][1][j] = fma(xy, y[j], acc[i][1][j]);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&p.empty[s]);
        if (++s == g.stages) {
            s = 0;
            ph ^= 1;
        }
    }
    double* gp = a.Gpart + static_cast<size_t>(blockIdx.x) * B * n;
#pragma unroll
    for (int i = 0; i < kMaxPairs; ++i) {
        const int c0 = 2 * (ct + i * kConsumers);
#pragma unroll
        for (int j = 0; j < B; ++j) {
            if (c0 < n) gp[static_cast<size_t>(j) * n + c0] = acc[i][0][j];
            if (c0 + 1 < n) gp[static_cast<size_t>(j) * n + c0 + 1] = acc[i][1][j];
        }
    }
}

size_t apply_smem(const StreamGeom& g) {
    const size_t extra = sizeof(double) * 2 * g.stages * 8 * kRedSlots + 64 * sizeof(int);
    return bar_bytes(g.stages) + ((extra + 127) / 128) * 128 + g.stages * g.stage_bytes;
}

int64_t env_int(const char* name, int64_t dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoll(v) : dflt;
}

// re-chunk a geometry: rows per stage from a target stage size, stage count
// from a shared-memory budget (env MSVD_STAGE_KB / MSVD_STAGE_BUDGET_KB
// override, for tuning sweeps)
StreamGeom rechunk(StreamGeom g, int64_t target_kb, int64_t budget_kb) {
    const int64_t row_bytes = static_cast<int64_t>(g.ld_s) * 8;
    const int64_t target = env_int("MSVD_STAGE_KB", target_kb) * 1024;
    const int64_t budget = env_int("MSVD_STAGE_BUDGET_KB", budget_kb) * 1024;
    g.rc = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(target / row_bytes, 64)));
    g.stage_bytes = ((static_cast<size_t>(g.rc) * row_bytes + 127) / 128) * 128;
    g.stages = static_cast<int32_t>(std::max<size_t>(2, std::min<size_t>(8, budget / g.stage_bytes)));
    return g;
}

// cap rows per chunk (stage geometry recomputed for the smaller chunk)
StreamGeom cap_rows(StreamGeom g, int maxrc) {
    if (g.rc <= maxrc) return g;
    const int64_t row_bytes = static_cast<int64_t>(g.ld_s) * 8;
    g.rc = maxrc;
    g.stage_bytes = ((static_cast<size_t>(g.rc) * row_bytes + 127) / 128) * 128;
    g.stages = static_cast<int32_t>(std::max<size_t>(2, std::min<size_t>(8, kStageBudget / g.stage_bytes)));
    return g;
}
size_t gram_smem(const StreamGeom& g, int B) {
    const size_t extra = sizeof(double) * kMaxK * 2 * kMaxB + sizeof(double) * g.stages * g.rc * B;
    return bar_bytes(g.stages) + ((extra + 127) / 128) * 128 + g.stages * g.stage_bytes;
}

template <int B, int PL, int KM, bool GR, bool EX = false>
void apply_rows_b(Ctx& c, const ApplyArgs& a) {
    optin_smem(c, apply_rows_kernel<B, PL, KM, GR>);
    // self-fed form: faster for the one-pass and wider blocks; the producer
    // form stays ahead for the plain b = 1 pass (measured, C2)
    const bool self = a.g.tma && !std::getenv("MSVD_APPLY_PRODUCER") && (GR || B > 1 || std::getenv("MSVD_APPLY_SELF"));
    if (self) {
        optin_smem(c, apply_self_kernel<B, PL, KM, GR, EX>);
        const size_t tsqr = KM > 0 ? sizeof(double) * 8 * (KM * KM + 32 * KM + 2 * kRowsFused * KM) : 0;
        const size_t sm = bar_bytes(a.g.stages) + ((tsqr + 127) / 128) * 128 + a.g.stages * a.g.stage_bytes;
        apply_self_kernel<B, PL, KM, GR, EX><<<a.g.grid, 256, sm, c.stream>>>(a);
        MSVD_CUDA(cudaGetLastError());
        ++c.launches;
        c.paths |= kPathSelf;
        return;
    }
    const size_t tsqr = (KM > 0 ? sizeof(double) * 8 * (KM * KM + 32 * KM + 2 * kRowsFused * KM) : 0) +
                        (GR ? sizeof(double) * ((a.g.n + 1) & ~1) * B : 0);
    const size_t sm = bar_bytes(a.g.stages) + ((tsqr + 127) / 128) * 128 + a.g.stages * a.g.stage_bytes;
    apply_rows_kernel<B, PL, KM, GR><<<a.g.grid, 32 + kConsumers, sm, c.stream>>>(a);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    c.paths |= kPathRows;
}

// dispatch on the fused-TSQR width (KM = k rounded up to 4/8/16)
template <int B, int PL>
void apply_rows_km(Ctx& c, const ApplyArgs& a) {
    if (a.gpart) {  // one-pass mode (B * PL <= 16: registers); fused TSQR only in the k <= 4 form
        if constexpr (B * PL <= 16) {
            if (!a.ts.Rparts) return apply_rows_b<B, PL, 0, true>(c, a);
            return apply_rows_b<B, PL, 4, true>(c, a);
        } else {
            fail(MSVD_ERR_INVALID, "msvd: one-pass A*W / A^T A W launch on an unsupported shape");
        }
    }
    if (!a.ts.Rparts) return apply_rows_b<B, PL, 0, false>(c, a);
    if (a.ts.k <= 4) return apply_rows_b<B, PL, 4, false>(c, a);
    if (a.ts.k <= 8) return apply_rows_b<B, PL, 8, false>(c, a);
    return apply_rows_b<B, PL, 16, false>(c, a);
}

// shared memory the narrow kernels need besides the stage ring
size_t rows_extra_bytes(const StreamGeom& g0, int b, const TsqrFuse* ts, bool gram) {
    const int km = ts && ts->Rparts ? (ts->k <= 4 ? 4 : (ts->k <= 8 ? 8 : 16)) : 0;
    const size_t tsqr = km ? sizeof(double) * 8 * (km * km + 32 * km + 2 * kRowsFused * km) : 0;
    const size_t ws = gram && !(g0.tma && !std::getenv("MSVD_APPLY_PRODUCER")) ? sizeof(double) * ((g0.n + 1) & ~1) * b
                                                                               : 0;  // (self-fed GR keeps W in registers)
    return ((tsqr + ws + 127) / 128) * 128;
}

// geometry of the narrow variant: ~8 KB stages, as deep a ring as shared
// memory allows (<= 4 stages per warp)
StreamGeom rows_geom(const Ctx& c, StreamGeom g, size_t extra) {
    const int64_t row_bytes = static_cast<int64_t>(g.ld_s) * 8;
    const int64_t target = env_int("MSVD_ROWS_STAGE_KB", 8) * 1024;
    g.rc = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(target / row_bytes, 64)));
    g.stage_bytes = ((static_cast<size_t>(g.rc) * row_bytes + 127) / 128) * 128;
    const int64_t avail = static_cast<int64_t>(c.smem_optin) - static_cast<int64_t>(extra) - 1024;
    const int64_t budget = std::min<int64_t>(env_int("MSVD_ROWS_BUDGET_KB", 168) * 1024, avail);  // measured: 2 stages per warp
    // chunk c goes to warp c % 8 and stage c % stages: with stages a multiple
    // of 8 every stage is only ever consumed by one warp, in order, so a
    // warp can never run two mbarrier phases ahead of a stage (parity ABA)
    const int64_t per_warp = std::max<int64_t>(2, std::min<int64_t>(4, budget / (8 * static_cast<int64_t>(g.stage_bytes))));
    g.stages = static_cast<int32_t>(8 * per_warp);
    return g;
}

// can the narrow kernel take this launch (b, n, fused TSQR width, one-pass gram)?
bool rows_ok(const Ctx& c, const StreamGeom& g0, int b, const TsqrFuse* ts, bool gram) {
    if (std::getenv("MSVD_APPLY_TICKET")) return false;
    const int npairs = (g0.n + 1) / 2;
    const int pl = (npairs + 31) / 32;
    const bool pl_ok = (b == 1 && pl <= 32) || (b == 2 && pl <= 16) || ((b == 3 || b == 4) && pl <= 8);
    if (!pl_ok) return false;
    const int plt = pl <= 4 ? 4 : (pl <= 8 ? 8 : (pl <= 16 ? 16 : 32));
    if (gram && b * plt > 16) return false;  // one-pass registers: the pair kernel takes it
    if (ts && ts->Rparts && (ts->k > (gram ? 4 : 16) || ts->k < b)) return false;
    const size_t extra = rows_extra_bytes(g0, b, ts, gram);
    const StreamGeom g = rows_geom(c, g0, extra);
    if (ts && ts->Rparts && g.rc > kRowsFused) return false;  // tiny n: separate TSQR pass
    if (g.stages * g.stage_bytes + bar_bytes(g.stages) + extra > c.smem_optin) return false;
    if (gram && sizeof(double) * 8 * b * g0.n > static_cast<size_t>(g.stages) * g.stage_bytes) return false;
    return true;
}

// ---- warp-pair one-pass kernel -------------------------------------------
int pair_pl(int n) {
    const int half = ((n + 1) / 2 + 1) / 2;
    const int pl = (half + 31) / 32;
    return pl <= 4 ? 4 : (pl <= 8 ? 8 : (pl <= 16 ? 16 : 32));
}

StreamGeom pair_geom(const Ctx& c, StreamGeom g) {
    const int64_t row_bytes = static_cast<int64_t>(g.ld_s) * 8;
    const int64_t target = env_int("MSVD_PAIR_STAGE_KB", 8) * 1024;
    g.rc = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(target / row_bytes, 64)));
    g.stage_bytes = ((static_cast<size_t>(g.rc) * row_bytes + 127) / 128) * 128;
    const int64_t avail = static_cast<int64_t>(c.smem_optin) - 2048;
    const int64_t budget = std::min<int64_t>(env_int("MSVD_PAIR_BUDGET_KB", 168) * 1024, avail);
    // stages a multiple of 4: a stage is only ever consumed by one pair, in order
    const int64_t per_pair = std::max<int64_t>(2, std::min<int64_t>(8, budget / (4 * static_cast<int64_t>(g.stage_bytes))));
    g.stages = static_cast<int32_t>(4 * per_pair);
    return g;
}

// b * (register pairs per lane) <= 16 keeps W, the accumulators and the
// half-row values in registers
bool pair_ok(const Ctx& c, const StreamGeom& g0, int b, bool ex) {
    if (!g0.tma || b < 1 || b > 4 || std::getenv("MSVD_NO_PAIR")) return false;
    const int bg = b + (ex ? 1 : 0);
    if (bg * pair_pl(g0.n) > 16) return false;
    const StreamGeom g = pair_geom(c, g0);
    if (g.stages * g.stage_bytes + bar_bytes(g.stages) + 1024 > c.smem_optin) return false;
    return sizeof(double) * 4 * bg * g0.n <= static_cast<size_t>(g.stages) * g.stage_bytes;
}

template <int B, int PL, bool EX = false>
void apply_pair_b(Ctx& c, const ApplyArgs& a) {
    optin_smem(c, apply_pair_kernel<B, PL, EX>);
    const size_t sm = bar_bytes(a.g.stages) + 128 * ((sizeof(double) * 16 * B + 127) / 128) + a.g.stages * a.g.stage_bytes;
    apply_pair_kernel<B, PL, EX><<<a.g.grid, 256, sm, c.stream>>>(a);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    c.paths |= EX ? kPathPairEx : kPathPair;
}

void launch_pair(Ctx& c, const ApplyArgs& a0, int b) {
    ApplyArgs a = a0;
    a.g = pair_geom(c, a0.g);
    const int pl = pair_pl(a0.g.n);
    switch (b * 100 + pl) {
        case 104: apply_pair_b<1, 4>(c, a); break;
        case 108: apply_pair_b<1, 8>(c, a); break;
        case 116: apply_pair_b<1, 16>(c, a); break;
        case 204: apply_pair_b<2, 4>(c, a); break;
        case 208: apply_pair_b<2, 8>(c, a); break;
        case 304: apply_pair_b<3, 4>(c, a); break;
        case 404: apply_pair_b<4, 4>(c, a); break;
        default: fail(MSVD_ERR_INVALID, "msvd: one-pass pair kernel on an unsupported shape");
    }
}

// true if launched (the fused TSQR, when requested, was then done too)
bool try_apply_rows(Ctx& c, const ApplyArgs& a0, int b) {
    if (!rows_ok(c, a0.g, b, &a0.ts, a0.gpart != nullptr)) return false;
    const int npairs = (a0.g.n + 1) / 2;
    const int pl = (npairs + 31) / 32;
    ApplyArgs a = a0;
    a.g = rows_geom(c, a0.g, rows_extra_bytes(a0.g, b, &a0.ts, a0.gpart != nullptr));
    if (b == 1) {
        if (pl <= 4) return apply_rows_km<1, 4>(c, a), true;
        if (pl <= 8) return apply_rows_km<1, 8>(c, a), true;
        if (pl <= 16) return apply_rows_km<1, 16>(c, a), true;
        if (pl <= 32) return apply_rows_km<1, 32>(c, a), true;
    } else if (b == 2) {
        if (pl <= 4) return apply_rows_km<2, 4>(c, a), true;
        if (pl <= 8) return apply_rows_km<2, 8>(c, a), true;
        if (pl <= 16) return apply_rows_km<2, 16>(c, a), true;
    } else if (b == 4 || b == 3) {
        if (pl <= 4) return (b == 4 ? apply_rows_km<4, 4>(c, a) : apply_rows_km<3, 4>(c, a)), true;
        if (pl <= 8) return (b == 4 ? apply_rows_km<4, 8>(c, a) : apply_rows_km<3, 8>(c, a)), true;
    }
    return false;
}

template <int B>
void apply_b(Ctx& c, const ApplyArgs& a) {
    const size_t sm = apply_smem(a.g);
    optin_smem(c, apply_kernel<B>);
    apply_kernel<B><<<a.g.grid, 32 + kConsumers, sm, c.stream>>>(a);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    c.paths |= kPathTicket;
}

template <int B>
void gram_b(Ctx& c, const GramArgs& a) {
    const size_t sm = gram_smem(a.g, B);
    optin_smem(c, gram_kernel<B>);
    gram_kernel<B><<<a.g.grid, 64 + kConsumers, sm, c.stream>>>(a);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    c.paths |= kPathGram;
}

}  // namespace

StreamGeom make_geom(const Ctx& c, const double* A, int64_t m, int32_t n, int64_t ld) {
    if (n < 1 || n > kMaxN)
        fail(MSVD_ERR_DIMENSION, "msvd: column count " + std::to_string(n) +
                                     " outside the supported range [1, " + std::to_string(kMaxN) + "]");
    StreamGeom g{};
    g.A = A;
    g.m = m;
    g.n = n;
    g.ld = ld;
    g.tma = (ld % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) ? 1 : 0;
    g.ld_s = g.tma ? static_cast<int32_t>(ld) : static_cast<int32_t>((n + 1) & ~1);
    const int64_t row_bytes = static_cast<int64_t>(g.ld_s) * 8;
    if (row_bytes > kStageBudget / 2)
        fail(MSVD_ERR_DIMENSION, "msvd: leading dimension too large for the stream pipeline");
    const int64_t target = env_int("MSVD_STAGE_KB", kStageTarget / 1024) * 1024;
    const int64_t budget = env_int("MSVD_STAGE_BUDGET_KB", kStageBudget / 1024) * 1024;
    g.rc = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(target / row_bytes, 64)));
    g.stage_bytes = ((static_cast<size_t>(g.rc) * row_bytes + 127) / 128) * 128;
    g.stages = static_cast<int32_t>(std::max<size_t>(2, std::min<size_t>(8, budget / g.stage_bytes)));
    g.grid = c.num_sms * static_cast<int32_t>(env_int("MSVD_CTAS_PER_SM", 1));
    return g;
}

bool apply_gram_supported(const Ctx& c, const StreamGeom& g, int b, const TsqrFuse* fuse) {
    const int pl = ((g.n + 1) / 2 + 31) / 32;
    const int plt = pl <= 4 ? 4 : (pl <= 8 ? 8 : (pl <= 16 ? 16 : 32));  // the PL template the launch picks
    if (b * plt <= 16 && rows_ok(c, g, b, fuse, true)) return true;
    return !fuse && pair_ok(c, g, b, false);  // the pair kernel has no fused TSQR
}

// b = 1 pass that also accumulates A^T e for an m-vector e: gpart[grid][2][n]
// = [A_cta^T (A_cta w), A_cta^T e_cta] (the one-pass check refresh)
// team geometry: stages a multiple of the team count
constexpr int kTeam = 4;
int team_pl(int n) {
    const int part = ((n + 1) / 2 + kTeam - 1) / kTeam;
    const int pl = (part + 31) / 32;
    return pl <= 2 ? 2 : (pl <= 4 ? 4 : (pl <= 8 ? 8 : 16));
}
// kTeamRows rows per stage (one team barrier per stage), as many stages per
// team as the shared memory holds
StreamGeom team_geom(const Ctx& c, StreamGeom g) {
    const int64_t row_bytes = static_cast<int64_t>(g.ld_s) * 8;
    g.rc = kTeamRows;
    g.stage_bytes = ((static_cast<size_t>(g.rc) * row_bytes + 127) / 128) * 128;
    const int64_t xbytes = sizeof(double) * (8 / kTeam) * 2 * kTeam * kTeamRows * 4;  // b <= 4
    const int64_t avail = static_cast<int64_t>(c.smem_optin) - 2048 - xbytes;
    const int64_t per_team =
        std::max<int64_t>(2, std::min<int64_t>(8, avail / ((8 / kTeam) * static_cast<int64_t>(g.stage_bytes))));
    g.stages = static_cast<int32_t>((8 / kTeam) * per_team);
    return g;
}
bool team_ok(const Ctx& c, const StreamGeom& g0, int b) {
    if (!g0.tma || b < 2 || b > 4 || std::getenv("MSVD_NO_PAIR")) return false;
    if (b * team_pl(g0.n) > 8) return false;  // b = 2 to n = 1024, b = 3, 4 to n = 512
    const StreamGeom g = team_geom(c, g0);
    const size_t xbytes = sizeof(double) * (8 / kTeam) * 2 * kTeam * kTeamRows * 4;
    if (g.stages * g.stage_bytes + bar_bytes(g.stages) + xbytes + 1024 > c.smem_optin) return false;
    return sizeof(double) * (8 / kTeam) * 2 * b * g0.n <= static_cast<size_t>(g.stages) * g.stage_bytes;
}

bool apply_ex_supported(const Ctx& c, const StreamGeom& g, int b) {
    return b == 1 ? pair_ok(c, g, 1, true) : team_ok(c, g, b);
}

bool launch_apply_ex(Ctx& c, const StreamGeom& g, const double* W, int b, OutCols out, const double* ex,
                     int64_t ld_ex, double* gpart, const TsqrFuse* fuse) {
    if (!apply_ex_supported(c, g, b)) fail(MSVD_ERR_INVALID, "msvd: A*W + A^T e pass on an unsupported shape");
    if (g.m == 0) {
        MSVD_CUDA(cudaMemsetAsync(gpart, 0, sizeof(double) * g.grid * 2 * b * g.n, c.stream));
        return false;
    }
    ProfScope prof(c, kProfApply);
    if (b >= 2) {
        ApplyArgs a{team_geom(c, g), W, out, TsqrFuse{}, gpart, nullptr};
        Cols ec{};
        for (int j = 0; j < b; ++j) ec.p[j] = ex + j * ld_ex;
        const size_t sm = bar_bytes(a.g.stages) +
                          128 * ((sizeof(double) * (8 / kTeam) * 2 * kTeam * kTeamRows * 4 + 127) / 128) +
                          a.g.stages * a.g.stage_bytes;
        auto go = [&](auto kernel) {
            optin_smem(c, kernel);
            kernel<<<a.g.grid, 256, sm, c.stream>>>(a, ec);
        };
        const int pl = team_pl(g.n);
        if (b == 2 && pl <= 2) go(apply_team_ex_kernel<2, 2, kTeam>);
        else if (b == 2) go(apply_team_ex_kernel<2, 4, kTeam>);
        else if (b == 3) go(apply_team_ex_kernel<3, 2, kTeam>);
        else go(apply_team_ex_kernel<4, 2, kTeam>);
        MSVD_CUDA(cudaGetLastError());
        ++c.launches;
        c.paths |= kPathTeamEx;
        return false;
    }
    // single-warp form with the fused TSQR when e is its first trial column
    // (the TSQR prefetch brings e's rows) and [8][2][n] fits the stage ring
    if (std::getenv("MSVD_EX_SINGLE") && fuse && fuse->Rparts && fuse->k <= 4 && fuse->k > 1 && fuse->T.p[0] == ex &&
        g.tma && !std::getenv("MSVD_APPLY_PRODUCER") && rows_ok(c, g, 1, fuse, true)) {
        const int npairs = (g.n + 1) / 2;
        const int pl = (npairs + 31) / 32;
        ApplyArgs a1{g, W, out, *fuse, gpart, nullptr};
        a1.g = rows_geom(c, g, rows_extra_bytes(g, 1, fuse, true));
        if (sizeof(double) * 8 * 2 * g.n <= static_cast<size_t>(a1.g.stages) * a1.g.stage_bytes) {
            if (pl <= 4) return apply_rows_b<1, 4, 4, true, true>(c, a1), true;
            if (pl <= 8) return apply_rows_b<1, 8, 4, true, true>(c, a1), true;
            if (pl <= 16) return apply_rows_b<1, 16, 4, true, true>(c, a1), true;
        }
    }
    ApplyArgs a{pair_geom(c, g), W, out, TsqrFuse{}, gpart, ex};
    switch (pair_pl(g.n)) {
        case 4: apply_pair_b<1, 4, true>(c, a); break;
        case 8: apply_pair_b<1, 8, true>(c, a); break;
        default: fail(MSVD_ERR_INVALID, "msvd: A*W + A^T e pass on an unsupported shape");
    }
    return false;
}

bool launch_apply(Ctx& c, const StreamGeom& g, const double* W, int b, OutCols out, const TsqrFuse* fuse,
                  double* gpart) {
    if (g.m == 0) {
        if (gpart) MSVD_CUDA(cudaMemsetAsync(gpart, 0, sizeof(double) * g.grid * b * g.n, c.stream));
        return false;
    }
    ProfScope prof(c, kProfApply);
    TsqrFuse none{};
    if (try_apply_rows(c, ApplyArgs{g, W, out, fuse ? *fuse : none, gpart, nullptr}, b)) return fuse != nullptr;
    if (gpart && pair_ok(c, g, b, false)) {  // one-pass, rows split over warp pairs (no fused TSQR)
        launch_pair(c, ApplyArgs{g, W, out, none, gpart, nullptr}, b);
        return false;
    }
    if (gpart) fail(MSVD_ERR_INVALID, "msvd: one-pass A*W / A^T A W launch on an unsupported shape");
    // ticket variant: large stages amortize the per-chunk cross-warp finish
    // (measured: 48 KB x 3 stages best at n = 2000, b = 5)
    ApplyArgs a{cap_rows(rechunk(g, 48, 144), kRedSlots / std::max(1, b)), W, out, none, nullptr};
    switch (b) {
        case 1: apply_b<1>(c, a); break;
        case 2: apply_b<2>(c, a); break;
        case 3: apply_b<3>(c, a); break;
        case 4: apply_b<4>(c, a); break;
        case 5: apply_b<5>(c, a); break;
        case 6: apply_b<6>(c, a); break;
        case 7: apply_b<7>(c, a); break;
        case 8: apply_b<8>(c, a); break;
        default: fail(MSVD_ERR_DIMENSION, "msvd: block size above 8 is not supported");
    }
    return false;
}

void launch_gram(Ctx& c, const StreamGeom& g, Cols T, int k, const double* Cm, int q, int b,
                 OutCols out, bool direct, double* Gpart, const int* skip) {
    ProfScope prof(c, kProfGram);
    // stage geometry by block size (tuning sweep, profiles/README.md):
    // b = 1: 32 KB x 3, b = 2: 48 KB x 3, b >= 3: 64 KB x 2
    const StreamGeom gg = b == 1 ? rechunk(g, 32, 96) : (b == 2 ? rechunk(g, 48, 144) : rechunk(g, 64, 128));
    GramArgs a{gg, T, k, Cm, q, out, direct ? 1 : 0, Gpart, skip};
    if (g.m == 0) {
        MSVD_CUDA(cudaMemsetAsync(Gpart, 0, sizeof(double) * g.grid * b * g.n, c.stream));
        return;
    }
    switch (b) {
        case 1: gram_b<1>(c, a); break;
        case 2: gram_b<2>(c, a); break;
        case 3: gram_b<3>(c, a); break;
        case 4: gram_b<4>(c, a); break;
        case 5: gram_b<5>(c, a); break;
        case 6: gram_b<6>(c, a); break;
        case 7: gram_b<7>(c, a); break;
        case 8: gram_b<8>(c, a); break;
        default: fail(MSVD_ERR_DIMENSION, "msvd: block size above 8 is not supported");
    }
}

}  // namespace msvd
