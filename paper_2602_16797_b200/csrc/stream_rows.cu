// K3 narrow-block variants (one warp per row): apply_rows_kernel (producer
// warp) and apply_self_kernel (TMA rows, one-pass and fused TSQR forms); see
// stream_impl.cuh.
#include "stream_impl.cuh"

namespace msvd {
namespace strm {
namespace {

// K3, narrow-block variant (b small): every chunk is owned by ONE consumer
// warp (chunk c -> warp c mod 8), lanes own fixed column pairs and keep W in
// registers, and a row's b dot products are finished with warp butterflies.
// No cross-warp reduction at all; the ring is deep (many small stages), so
// the producer always has bytes in flight while each warp works on its chunk.

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
    // the fused TSQR exists for b = 1, k <= 4 only (the solver's trial block
    // [AV AX AW]); wider blocks measured faster with a separate TSQR pass, so
    // their fused instantiations (which also spilled) are not built
    if (a.gpart) {  // one-pass mode (B * PL <= 16: registers)
        if constexpr (B * PL <= 16) {
            if (!a.ts.Rparts) return apply_rows_b<B, PL, 0, true>(c, a);
            if constexpr (B == 1) return apply_rows_b<1, PL, 4, true>(c, a);
        }
        fail(MSVD_ERR_INVALID, "msvd: one-pass A*W / A^T A W launch on an unsupported shape");
    }
    if (!a.ts.Rparts) return apply_rows_b<B, PL, 0, false>(c, a);
    if constexpr (B == 1) return apply_rows_b<1, PL, 4, false>(c, a);
    fail(MSVD_ERR_INVALID, "msvd: fused TSQR launch on an unsupported shape");
}

}  // namespace

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

}  // namespace strm
}  // namespace msvd
