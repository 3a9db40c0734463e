// K3 one-pass kernel that splits a row over a warp pair, half a row each
// (apply_pair_kernel; b = 1: the rows too wide for one warp's registers, and
// with EX the b = 1 check refresh); see stream_impl.cuh.  b = 2..4 run the
// split-role kernel (stream_split.cu), which replaced this file's warp-pair and
// four-warp team forms for those block sizes in round 2.
#include "stream_impl.cuh"

namespace msvd {
namespace strm {
namespace {


// One-pass form for wide rows: a row is split across a warp PAIR (warp
// 2q + h takes the column pairs [h * half, (h + 1) * half)), so W, the
// A^T (A W) accumulators and the row values of half a row fit in registers
// where a whole row does not (b = 1 up to n = 2048).  Chunk c belongs to pair c % 4 and stage c % stages
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

template <int B, int PL, bool EX = false>
void apply_pair_b(Ctx& c, const ApplyArgs& a) {
    optin_smem(c, apply_pair_kernel<B, PL, EX>);
    const size_t sm = bar_bytes(a.g.stages) + 128 * ((sizeof(double) * 16 * B + 127) / 128) + a.g.stages * a.g.stage_bytes;
    apply_pair_kernel<B, PL, EX><<<a.g.grid, 256, sm, c.stream>>>(a);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    c.paths |= EX ? kPathPairEx : kPathPair;
}

}  // namespace

void launch_pair(Ctx& c, const ApplyArgs& a0, int b) {
    ApplyArgs a = a0;
    a.g = pair_geom(c, a0.g);
    const int pl = pair_pl(a0.g.n);
    switch (b * 100 + pl) {
        case 104: apply_pair_b<1, 4>(c, a); break;
        case 108: apply_pair_b<1, 8>(c, a); break;
        case 116: apply_pair_b<1, 16>(c, a); break;
        default: fail(MSVD_ERR_INVALID, "msvd: one-pass pair kernel on an unsupported shape");
    }
}

void launch_pair_ex(Ctx& c, const ApplyArgs& a) {
    switch (pair_pl(a.g.n)) {
        case 4: apply_pair_b<1, 4, true>(c, a); break;
        case 8: apply_pair_b<1, 8, true>(c, a); break;
        default: fail(MSVD_ERR_INVALID, "msvd: A*W + A^T e pass on an unsupported shape");
    }
}

}  // namespace strm
}  // namespace msvd
