// K3 one-pass kernels that split a row over several warps: apply_pair_kernel
// (a warp pair, half a row each; with EX the b = 1 check refresh) and
// apply_team_ex_kernel (a team of four warps; the b = 2..4 check refresh);
// see stream_impl.cuh.
#include "stream_impl.cuh"

namespace msvd {
namespace strm {
namespace {


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

// EX = false: the plain one-pass pass (A W and A^T (A W)) in the same
// four-rows-per-barrier form, for b = 3, 4 where the warp-pair kernel's
// per-row barrier and butterflies cap it at ~0.55 of the HBM roofline (C4).
template <int B, int PL, int T, bool EX = true>
__global__ void __launch_bounds__(256, 1) apply_team_ex_kernel(ApplyArgs a, Cols ex) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int TEAMS = 8 / T;
    constexpr int BG = EX ? 2 * B : B;
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
        if (!EX || cc >= nchunks) return;
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
                    e[j] = EX ? __shfl_sync(kFull, rr < 32 ? exc[0][j] : exc[1][j], rr & 31) : 0.0;
                }
#pragma unroll
                for (int i = 0; i < PL; ++i) {
                    double2 x = *reinterpret_cast<const double2*>(row + off[i]);
                    x.y = keepy[i] ? x.y : 0.0;
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        ga[i][0][j] = fma(x.x, y[j], ga[i][0][j]);
                        ga[i][1][j] = fma(x.y, y[j], ga[i][1][j]);
                        if constexpr (EX) {
                            ga[i][0][B + j] = fma(x.x, e[j], ga[i][0][B + j]);
                            ga[i][1][B + j] = fma(x.y, e[j], ga[i][1][B + j]);
                        }
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
        case 204: apply_pair_b<2, 4>(c, a); break;
        case 208: apply_pair_b<2, 8>(c, a); break;
        case 304: apply_pair_b<3, 4>(c, a); break;
        case 404: apply_pair_b<4, 4>(c, a); break;
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

void launch_team(Ctx& c, const ApplyArgs& a, int b, int T) {
    const size_t sm = bar_bytes(a.g.stages) + 128 * ((sizeof(double) * 2 * 8 * kTeamRows * 4 + 127) / 128) +
                      a.g.stages * a.g.stage_bytes;
    auto go = [&](auto kernel) {
        optin_smem(c, kernel);
        kernel<<<a.g.grid, 256, sm, c.stream>>>(a, Cols{});
    };
    const int pl = team_pl(a.g.n, T);
    if (T == 4) {
        if (b == 2 && pl <= 2) go(apply_team_ex_kernel<2, 2, 4, false>);
        else if (b == 2) go(apply_team_ex_kernel<2, 4, 4, false>);
        else if (b == 3) go(apply_team_ex_kernel<3, 2, 4, false>);
        else go(apply_team_ex_kernel<4, 2, 4, false>);
    } else {
        if (b == 2 && pl <= 4) go(apply_team_ex_kernel<2, 4, 2, false>);
        else if (b == 2) go(apply_team_ex_kernel<2, 8, 2, false>);
        else if (b == 3) go(apply_team_ex_kernel<3, 4, 2, false>);
        else go(apply_team_ex_kernel<4, 4, 2, false>);
    }
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    c.paths |= kPathTeam;
}

void launch_team_ex(Ctx& c, const ApplyArgs& a, Cols ec, int b) {
    const size_t sm = bar_bytes(a.g.stages) + 128 * ((sizeof(double) * 2 * 8 * kTeamRows * 4 + 127) / 128) +
                      a.g.stages * a.g.stage_bytes;
    auto go = [&](auto kernel) {
        optin_smem(c, kernel);
        kernel<<<a.g.grid, 256, sm, c.stream>>>(a, ec);
    };
    const int pl = team_pl(a.g.n);
    if (b == 2 && pl <= 2) go(apply_team_ex_kernel<2, 2, kTeam>);
    else if (b == 2) go(apply_team_ex_kernel<2, 4, kTeam>);
    else if (b == 3) go(apply_team_ex_kernel<3, 2, kTeam>);
    else go(apply_team_ex_kernel<4, 2, kTeam>);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    c.paths |= kPathTeamEx;
}

}  // namespace strm
}  // namespace msvd
