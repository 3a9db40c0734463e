// K3 one-pass kernel with split warp roles (b = 2..4): apply_split_kernel.
//
// The one-pass pass forms, per row a of A, y = a W (b dot products over n) and
// then acc += a^T y (a rank-one update of the n x b accumulator of
// A^T (A W)).  The warp-pair and team kernels (stream_pair.cu) do both in the
// same warps: W, the accumulators and the row values all live in one warp's
// registers (8 warps per SM at ~220 registers), and the dot products' shuffle
// chain and the cross-warp barrier sit on every warp's critical path -- the
// b = 4 pass stalls at 0.56-0.69 of the copy peak with the FP64 pipe under 40%.
//
// Here the two halves of the work run in different warps:
//   * DOT warps hold only W (their part of the row): per stage they form the
//     partial dot products of RG rows at a time, transpose-reduce them across
//     the lanes and leave the per-member partials in shared memory, then arrive
//     on the stage's `ydone` mbarrier;
//   * ACC warps hold only the accumulators (their part of the columns): they
//     wait for `ydone`, sum the members' partials in member order (the same
//     bits in every warp), and stream the rows once more from shared memory
//     into the accumulators -- no shuffles, no barrier among them;
//   * the LAST of a stage's DOT and ACC warps to finish with it (a shared-memory
//     ticket) refills it: 1-D TMA bulk copy, mbarrier complete_tx.  No producer
//     warp and no empty barrier.
// G groups of (TD dot + TA acc) warps work on stages c % G, so 12-16 warps of
// 128-168 registers are resident instead of 8 (registers are allotted per four
// warps: 16 warps leave 128 each) and the reduction latency of one group hides
// behind the streaming FMAs of the others.
//
// With EX (the check refresh, solver.cpp:439 on the next pass) a second set of
// ACC warps accumulates A^T E for the b columns E = A V' of the previous check
// iterate (they take E from global memory and never wait for the DOT warps):
// gpart holds [grid][2b][n].
//
// Every sum has a fixed order: the pass is bitwise repeatable.
#include <string>
#include <type_traits>

#include "stream_impl.cuh"

namespace msvd {
namespace strm {
namespace {

constexpr int kSplitMaxRc = 8;  // rows per stage cap
constexpr int kYSlots = 32;    // y values per (stage, member): rc * Bp <= 32, one lane each

struct SplitSmem {
    uint64_t* full;
    uint64_t* ydone;
    unsigned* ticket;  // per stage: warps done with it
    double* ypart;  // [stages][TD][kYSlots]
    double* ebuf;   // [acc warps][kYSlots]: the warp's coefficient rows (summed y, or E)
    unsigned char* stage0;
};

__host__ __device__ constexpr size_t split_bar_bytes(int stages) {
    return ((24 * static_cast<size_t>(stages) + 127) / 128) * 128;
}
__host__ __device__ constexpr size_t split_extra_bytes(int stages, int td, int acc_warps) {
    return ((sizeof(double) * (static_cast<size_t>(stages) * td + acc_warps) * kYSlots + 127) / 128) * 128;
}

// partial dot products of RG rows starting at `rows` (nr of them valid) against the
// lane's W entries: lane partials in v[q * Bp + j]
template <int B, int Bp, int PLD, int RG, bool ODD, bool FULLG>
__device__ __forceinline__ void split_dots(const double* rows, int nr, int ld_s, const int (&off)[PLD],
                                           const bool (&keepy)[PLD], const double (&w)[PLD][2][B],
                                           double (&v)[RG * Bp]) {
#pragma unroll
    for (int q = 0; q < RG; ++q) {
        const double* row = rows + static_cast<int64_t>(FULLG || q < nr ? q : 0) * ld_s;
#pragma unroll
        for (int i = 0; i < PLD; ++i) {
            double2 x = *reinterpret_cast<const double2*>(row + off[i]);
            if (ODD) x.y = keepy[i] ? x.y : 0.0;  // odd n: the pad column is not A
#pragma unroll
            for (int j = 0; j < B; ++j) {
                const int t = q * Bp + j;
                v[t] = i == 0 ? x.x * w[0][0][j] : fma(x.x, w[i][0][j], v[t]);
                v[t] = fma(x.y, w[i][1][j], v[t]);
            }
        }
        if (!FULLG && q >= nr) {
#pragma unroll
            for (int j = 0; j < B; ++j) v[q * Bp + j] = 0.0;
        }
    }
}

template <int B, int PLD, int PLA, int TD, int TA, int G, int RG, bool EX>
__global__ void __launch_bounds__(32 * G * (TD + TA), 1) apply_split_kernel(ApplyArgs a, Cols ex) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int Bp = B <= 2 ? 2 : 4;  // y slots per row
    constexpr int NV = RG * Bp;         // values per transpose-reduce
    constexpr int BG = EX ? 2 * B : B;  // accumulated columns
    constexpr int NDOT = G * TD, NACC = G * TA;
    constexpr int NT = 32 * (NDOT + NACC);
    static_assert(NV >= 2 && NV <= 32 && (NV & (NV - 1)) == 0, "transpose-reduce width");
    const StreamGeom& g = a.g;
    SplitSmem p;
    p.full = reinterpret_cast<uint64_t*>(smem);
    p.ydone = p.full + g.stages;
    p.ticket = reinterpret_cast<unsigned*>(p.ydone + g.stages);
    p.ypart = reinterpret_cast<double*>(smem + split_bar_bytes(g.stages));
    p.ebuf = p.ypart + static_cast<size_t>(g.stages) * TD * kYSlots;
    p.stage0 = smem + split_bar_bytes(g.stages) + split_extra_bytes(g.stages, TD, NACC);
    int64_t r_begin, r_end;
    cta_rows(g.m, r_begin, r_end);
    if (threadIdx.x == 0) {
        for (int s = 0; s < g.stages; ++s) {
            mbar_init(&p.full[s], 1);
            mbar_init(&p.ydone[s], TD);
            p.ticket[s] = 0;
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int cw = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nchunks = ceil_div(r_end - r_begin, g.rc);
    const int n = g.n;
    const int npairs = (n + 1) >> 1;

    const uint64_t pol = l2_evict_first_policy();
    auto issue = [&](int64_t c, int s) {
        const int64_t r0 = r_begin + c * g.rc;
        const int64_t rc = min(static_cast<int64_t>(g.rc), r_end - r0);
        const uint32_t bytes = static_cast<uint32_t>(rc * g.ld * 8);
        mbar_arrive_expect_tx(&p.full[s], bytes);
        bulk_g2s(p.stage0 + s * g.stage_bytes, g.A + r0 * g.ld, bytes, &p.full[s], pol);
    };
    // a warp is done with chunk c in stage s: the last of the stage's TD + TA warps refills it
    auto release = [&](int64_t c, int s) {
        unsigned old;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(&p.ticket[s])) : "memory");
        if (old == TD + TA - 1) {
            p.ticket[s] = 0;
            if (c + g.stages < nchunks) issue(c + g.stages, s);
        }
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < g.stages && s < nchunks; ++s) issue(s, s);

    if (cw < NDOT) {
        // ---- dot warps: member hd of group grp, column pairs [p0, pend) ----
        const int grp = cw / TD, hd = cw % TD;
        const int part = (npairs + TD - 1) / TD;
        const int p0 = hd * part;
        const int pend = min(npairs, p0 + part);
        double w[PLD][2][B];
        int off[PLD];  // element offset of slot i's column pair (lanes past the part re-read a pair with zero weights)
        bool keepy[PLD];
#pragma unroll
        for (int i = 0; i < PLD; ++i) {
            const int pi = p0 + lane + 32 * i;
            const bool mine = pi < pend;
            const int pc = mine ? pi : max(0, min(npairs - 1, pend - 1));
            off[i] = 2 * pc;
            keepy[i] = 2 * pc + 1 < n;
#pragma unroll
            for (int j = 0; j < B; ++j) {
                w[i][0][j] = mine ? a.W[2 * pc + static_cast<int64_t>(j) * n] : 0.0;
                w[i][1][j] = mine && keepy[i] ? a.W[2 * pc + 1 + static_cast<int64_t>(j) * n] : 0.0;
            }
        }
        const bool odd = n & 1;
        int s = grp;
        uint32_t ph = 0;
        for (int64_t c = grp; c < nchunks; c += G) {
            mbar_wait(&p.full[s], ph);
            const double* As = reinterpret_cast<const double*>(p.stage0 + s * g.stage_bytes);
            const int64_t r0 = r_begin + c * g.rc;
            const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
            double* yp = p.ypart + (static_cast<size_t>(s) * TD + hd) * kYSlots;
            for (int r = 0; r < rc; r += RG) {
                double v[NV];
#pragma unroll
                for (int t = 0; t < NV; ++t) v[t] = 0.0;
                const double* rows = As + static_cast<int64_t>(r) * g.ld_s;
                const int nr = rc - r;
                if (nr >= RG) {
                    if (odd) split_dots<B, Bp, PLD, RG, true, true>(rows, RG, g.ld_s, off, keepy, w, v);
                    else split_dots<B, Bp, PLD, RG, false, true>(rows, RG, g.ld_s, off, keepy, w, v);
                } else {
                    split_dots<B, Bp, PLD, RG, true, false>(rows, nr, g.ld_s, off, keepy, w, v);
                }
                const double sum = warp_transpose_reduce<NV>(v);  // slot lane % NV on every lane
                if (lane < NV) yp[r * Bp + lane] = sum;
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&p.ydone[s]);  // release: the partials above are visible to the waiters
                release(c, s);             // this member is done with the stage's rows
            }
            s += G;
            if (s >= g.stages) {
                s -= g.stages;
                ph ^= 1;
            }
        }
    } else {
        // ---- acc warps: member ha of group grp, column pairs [p0, pend) ----
        // (no masks here: a pad column's or a re-read pair's accumulator is never stored)
        const int aw = cw - NDOT;
        const int grp = aw / TA, ha = aw % TA;
        // EX: the TA members are two sets of TA / 2 -- role 0 accumulates A^T (A W) (it needs the
        // dot warps' y), role 1 A^T E (E comes from global memory: it never waits for the dot
        // warps and runs ahead of them, bounded only by the stage ring)
        constexpr int TAH = EX ? TA / 2 : TA;
        const int role = EX ? ha / TAH : 0, hh = ha % TAH;
        const int part = (npairs + TAH - 1) / TAH;
        const int p0 = hh * part;
        const int pend = min(npairs, p0 + part);
        double ga[PLA][2][B];
        int off[PLA];
        bool keepy[PLA], mine[PLA];
#pragma unroll
        for (int i = 0; i < PLA; ++i) {
            const int pi = p0 + lane + 32 * i;
            mine[i] = pi < pend;
            const int pc = mine[i] ? pi : max(0, min(npairs - 1, pend - 1));
            off[i] = 2 * pc;
            keepy[i] = 2 * pc + 1 < n;
#pragma unroll
            for (int j = 0; j < B; ++j) ga[i][0][j] = ga[i][1][j] = 0.0;
        }
        // this warp's copy of the stage's coefficient rows -- y (the members' partials summed
        // once per stage) or, role 1, its E rows: [row][Bp], read back as broadcasts
        double* cb = p.ebuf + static_cast<size_t>(aw) * kYSlots;
        // role 1: lane l = row * Bp + j of the chunk's E values, one chunk ahead
        double en = 0.0;
        auto ex_load = [&](int64_t cc) {
            if (!EX || cc >= nchunks) return;
            const int64_t rr0 = r_begin + cc * g.rc;
            const int rcc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - rr0));
            const int row = lane / Bp, j = lane % Bp;
            en = (row < rcc && j < B) ? ex.p[j][rr0 + row] : 0.0;
        };
        if (role == 1) ex_load(grp);
        int s = grp;
        uint32_t ph = 0;
        for (int64_t c = grp; c < nchunks; c += G) {
            const int64_t r0 = r_begin + c * g.rc;
            const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
            if (role == 1) {
                cb[lane] = en;  // (the previous chunk's reads ended at its closing __syncwarp)
                ex_load(c + G);
            } else {
                mbar_wait(&p.ydone[s], ph);
            }
            mbar_wait(&p.full[s], ph);  // this warp's own acquire of the TMA-written rows
            if (role == 0) {
                const double* yp = p.ypart + static_cast<size_t>(s) * TD * kYSlots;
                double t = yp[lane];
#pragma unroll
                for (int mm = 1; mm < TD; ++mm) t += yp[mm * kYSlots + lane];  // members in order: the same bits in every warp
                cb[lane] = t;
                const int row = lane / Bp, j = lane % Bp;
                if (hh == 0 && row < rc && j < B) a.out.p[j][r0 + row] = t;  // the chunk's y = A W rows
            }
            __syncwarp();
            const double* As = reinterpret_cast<const double*>(p.stage0 + s * g.stage_bytes);
#pragma unroll 2
            for (int r = 0; r < rc; ++r) {
                double y[Bp];
#pragma unroll
                for (int j2 = 0; j2 < Bp; j2 += 2) {
                    const double2 t = *reinterpret_cast<const double2*>(cb + r * Bp + j2);
                    y[j2] = t.x;
                    y[j2 + 1] = t.y;
                }
                const double* row = As + static_cast<int64_t>(r) * g.ld_s;
#pragma unroll
                for (int i = 0; i < PLA; ++i) {
                    const double2 x = *reinterpret_cast<const double2*>(row + off[i]);
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        ga[i][0][j] = fma(x.x, y[j], ga[i][0][j]);
                        ga[i][1][j] = fma(x.y, y[j], ga[i][1][j]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) release(c, s);
            s += G;
            if (s >= g.stages) {
                s -= g.stages;
                ph ^= 1;
            }
        }
        named_sync(1, NT);  // (1) every chunk consumed: the stage ring is free
        double* red = reinterpret_cast<double*>(p.stage0);  // [G][BG][n]
#pragma unroll
        for (int i = 0; i < PLA; ++i) {
            if (!mine[i]) continue;
            const int c0 = off[i];
#pragma unroll
            for (int j = 0; j < B; ++j) {
                red[(static_cast<size_t>(grp) * BG + role * B + j) * n + c0] = ga[i][0][j];
                if (keepy[i]) red[(static_cast<size_t>(grp) * BG + role * B + j) * n + c0 + 1] = ga[i][1][j];
            }
        }
    }
    if (cw < NDOT) named_sync(1, NT);  // (1) for the dot warps
    named_sync(1, NT);  // (2) the groups' accumulators are in shared memory
    const double* red = reinterpret_cast<const double*>(p.stage0);
    double* gp = a.gpart + static_cast<size_t>(blockIdx.x) * BG * n;
    for (int i = threadIdx.x; i < BG * n; i += blockDim.x) {
        double sum = red[i];
#pragma unroll
        for (int q = 1; q < G; ++q) sum += red[static_cast<size_t>(q) * BG * n + i];
        gp[i] = sum;
    }
}

template <int B, int PL, int G, bool EX>
void split_launch(Ctx& c, const ApplyArgs& a, const Cols& ec) {
    constexpr int TD = 2, TA = EX ? 4 : 2;
    constexpr int PLA = PL;  // EX: two sets of two acc warps (A^T A W and A^T E), half a row each
    constexpr int RG = (B == 2 && PL == 8) ? 2 : 4;
    auto kernel = apply_split_kernel<B, PL, PLA, TD, TA, G, RG, EX>;
    optin_smem(c, kernel);
    const size_t sm = split_bar_bytes(a.g.stages) + split_extra_bytes(a.g.stages, TD, G * TA) +
                      a.g.stages * a.g.stage_bytes;
    kernel<<<a.g.grid, 32 * G * (TD + TA), sm, c.stream>>>(a, ec);
    MSVD_CUDA(cudaGetLastError());
    ++c.launches;
    c.paths |= EX ? kPathSplitEx : kPathSplit;
}

}  // namespace

// lanes' column pairs per dot warp (half a row): 1, 2, 4 or 8
int split_pl(int n) {
    const int half = ((n + 1) / 2 + 1) / 2;
    const int pl = (half + 31) / 32;
    return pl <= 1 ? 1 : (pl <= 2 ? 2 : (pl <= 4 ? 4 : (pl <= 8 ? 8 : 16)));
}

int split_groups(bool ex) {
    // measured (B200, msvd_aw_gram): three groups on 32 KB stages beat four on 16 KB
    // (b = 4, n = 500: 6.6 vs 6.2 TB/s; b = 2, n = 1000: 7.1 vs 6.8)
    return static_cast<int>(ex ? 2 : (env_int("MSVD_SPLIT_GROUPS", 3) == 4 ? 4 : 3));
}

// stages of ~32 KB: rc rows (a multiple of the reduce group, rc * Bp <= 32),
// as many stages per group as shared memory holds (2..4)
StreamGeom split_geom(const Ctx& c, StreamGeom g, int b, bool ex) {
    const int G = split_groups(ex);
    const int pl = split_pl(g.n);
    const int rg = (b == 2 && pl == 8) ? 2 : 4;
    const int bp = b <= 2 ? 2 : 4;
    const int64_t row_bytes = static_cast<int64_t>(g.ld_s) * 8;
    const int64_t target = env_int("MSVD_SPLIT_STAGE_KB", 32) * 1024;
    int64_t rc = std::max<int64_t>(rg, (target / row_bytes) / rg * rg);
    rc = std::min<int64_t>(rc, std::min<int64_t>(kSplitMaxRc, kYSlots / bp));
    g.rc = static_cast<int32_t>(rc);
    g.stage_bytes = ((static_cast<size_t>(g.rc) * row_bytes + 127) / 128) * 128;
    const int64_t avail = static_cast<int64_t>(c.smem_optin) - 1024 - static_cast<int64_t>(split_bar_bytes(4 * G)) -
                          static_cast<int64_t>(split_extra_bytes(4 * G, 2, 4 * G));
    const int64_t per_group = std::min<int64_t>(env_int("MSVD_SPLIT_DEPTH", 4), avail / (G * static_cast<int64_t>(g.stage_bytes)));
    g.stages = static_cast<int32_t>(G * std::max<int64_t>(per_group, 0));
    return g;
}

bool split_ok(const Ctx& c, const StreamGeom& g0, int b, bool ex) {
    if (!g0.tma || b < 2 || b > 4 || g0.n > kMaxN || std::getenv("MSVD_NO_SPLIT")) return false;
    const int pl = split_pl(g0.n);
    if (b * pl > 16) return false;  // W of half a row in a dot warp's registers
    const StreamGeom g = split_geom(c, g0, b, ex);
    const int G = split_groups(ex);
    if (g.stages < 2 * G) return false;
    // the groups' accumulators are summed through the idle stage ring
    return sizeof(double) * G * (ex ? 2 : 1) * b * g0.n <= static_cast<size_t>(g.stages) * g.stage_bytes;
}

void launch_split(Ctx& c, const ApplyArgs& a0, int b, const Cols* ex) {
    ApplyArgs a = a0;
    const bool isex = ex != nullptr;
    a.g = split_geom(c, a0.g, b, isex);
    const Cols ec = ex ? *ex : Cols{};
    const int pl = split_pl(a0.g.n);
    const int G = split_groups(isex);
    const int key = ((b * 100 + pl) * 10 + G) * 2 + (isex ? 1 : 0);
#define MSVD_SPLIT_CASE(B_, PL_, G_, EX_) \
    case ((B_ * 100 + PL_) * 10 + G_) * 2 + (EX_ ? 1 : 0): split_launch<B_, PL_, G_, EX_>(c, a, ec); break;
#define MSVD_SPLIT_BPL(B_, PL_)        \
    MSVD_SPLIT_CASE(B_, PL_, 4, false) \
    MSVD_SPLIT_CASE(B_, PL_, 3, false) \
    MSVD_SPLIT_CASE(B_, PL_, 2, true)
    switch (key) {
        MSVD_SPLIT_BPL(2, 1)
        MSVD_SPLIT_BPL(2, 2)
        MSVD_SPLIT_BPL(2, 4)
        MSVD_SPLIT_BPL(2, 8)
        MSVD_SPLIT_BPL(3, 1)
        MSVD_SPLIT_BPL(3, 2)
        MSVD_SPLIT_BPL(3, 4)
        MSVD_SPLIT_BPL(4, 1)
        MSVD_SPLIT_BPL(4, 2)
        MSVD_SPLIT_BPL(4, 4)
        default: fail(MSVD_ERR_INVALID, "msvd: split-role one-pass kernel on an unsupported shape");
    }
#undef MSVD_SPLIT_BPL
#undef MSVD_SPLIT_CASE
}

}  // namespace strm
}  // namespace msvd
