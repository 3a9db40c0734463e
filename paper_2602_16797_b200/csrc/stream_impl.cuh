// Shared pieces of the streaming passes over the tall row-major A (SURVEY 2.3
// K2/K3), split over translation units so the kernel families compile in
// parallel:
//   stream.cu         geometry, support queries and the launch entry points
//   stream_rows.cu    apply_rows_kernel / apply_self_kernel (one warp per row)
//   stream_pair.cu    apply_pair_kernel (b = 1: a warp pair per row; the b = 1 check refresh)
//   stream_split.cu   apply_split_kernel (b = 2..4 one-pass: dot, acc and producer warps)
//   stream_ticket.cu  apply_kernel (b >= 5) and gram_kernel (K2)
#pragma once

#include <cstdlib>

#include "common.cuh"
#include "fold.cuh"
#include "msvd_internal.h"

namespace msvd {
namespace strm {

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
static __device__ void produce(const StreamGeom& g, const Pipe& p, int64_t r_begin, int64_t r_end) {
    const int lane = threadIdx.x & 31;
    const int64_t nrows = r_end - r_begin;
    const int64_t nchunks = ceil_div(nrows, g.rc);
    if (g.tma && g.rowcopy) {
        // a column panel: the chunk's rows are ld-pitched segments of ld_s
        // doubles, one bulk copy per row, spread over the lanes; the expected
        // bytes are posted before any copy is issued
        const uint64_t pol = l2_evict_first_policy();
        const uint32_t row_bytes = static_cast<uint32_t>(g.ld_s) * 8u;
        int s = 0;
        uint32_t ph = 1;
        for (int64_t c = 0; c < nchunks; ++c) {
            if (c >= g.stages) mbar_wait(&p.empty[s], ph);
            const int64_t r0 = r_begin + c * g.rc;
            const int rc = static_cast<int>(min(static_cast<int64_t>(g.rc), r_end - r0));
            if (lane == 0) mbar_arrive_expect_tx(&p.full[s], row_bytes * static_cast<uint32_t>(rc));
            __syncwarp();
            for (int r = lane; r < rc; r += 32)
                bulk_g2s(p.stage0 + s * p.stage_bytes + static_cast<size_t>(r) * row_bytes, g.A + (r0 + r) * g.ld,
                         row_bytes, &p.full[s], pol);
            if (++s == g.stages) {
                s = 0;
                ph ^= 1;
            }
        }
        return;
    }
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
    int64_t wstride;  // ticket kernel, column panel: W's column stride (0: g.n)
    int accum;        // ticket kernel, column panel: out += the panel's A W (panels after the first)
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


constexpr int kRowsFused = 4;  // rows per chunk supported by the fused TSQR prefetch

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
    int64_t gstride;   // column panel: Gpart's (cta, column) row stride (0: g.n); a null
                       // out.p[j] skips that output (the panels after the first)
};

// ---- geometry helpers (stream.cu) ---------------------------------------
size_t apply_smem(const StreamGeom& g);
int64_t env_int(const char* name, int64_t dflt);
StreamGeom rechunk(StreamGeom g, int64_t target_kb, int64_t budget_kb);
StreamGeom cap_rows(StreamGeom g, int maxrc);
size_t gram_smem(const StreamGeom& g, int B);
size_t rows_extra_bytes(const StreamGeom& g0, int b, const TsqrFuse* ts, bool gram);
StreamGeom rows_geom(const Ctx& c, StreamGeom g, size_t extra);
bool rows_ok(const Ctx& c, const StreamGeom& g0, int b, const TsqrFuse* ts, bool gram);
int pair_pl(int n);
StreamGeom pair_geom(const Ctx& c, StreamGeom g);
bool pair_ok(const Ctx& c, const StreamGeom& g0, int b, bool ex);
// stream_split.cu: split-role one-pass kernel (dot / acc / producer warps), b = 2..4
bool split_ok(const Ctx& c, const StreamGeom& g0, int b, bool ex);
void launch_split(Ctx& c, const ApplyArgs& a0, int b, const Cols* ex);  // ex: the check refresh's E columns

// ---- kernel-family launchers ---------------------------------------------
// stream_rows.cu: true if launched (the fused TSQR, when requested, too)
bool try_apply_rows(Ctx& c, const ApplyArgs& a0, int b);
// stream_pair.cu: b = 1 one-pass pass with rows split over warp pairs; the b = 1
// check-refresh pass (EX)
void launch_pair(Ctx& c, const ApplyArgs& a0, int b);
void launch_pair_ex(Ctx& c, const ApplyArgs& a);
// stream_ticket.cu: the ticket A*W pass (any b <= 8) and the K2 gram pass
void launch_ticket(Ctx& c, const ApplyArgs& a, int b);
void launch_gram_b(Ctx& c, const GramArgs& a, int b);

}  // namespace strm
}  // namespace msvd
