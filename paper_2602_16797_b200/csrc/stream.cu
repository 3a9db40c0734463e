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
//
// This file: stream geometry, the support queries the solver asks, and the
// launch entry points; the kernels live in stream_rows.cu, stream_pair.cu and
// stream_ticket.cu (stream_impl.cuh).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "stream_impl.cuh"

namespace msvd {
namespace strm {

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

// shared memory the narrow kernels need besides the stage ring
size_t rows_extra_bytes(const StreamGeom& g0, int b, const TsqrFuse* ts, bool gram) {
    const int km = ts && ts->Rparts ? 4 : 0;
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
    if (std::getenv("MSVD_APPLY_TICKET") || g0.n > kMaxN) return false;
    const int npairs = (g0.n + 1) / 2;
    const int pl = (npairs + 31) / 32;
    const bool pl_ok = (b == 1 && pl <= 32) || (b == 2 && pl <= 16) || ((b == 3 || b == 4) && pl <= 8);
    if (!pl_ok) return false;
    const int plt = pl <= 4 ? 4 : (pl <= 8 ? 8 : (pl <= 16 ? 16 : 32));
    if (gram && b * plt > 16) return false;  // one-pass registers: the pair kernel takes it
    if (ts && ts->Rparts && (b != 1 || ts->k > 4 || ts->k < b)) return false;
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
    if (!g0.tma || b != 1 || g0.n > kMaxN || std::getenv("MSVD_NO_PAIR")) return false;
    const int bg = b + (ex ? 1 : 0);
    if (bg * pair_pl(g0.n) > 16) return false;
    const StreamGeom g = pair_geom(c, g0);
    if (g.stages * g.stage_bytes + bar_bytes(g.stages) + 1024 > c.smem_optin) return false;
    return sizeof(double) * 4 * bg * g0.n <= static_cast<size_t>(g.stages) * g.stage_bytes;
}


}  // namespace strm

using namespace strm;

StreamGeom make_geom(const Ctx& c, const double* A, int64_t m, int32_t n, int64_t ld) {
    if (n < 1 || n > kMaxCols)
        fail(MSVD_ERR_DIMENSION, "msvd: column count " + std::to_string(n) +
                                     " outside the supported range [1, " + std::to_string(kMaxCols) + "]");
    StreamGeom g{};
    g.A = A;
    g.m = m;
    g.n = n;
    g.ld = ld;
    g.tma = (ld % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) ? 1 : 0;
    g.grid = c.num_sms * static_cast<int32_t>(env_int("MSVD_CTAS_PER_SM", 1));
    if (n > kMaxN) return g;  // streamed in column panels (panel_geom); no whole-row stages
    g.ld_s = g.tma ? static_cast<int32_t>(ld) : static_cast<int32_t>((n + 1) & ~1);
    const int64_t row_bytes = static_cast<int64_t>(g.ld_s) * 8;
    if (row_bytes > kStageBudget / 2)
        fail(MSVD_ERR_DIMENSION, "msvd: leading dimension too large for the stream pipeline");
    const int64_t target = env_int("MSVD_STAGE_KB", kStageTarget / 1024) * 1024;
    const int64_t budget = env_int("MSVD_STAGE_BUDGET_KB", kStageBudget / 1024) * 1024;
    g.rc = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(target / row_bytes, 64)));
    g.stage_bytes = ((static_cast<size_t>(g.rc) * row_bytes + 127) / 128) * 128;
    g.stages = static_cast<int32_t>(std::max<size_t>(2, std::min<size_t>(8, budget / g.stage_bytes)));
    return g;
}

// ---- column panels of a wide A (n > kMaxN) ---------------------------------
// The register-tiled passes hold <= kMaxN columns per CTA (W or the G
// accumulators, kMaxPairs column pairs per consumer thread).  A wider A is
// streamed as P = ceil(n / kMaxN) column panels of even width, one launch each:
// the panels partition the columns, so A is still read exactly once per pass
// (8 m n bytes); each row's panel segment is one bulk copy (rowcopy) when A's
// rows are TMA-aligned, else the LDG producer re-pitches it.  Y = A W sums the
// panels' partial products in panel order (deterministic); A^T Y writes each
// panel's columns of the partials directly.
int panel_count(int n) { return static_cast<int>(ceil_div(n, kMaxN)); }

StreamGeom panel_geom(const StreamGeom& g, int p, int* c0_out) {
    const int P = panel_count(g.n);
    const int w = ((static_cast<int>(ceil_div(g.n, P)) + 1) & ~1);  // even: panel starts stay 16-byte aligned
    const int c0 = p * w;
    const int np = std::min(w, g.n - c0);
    StreamGeom q = g;
    q.A = g.A + c0;
    q.n = np;
    q.ld_s = (np + 1) & ~1;  // an odd last panel (odd n) copies one pad column of the even ld
    q.rowcopy = g.tma;
    const int64_t row_bytes = static_cast<int64_t>(q.ld_s) * 8;
    q.rc = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(kStageTarget / row_bytes, 64)));
    q.stage_bytes = ((static_cast<size_t>(q.rc) * row_bytes + 127) / 128) * 128;
    q.stages = static_cast<int32_t>(std::max<size_t>(2, std::min<size_t>(8, kStageBudget / q.stage_bytes)));
    *c0_out = c0;
    return q;
}

bool apply_gram_supported(const Ctx& c, const StreamGeom& g, int b, const TsqrFuse* fuse) {
    const int pl = ((g.n + 1) / 2 + 31) / 32;
    const int plt = pl <= 4 ? 4 : (pl <= 8 ? 8 : (pl <= 16 ? 16 : 32));  // the PL template the launch picks
    if (b * plt <= 16 && rows_ok(c, g, b, fuse, true)) return true;
    return !fuse && (pair_ok(c, g, b, false) || split_ok(c, g, b, false));  // neither has a fused TSQR
}

bool apply_ex_supported(const Ctx& c, const StreamGeom& g, int b) {
    return b == 1 ? pair_ok(c, g, 1, true) : split_ok(c, g, b, true);
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
        Cols ec{};
        for (int j = 0; j < b; ++j) ec.p[j] = ex + j * ld_ex;
        launch_split(c, ApplyArgs{g, W, out, TsqrFuse{}, gpart, nullptr}, b, &ec);
        return false;
    }
    (void)fuse;  // the b = 1 refresh pass runs the TSQR separately
    launch_pair_ex(c, ApplyArgs{pair_geom(c, g), W, out, TsqrFuse{}, gpart, ex});
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
    if (g.n > kMaxN) {  // column panels: out = sum over panels of A_p W_p, in panel order
        if (gpart) fail(MSVD_ERR_INVALID, "msvd: one-pass A*W / A^T A W launch on an unsupported shape");
        for (int p = 0; p < panel_count(g.n); ++p) {
            int c0 = 0;
            const StreamGeom pg = panel_geom(g, p, &c0);
            ApplyArgs a{cap_rows(rechunk(pg, 48, 144), kRedSlots / std::max(1, b)), W + c0, out, none, nullptr,
                        nullptr, g.n, p > 0 ? 1 : 0};
            launch_ticket(c, a, b);
        }
        return false;
    }
    if (try_apply_rows(c, ApplyArgs{g, W, out, fuse ? *fuse : none, gpart, nullptr}, b)) return fuse != nullptr;
    // b = 2..4: the split-role kernel (stream_split.cu: dot and acc warps).  It replaced the
    // warp-pair and team forms (one warp set doing both halves of the work behind a barrier
    // per row or per four rows): b = 4, n = 500 plain pass 6.6 TB/s against 5.7 (team) and
    // 3.9 (pair), check refresh 5.2 against 2.6; b = 2, n = 1000 7.1 against 6.8 (pair).
    if (gpart && split_ok(c, g, b, false)) {
        launch_split(c, ApplyArgs{g, W, out, none, gpart, nullptr}, b, nullptr);
        return false;
    }
    if (gpart && pair_ok(c, g, b, false)) {  // b = 1, wide rows: split over warp pairs (no fused TSQR)
        launch_pair(c, ApplyArgs{g, W, out, none, gpart, nullptr}, b);
        return false;
    }
    if (gpart) fail(MSVD_ERR_INVALID, "msvd: one-pass A*W / A^T A W launch on an unsupported shape");
    // ticket variant: large stages amortize the per-chunk cross-warp finish
    // (measured: 48 KB x 3 stages best at n = 2000, b = 5)
    ApplyArgs a{cap_rows(rechunk(g, 48, 144), kRedSlots / std::max(1, b)), W, out, none, nullptr};
    launch_ticket(c, a, b);
    return false;
}

void launch_gram(Ctx& c, const StreamGeom& g, Cols T, int k, const double* Cm, int q, int b,
                 OutCols out, bool direct, double* Gpart, const int* skip) {
    ProfScope prof(c, kProfGram);
    // stage geometry by block size (tuning sweep, profiles/README.md):
    // b = 1: 32 KB x 3, b = 2: 48 KB x 3, b >= 3: 64 KB x 2
    if (g.m == 0) {
        MSVD_CUDA(cudaMemsetAsync(Gpart, 0, sizeof(double) * g.grid * b * g.n, c.stream));
        return;
    }
    if (g.n > kMaxN) {  // column panels: each writes its columns of Gpart; the first also the outputs
        for (int p = 0; p < panel_count(g.n); ++p) {
            int c0 = 0;
            const StreamGeom pg0 = panel_geom(g, p, &c0);
            const StreamGeom pg = b == 1 ? rechunk(pg0, 32, 96) : (b == 2 ? rechunk(pg0, 48, 144) : rechunk(pg0, 64, 128));
            GramArgs ap{pg, T, k, Cm, q, p == 0 ? out : OutCols{}, direct ? 1 : 0, Gpart + c0, skip, g.n};
            launch_gram_b(c, ap, b);
        }
        return;
    }
    const StreamGeom gg = b == 1 ? rechunk(g, 32, 96) : (b == 2 ? rechunk(g, 48, 144) : rechunk(g, 64, 128));
    launch_gram_b(c, GramArgs{gg, T, k, Cm, q, out, direct ? 1 : 0, Gpart, skip}, b);
}

}  // namespace msvd

