// K3 ticket variant (apply_kernel, any b <= 8) and the K2 gram pass
// (gram_kernel); see stream_impl.cuh.
#include "stream_impl.cuh"

namespace msvd {
namespace strm {
namespace {


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
    const int64_t ws = a.wstride ? a.wstride : n;  // W's column stride (the full n for a column panel)
    double w[kMaxPairs][2][B];
#pragma unroll
    for (int i = 0; i < kMaxPairs; ++i) {
        const int c0 = 2 * (ct + i * kConsumers);
#pragma unroll
        for (int j = 0; j < B; ++j) {
            w[i][0][j] = c0 < n ? a.W[c0 + static_cast<int64_t>(j) * ws] : 0.0;
            w[i][1][j] = c0 + 1 < n ? a.W[c0 + 1 + static_cast<int64_t>(j) * ws] : 0.0;
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
                if (a.accum) sum = a.out.p[j][r0 + rr] + sum;  // panels in order: deterministic
                a.out.p[j][r0 + rr] = sum;
            }
            __syncwarp();
            if (lane == 0) ticket[slot] = 0;
        }
        if (++slot == nslot) slot = 0;
    }
}


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
                                    if (a.out.p[j]) a.out.p[j][gr] = y;
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
    const size_t gs = a.gstride ? static_cast<size_t>(a.gstride) : static_cast<size_t>(n);
    double* gp = a.Gpart + static_cast<size_t>(blockIdx.x) * B * gs;
#pragma unroll
    for (int i = 0; i < kMaxPairs; ++i) {
        const int c0 = 2 * (ct + i * kConsumers);
#pragma unroll
        for (int j = 0; j < B; ++j) {
            if (c0 < n) gp[j * gs + c0] = acc[i][0][j];
            if (c0 + 1 < n) gp[j * gs + c0 + 1] = acc[i][1][j];
        }
    }
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

void launch_ticket(Ctx& c, const ApplyArgs& a, int b) {
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
}

void launch_gram_b(Ctx& c, const GramArgs& a, int b) {
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

}  // namespace strm
}  // namespace msvd
