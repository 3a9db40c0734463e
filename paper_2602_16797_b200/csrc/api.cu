// Host side of libmsvd_cuda.so: the C ABI of include/msvd.h and the device
// solve loop that replaces lobpcg_solve (solver.cpp:301-477).
//
// The host only orchestrates: it validates options exactly like the
// reference (solver.cpp:306-315, prepare() :128-145, build_sparsestack
// :36-41), launches the kernels of one iteration back to back on the context
// stream, and synchronizes only at check iterations (solver.cpp:439) to read
// the device stop/error word.  Every number the solver produces is computed
// on the GPU; there is no CPU fallback.
#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "msvd_internal.h"

namespace msvd {
// rawio.cu: raw binary interchange of A
void raw_write(const char* path, const double* hA, int64_t m, int64_t n, int64_t ld);
void raw_info(const char* path, int64_t* m, int64_t* n);
void raw_read_rows(const char* path, int64_t row0, int64_t rows, double* hA, int64_t ld);
void raw_load_device(Ctx& c, const char* path, int64_t row0, int64_t rows, double* dA, int64_t ld);
}  // namespace msvd

namespace msvd {

thread_local std::string g_last_error;

[[noreturn]] void fail(int code, const std::string& msg) { throw Fail(code, msg); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(MSVD_ERR_CUDA, std::string(cudaGetErrorString(e)) + " in " + what);
}

void* Ctx::ensure_sar(size_t bytes) {
    if (bytes > sar_bytes) {
        if (sar) MSVD_CUDA(cudaFree(sar));
        sar = nullptr;
        MSVD_CUDA(cudaMalloc(&sar, bytes));
        sar_bytes = bytes;
    }
    return sar;
}

void* Ctx::ensure_sa(size_t bytes) {
    if (bytes > sa_bytes) {
        if (sa) MSVD_CUDA(cudaFree(sa));
        sa = nullptr;
        MSVD_CUDA(cudaMalloc(&sa, bytes));
        sa_bytes = bytes;
    }
    return sa;
}

void* Ctx::ensure_scratch(size_t bytes) {
    if (bytes > scratch_bytes) {
        if (scratch) MSVD_CUDA(cudaFree(scratch));
        scratch = nullptr;
        MSVD_CUDA(cudaMalloc(&scratch, bytes));
        scratch_bytes = bytes;
    }
    return scratch;
}

ProfScope::ProfScope(Ctx& ctx, int s) : c(ctx), slot(s) {
    if (!c.profiling || (c.profiling == 1 && slot != kProfApply && slot != kProfGram)) return;
    size_t& used = c.prof_used[slot];
    auto& v = c.prof_ev[slot];
    if (used == v.size()) {
        std::pair<cudaEvent_t, cudaEvent_t> e;
        MSVD_CUDA(cudaEventCreate(&e.first));
        MSVD_CUDA(cudaEventCreate(&e.second));
        v.push_back(e);
    }
    MSVD_CUDA(cudaEventRecord(v[used].first, c.stream));
    stop = v[used].second;
}
ProfScope::~ProfScope() {
    if (!stop) return;
    cudaEventRecord(stop, c.stream);
    ++c.prof_used[slot];
}

namespace {

template <class F>
int32_t guard(F&& f) {
    try {
        f();
        return MSVD_OK;
    } catch (const Fail& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return MSVD_ERR_INVALID;
    }
}

constexpr double kEps = 2.220446049250313e-16;

double default_tol(int64_t n) { return 2.0 * std::sqrt(static_cast<double>(n)) * kEps; }

struct Plan {
    double tol;
    int max_iter;
    bool skip;
    int64_t d;
};

// solver.cpp:306-315 + prepare() :128-145 + build_sparsestack :36-41, in order
Plan validate(int64_t m, int64_t n, const msvd_options& o) {
    const int64_t b = o.block_size;
    if (m < n) fail(MSVD_ERR_DIMENSION, "solver: matrix must have at least as many rows as columns");
    if (b < 1) fail(MSVD_ERR_DIMENSION, "solver: block size must be positive");
    if (n < 3 * b) fail(MSVD_ERR_DIMENSION, "solver: need at least 3x block size columns");
    Plan p{};
    p.tol = o.tol < 0.0 ? default_tol(n) : o.tol;
    if (!(p.tol >= 0.0 && p.tol < 1.0)) fail(MSVD_ERR_NUMERICAL, "solver: tol must lie in [0, 1)");
    p.max_iter = o.max_iter < 0 ? (b == 1 ? 200 : 100) : o.max_iter;
    if (p.max_iter < 0 || o.check_every < 1)
        fail(MSVD_ERR_NUMERICAL, "solver: max_iter must be >= 0 and check_every >= 1");
    p.skip = o.sketch_dim < 0 && m <= 4 * n;
    if (!p.skip) {
        if (o.sketch_dim < 0 && o.zeta <= 0)
            fail(MSVD_ERR_DIMENSION, "round_up_to_multiple: zeta must be positive");
        int64_t d = o.sketch_dim;
        if (d < 0) d = (4 * n) % o.zeta == 0 ? 4 * n : 4 * n + (o.zeta - (4 * n) % o.zeta);
        if (d < n) fail(MSVD_ERR_DIMENSION, "solver: sketch dimension below column count");
        if (d <= 0 || m <= 0) fail(MSVD_ERR_DIMENSION, "build_sparsestack: dimensions must be positive");
        if (o.zeta <= 0 || o.zeta > d) fail(MSVD_ERR_DIMENSION, "build_sparsestack: zeta must be in [1, d]");
        if (d % o.zeta != 0)
            fail(MSVD_ERR_DIMENSION, "build_sparsestack: zeta must divide d; use round_up_to_multiple(d, zeta) = " +
                                         std::to_string(d + (o.zeta - d % o.zeta)));
        p.d = d;
    }
    // limits of this build's register-tiled kernels (not reference errors);
    // n > 2048 streams in column panels (stream.cu)
    if (b > kMaxB) fail(MSVD_ERR_DIMENSION, "msvd: block size above 8 is not supported by this build");
    if (n > kMaxCols) fail(MSVD_ERR_DIMENSION, "msvd: more than 2^20 columns is not supported by this build");
    if (o.precond_kind < 0 || o.precond_kind > 2) fail(MSVD_ERR_INVALID, "msvd: unknown preconditioner kind");
    return p;
}

// all per-solve buffers carved from one ctx-owned allocation (grown on
// demand, reused across solves: no cudaMalloc/cudaFree inside a solve)
struct Arena {
    Ctx& c;
    std::vector<std::pair<void**, size_t>> req;
    explicit Arena(Ctx& ctx) : c(ctx) {}
    template <class T>
    void add(T** p, size_t count) {
        req.push_back({reinterpret_cast<void**>(p), ((sizeof(T) * std::max<size_t>(count, 1) + 255) / 256) * 256});
    }
    void commit() {
        size_t tot = 0;
        for (auto& r : req) tot += r.second;
        if (tot > c.arena_bytes) {
            if (c.arena) MSVD_CUDA(cudaFree(c.arena));
            c.arena = nullptr;
            MSVD_CUDA(cudaMalloc(&c.arena, tot));
            c.arena_bytes = tot;
        }
        size_t off = 0;
        for (auto& r : req) {
            *r.first = static_cast<unsigned char*>(c.arena) + off;
            off += r.second;
        }
    }
};

std::string err_message(const DevState& s) {
    char buf[160];
    switch (s.err_code) {
        case kErrNonfiniteW:
            std::snprintf(buf, sizeof buf, "solver: non-finite preconditioned residual at iteration %d", s.err_iter);
            return buf;
        case kErrNonfiniteAT:
            std::snprintf(buf, sizeof buf, "solver: non-finite trial products at iteration %d", s.err_iter);
            return buf;
        case kErrJacobi:
            return "one_sided_jacobi: no convergence after 60 sweeps";
        case kErrCgs2:
            return "cgs2: could not complete an orthonormal block";
        case kErrOrth:
            return "solver: history update basis collapsed";
        case kErrDrift:
            std::snprintf(buf, sizeof buf, "solver: cached product drifted from a fresh one at iteration %d",
                          s.err_iter);
            return buf;
        case kErrNonfiniteA:
            return "DenseOperator: non-finite entry";
        default:
            return "msvd: device error " + std::to_string(s.err_code);
    }
}

DevState read_state_raw(Ctx& c, const DevState* st) {
    DevState h;
    MSVD_CUDA(cudaMemcpyAsync(&h, st, sizeof(DevState), cudaMemcpyDeviceToHost, c.stream));
    MSVD_CUDA(cudaStreamSynchronize(c.stream));
    return h;
}

DevState read_state(Ctx& c, const DevState* st) {
    const DevState h = read_state_raw(c, st);
    if (h.err_code != kErrNone) fail(MSVD_ERR_NUMERICAL, err_message(h));
    return h;
}

// a deferred check row that stops: the speculative work of the next
// iteration is discarded, so its replacements and errors are too
DevState stopped_state(DevState h) {
    h.err_code = h.snap_err_code;
    h.err_iter = h.snap_err_iter;
    h.replacements = h.snap_replacements;
    if (h.err_code != kErrNone) fail(MSVD_ERR_NUMERICAL, err_message(h));
    return h;
}

void set_device(const Ctx& c) { MSVD_CUDA(cudaSetDevice(c.device)); }

StreamGeom geom_of(const Ctx& c, const msvd_matrix& M) {
    return make_geom(c, M.kind == kMatCsr ? nullptr : M.A, M.m_local, static_cast<int32_t>(M.n),
                     M.kind == kMatCsr ? M.n : M.ld);
}

}  // namespace

// ---- operator-generic passes (declared in msvd_internal.h) ----------------
void op_apply(Ctx& c, const msvd_matrix& M, const double* W, int b, OutCols out) {
    if (M.kind == kMatCsr) {
        csr_apply(c, M, W, b, out);
        return;
    }
    launch_apply(c, geom_of(c, M), W, b, out);
}

int op_parts(const Ctx& c, const msvd_matrix& M) {
    return M.kind == kMatCsr ? csr_parts(c, M) : geom_of(c, M).grid;
}

int op_adjoint(Ctx& c, const msvd_matrix& M, Cols Y, int b, double* Gpart) {
    if (M.kind == kMatCsr) return csr_adjoint_parts(c, M, Y, b, Gpart);
    const StreamGeom g = geom_of(c, M);
    launch_gram(c, g, Y, b, nullptr, b, b, OutCols{}, true, Gpart);
    return g.grid;
}

// Y = T C into `out` (q columns), then the partials of A^T Y[:, :b]
int op_gram(Ctx& c, const msvd_matrix& M, const StreamGeom& g, Cols T, int k, const double* Cm, int q, int b,
            OutCols out, double* Gpart) {
    if (M.kind == kMatCsr) {
        {
            ProfScope prof(c, kProfReduce);
            launch_tcombine(c, T, k, Cm, q, out, M.m_local);
        }
        Cols Y{};
        for (int j = 0; j < b; ++j) Y.p[j] = out.p[j];
        return csr_adjoint_parts(c, M, Y, b, Gpart);
    }
    launch_gram(c, g, T, k, Cm, q, b, out, false, Gpart);
    return g.grid;
}

namespace {

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

// ---------------------------------------------------------------------------
// lobpcg_solve on a device (row-sharded) dense operator
// ---------------------------------------------------------------------------
// optional host source of A: the H2D copy is chunked on a side stream and
// each chunk is sketched as soon as it lands (msvd_solve_host)
struct HostSource {
    const double* hA;
    int64_t ld;
};

// Cholesky QR2 of the trial block (trial_qr.cu): b >= 2 on one rank, unless
// MSVD_TRIAL_QR = householder.  Measured: it pays where the TSQR's merge of
// k x k parts is the cost (C4, k = 12: 10.5 -> 7.7 ms of loop at m = 6e4).
// b = 2 (k = 6) joined in round 2, once pass 1's Gram came from the carried
// images and the block's Gram pass kept its sums in registers: C5's TSQR +
// Rayleigh-Ritz merge 50.7 -> 16.9 ms per solve, the same iteration counts on
// every b = 2 parity case (C5's roundoff-chaotic second target included:
// tests/test_gpu_true_shapes.py).  b = 1 keeps the TSQR fused into the pass.
bool use_cholqr_req(int b, int ranks) {
    const char* e = std::getenv("MSVD_TRIAL_QR");
    return ranks == 1 && b >= 2 && !(e && std::string(e) == "householder");
}

void solve(msvd_matrix* M, const msvd_options& o, const msvd_truth* truth, msvd_result* res,
           const HostSource* hs = nullptr) {
    Ctx& c = M->ctx->c;
    set_device(c);
    Comm& comm = *c.comm;
    const int64_t n = M->n, m = M->m_global, ml = M->m_local;
    const Plan plan = validate(m, n, o);
    const int b = static_cast<int>(o.block_size);
    const int max_iter = plan.max_iter;
    const int kind = o.precond_kind;
    if (!res || !res->sigma || !res->v) fail(MSVD_ERR_INVALID, "msvd: result buffers missing");
    if (truth && !truth->v_min) fail(MSVD_ERR_DIMENSION, "solver: ground-truth vector length mismatch");
    const StreamGeom geom = geom_of(c, *M);
    const bool csr = M->kind == kMatCsr;
    const int gparts = op_parts(c, *M);  // partials of one A^T pass
    const int nparts = tsqr_parts(c);
    const int ranks = comm.nranks();
    const int kmax = 3 * b;
    const int nblk = static_cast<int>(ceil_div(n, 64));  // reduce_g column blocks

    for (int i = 0; i < 6; ++i)
        if (!c.ev[i]) MSVD_CUDA(cudaEventCreate(&c.ev[i]));
    MSVD_CUDA(cudaEventRecord(c.ev[0], c.stream));

    Arena ar(c);
    DevState* st;
    msvd_record_row* rows;
    double *rh, *th, *Vcol, *Vrow, *sig, *AVb[2], *AXb[2], *AW, *Vb[2], *Xb[2], *W, *Rres, *tmp, *Cm, *Gpart,
        *Gout, *nrm, *Rparts, *Rall, *tv, *dinv, *cpart, *fresh, *ZVb[2], *ZXb[2], *ZW, *V0b, *tq_buf;
    ar.add(&st, 1);
    ar.add(&rows, max_iter + 2);
    ar.add(&rh, max_iter + 2);
    ar.add(&th, max_iter + 2);
    ar.add(&Vcol, n * n);
    ar.add(&Vrow, n * n);
    ar.add(&V0b, n * b);
    ar.add(&sig, n);
    for (int i = 0; i < 2; ++i) {
        ar.add(&AVb[i], ml * b);
        ar.add(&AXb[i], ml * b);
        ar.add(&Vb[i], n * b);
        ar.add(&Xb[i], n * b);
        ar.add(&ZVb[i], n * b);
        ar.add(&ZXb[i], n * b);
    }
    ar.add(&ZW, n * b);
    ar.add(&AW, ml * b);
    ar.add(&W, n * b);
    ar.add(&Rres, n * b);
    ar.add(&tmp, n * b);
    ar.add(&Cm, kMaxK * 2 * kMaxB);
    ar.add(&Gpart, static_cast<size_t>(std::max(geom.grid, gparts)) * 2 * b * n);
    ar.add(&Gout, n * 2 * b);
    ar.add(&nrm, static_cast<size_t>(2 * b) * nblk);
    const int nparts_max = std::max(nparts, geom.grid);
    ar.add(&Rparts, static_cast<size_t>(nparts_max) * kmax * kmax);
    ar.add(&Rall, static_cast<size_t>(ranks) * nparts_max * kmax * kmax);
    ar.add(&tv, n);
    ar.add(&dinv, n);
    ar.add(&cpart, static_cast<size_t>(c.num_sms) * n);
    ar.add(&fresh, o.verify_cached_products ? ml * b : 1);
    ar.add(&tq_buf, static_cast<size_t>(4 * c.num_sms + 5) * kmax * kmax + 2);
    ar.commit();
    // Cholesky QR2 of the trial block (trial_qr.cu) for b >= 2 on one rank;
    // the TSQR kernels still run where its device flag says it failed
    TrialQr tq{};
    tq.gpart = tq_buf;
    tq.R1 = tq_buf + static_cast<size_t>(4 * c.num_sms) * kmax * kmax;  // after [4 num_sms][k][k] parts
    tq.R1inv = tq.R1 + kmax * kmax;
    tq.R2inv = tq.R1inv + kmax * kmax;
    tq.R = tq.R2inv + kmax * kmax;
    tq.flag = reinterpret_cast<int*>(tq.R + kmax * kmax);
    tq.disabled = tq.flag + 1;
    if (use_cholqr_req(b, ranks)) MSVD_CUDA(cudaMemsetAsync(tq.flag, 0, 2 * sizeof(int), c.stream));
    const bool use_cholqr = use_cholqr_req(b, ranks);

    launch_state_init(c, st, o.seed);
    double* theta_dev =
        reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(st) + offsetof(DevState, theta));
    if (truth) MSVD_CUDA(cudaMemcpyAsync(tv, truth->v_min, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));

    // ---- prepare (solver.cpp:128-145) ----
    double sigma1 = 0.0;
    int64_t nfloor = 0;
    // Cholesky-QR route (csrc/precond_chol.cu): P = R^-1 with sigma~_1 and V0
    // from block iterations, where no sigma~ can reach the floor and the
    // caller did not ask for the factors Vt / sigma~ themselves
    bool chol_route = false;
    const bool root = ranks == 1 || comm.rank() == 0;  // rank 0 factors, the others receive
    {
        double* SA = nullptr;
        int64_t sa_rows = 0;
        if (hs && plan.skip && ml > 0)
            MSVD_CUDA(cudaMemcpy2DAsync(const_cast<double*>(M->A), sizeof(double) * M->ld, hs->hA,
                                        sizeof(double) * hs->ld, sizeof(double) * n, ml, cudaMemcpyHostToDevice,
                                        c.stream));
        if (plan.skip) {
            // m <= 4n: P from a direct SVD of A (solver.cpp:132-134).  Assemble the
            // global A (exact: other ranks contribute zeros) and transpose it.
            double* Arm = nullptr;
            MSVD_CUDA(cudaMalloc(&Arm, sizeof(double) * m * n));
            MSVD_CUDA(cudaMalloc(&SA, sizeof(double) * m * n));
            MSVD_CUDA(cudaMemsetAsync(Arm, 0, sizeof(double) * m * n, c.stream));
            if (ml > 0 && csr) csr_scatter_dense(c, *M, Arm + M->row0 * n);
            if (ml > 0 && !csr)
                MSVD_CUDA(cudaMemcpy2DAsync(Arm + M->row0 * n, sizeof(double) * n, M->A, sizeof(double) * M->ld,
                                            sizeof(double) * n, ml, cudaMemcpyDeviceToDevice, c.stream));
            comm.allreduce_sum(Arm, static_cast<size_t>(m * n), c.stream);
            launch_transpose_rm_to_cm(c, Arm, m, n, n, SA);
            MSVD_CUDA(cudaStreamSynchronize(c.stream));
            MSVD_CUDA(cudaFree(Arm));
            sa_rows = m;
            // DenseOperator construction rejects non-finite data (operator.cpp:35-37);
            // a CSR operator was validated at attach (csr.cpp:29-30)
            if (!csr) launch_colnorms(c, geom, cpart, tmp);
        } else {
            SA = static_cast<double*>(c.ensure_sa(sizeof(double) * plan.d * n));
            if (csr) {
                csr_sketch(c, *M, plan.d, o.zeta, o.seed, SA);
            } else if (!hs) {
                sketch_dev(c, geom, M->row0, plan.d, o.zeta, o.seed, SA, st);
            } else {
                // overlap: chunk i is copied on the side stream while chunk i-1 is sketched
                ProfScope prof(c, kProfSketch);
                if (!c.copy_stream) MSVD_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
                if (!c.copy_ev) MSVD_CUDA(cudaEventCreateWithFlags(&c.copy_ev, cudaEventDisableTiming));
                MSVD_CUDA(cudaEventRecord(c.copy_ev, c.stream));  // device buffer free to overwrite
                MSVD_CUDA(cudaStreamWaitEvent(c.copy_stream, c.copy_ev, 0));
                double* SAr = sketch_begin(c, plan.d, n);
                const int64_t step = sketch_chunk_rows(M->ld);
                const SketchLists L = sketch_prepare(c, ml, M->row0, plan.d, o.zeta, o.seed, step);
                for (int64_t r = 0; r < ml; r += step) {
                    const int64_t rows = std::min(ml - r, step);
                    if (M->ld == n && hs->ld == n)  // contiguous rows: one linear DMA
                        MSVD_CUDA(cudaMemcpyAsync(const_cast<double*>(M->A) + r * n, hs->hA + r * n,
                                                  sizeof(double) * n * rows, cudaMemcpyHostToDevice, c.copy_stream));
                    else
                        MSVD_CUDA(cudaMemcpy2DAsync(const_cast<double*>(M->A) + r * M->ld, sizeof(double) * M->ld,
                                                    hs->hA + r * hs->ld, sizeof(double) * hs->ld, sizeof(double) * n,
                                                    rows, cudaMemcpyHostToDevice, c.copy_stream));
                    MSVD_CUDA(cudaEventRecord(c.copy_ev, c.copy_stream));
                    MSVD_CUDA(cudaStreamWaitEvent(c.stream, c.copy_ev, 0));
                    sketch_rows(c, L, M->A, M->ld, static_cast<int>(n), geom.tma, r / step, SAr, st);
                }
                sketch_finish(c, SAr, plan.d, n, SA);
            }
            comm.allreduce_sum(SA, static_cast<size_t>(plan.d * n), c.stream);
            sa_rows = plan.d;
        }
        MSVD_CUDA(cudaEventRecord(c.ev[1], c.stream));
        try {
            read_state(c, st);  // non-finite A surfaces here, like the DenseOperator ctor
            if (plan.skip && !csr) {
                // finite check of A for the skip path: column sums of squares
                std::vector<double> h(n);
                MSVD_CUDA(cudaMemcpy(h.data(), tmp, sizeof(double) * n, cudaMemcpyDeviceToHost));
                for (double v : h)
                    if (!std::isfinite(v)) fail(MSVD_ERR_NUMERICAL, "DenseOperator: non-finite entry");
            }
            if (root) {
                const char* pe = std::getenv("MSVD_PRECOND");
                const bool want_factors = res->vtilde || res->sigma_tilde;
                if (!want_factors && !(pe && std::string(pe) == "svd"))
                    chol_route = precond_build_chol(c, SA, sa_rows, n, b, Vcol, Vrow, sig, V0b, &sigma1, o.seed);
                if (!chol_route) precond_build_dev(c, SA, sa_rows, n, Vcol, Vrow, sig, &sigma1, &nfloor, b + 8);
            }
        } catch (...) {
            if (plan.skip) cudaFree(SA);
            throw;
        }
        if (plan.skip) MSVD_CUDA(cudaFree(SA));
        if (ranks > 1) {  // every rank uses rank 0's factorization bit for bit
            double hs[3] = {sigma1, static_cast<double>(nfloor), chol_route ? 1.0 : 0.0};
            MSVD_CUDA(cudaMemcpyAsync(tmp, hs, sizeof(hs), cudaMemcpyHostToDevice, c.stream));
            comm.bcast(tmp, 3, 0, c.stream);
            MSVD_CUDA(cudaMemcpyAsync(hs, tmp, sizeof(hs), cudaMemcpyDeviceToHost, c.stream));
            MSVD_CUDA(cudaStreamSynchronize(c.stream));
            sigma1 = hs[0];
            nfloor = static_cast<int64_t>(hs[1]);
            chol_route = hs[2] != 0.0;
            comm.bcast(Vcol, static_cast<size_t>(n * n), 0, c.stream);
            comm.bcast(Vrow, static_cast<size_t>(n * n), 0, c.stream);
            comm.bcast(sig, static_cast<size_t>(n), 0, c.stream);
            if (chol_route) comm.bcast(V0b, static_cast<size_t>(n * b), 0, c.stream);
        }
    }
    MSVD_CUDA(cudaEventRecord(c.ev[2], c.stream));
    if (kind == MSVD_PRECOND_DIAGONAL) {  // solver.cpp:336-340
        if (csr) csr_colsq(c, *M, dinv);
        else launch_colnorms(c, geom, cpart, dinv);
        comm.allreduce_sum(dinv, static_cast<size_t>(n), c.stream);
        std::vector<double> h(n);
        MSVD_CUDA(cudaMemcpyAsync(h.data(), dinv, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
        for (double& v : h) {
            const double cn = std::sqrt(v);
            v = cn > 0.0 ? 1.0 / (cn * cn) : 1.0;
        }
        MSVD_CUDA(cudaMemcpyAsync(dinv, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
    }

    auto cols_m = [&](std::initializer_list<std::pair<double*, int>> parts) {
        Cols t{};
        int at = 0;
        for (auto& pr : parts)
            for (int j = 0; j < pr.second; ++j) t.p[at++] = pr.first + static_cast<int64_t>(j) * ml;
        return t;
    };
    auto cols_n = [&](std::initializer_list<std::pair<double*, int>> parts) {
        Cols t{};
        int at = 0;
        for (auto& pr : parts)
            for (int j = 0; j < pr.second; ++j) t.p[at++] = pr.first + static_cast<int64_t>(j) * n;
        return t;
    };
    // A*W pass with the TSQR fused into it when the kernel supports it;
    // otherwise a separate TSQR pass over the trial block.  Per-rank R factors
    // are then gathered in rank order.
    // fused TSQR only for b = 1 (k <= 3): measured, the fold's registers slow
    // the wider A*W kernels more than a separate TSQR pass costs
    const bool fuse = !csr && b == 1 && !std::getenv("MSVD_NO_FUSED_TSQR");
    // One-pass mode: the A*W pass also forms A^T A W, and the n-side images
    // Z = A^T A [V X W] are carried through the Rayleigh-Ritz recurrences next
    // to V and X, so between checks the residual A^T A V' = Z C needs no
    // second pass over A (the Gram apply).  Same products as the
    // reference in exact arithmetic (solver.cpp:357-369 forms A^T (AT C) with
    // AT C from the cached products; here (A^T AT) C from the cached images).
    // Every check iteration (solver.cpp:439, the only place the stop rule
    // reads the residual) still runs the reference's Gram pass, whose result
    // also refreshes the image A^T A V'.  MSVD_ONE_PASS = 0 forces two passes.
    bool one_pass = false;
    {
        const char* e = std::getenv("MSVD_ONE_PASS");
        TsqrFuse probe{};
        probe.k = 3 * b;
        probe.Rparts = Rparts;
        // the stagnation test also reads the residual 5 rows back
        // (solver.cpp:190-200): that row must be a check row too
        const bool rows_exact = !o.use_stagnation || 5 % o.check_every == 0;
        one_pass = !csr && !(e && std::atoi(e) == 0) && o.check_every > 1 && rows_exact &&
                   apply_gram_supported(c, geom, b, fuse ? &probe : nullptr);
    }
    // ex != nullptr (one-pass check refresh): the pass also forms A^T E for
    // E = ex (m x b) into Gout[b n : 2 b n], next to A^T A W
    // trial-block Cholesky QR2 in one-pass mode: pass 1's Gram is S^T Z from the n-side basis S
    // = [V X W] and its carried images Z = A^T A S (set by the caller before each pass; ZW is
    // reduced first), so the m x k block is swept once, not twice.  MSVD_TRIAL_IMAGE_GRAM = 0
    // sweeps twice.
    Cols imgS{}, imgZ{};
    const bool image_gram = one_pass && !(std::getenv("MSVD_TRIAL_IMAGE_GRAM") &&
                                          std::atoi(std::getenv("MSVD_TRIAL_IMAGE_GRAM")) == 0);
    auto apply_tsqr = [&](Cols Tlead, int nlead, OutCols aw, Cols Tall, int k, int iter,
                          const double* ex = nullptr) -> std::pair<const double*, int> {
        TsqrFuse fz{};
        fz.T = Tlead;
        fz.k = k;
        fz.Rparts = Rparts;
        fz.st = st;
        fz.iter = iter;
        (void)nlead;
        int np = nparts;
        bool fused = false;
        if (ex) {
            const bool exfused = launch_apply_ex(c, geom, W, b, aw, ex, ml, Gpart, fuse ? &fz : nullptr);
            if (exfused) np = geom.grid;
            launch_reduce_g(c, Gpart, geom.grid, n, 2 * b, nullptr, st, 0, Gout, nrm, nblk);
            if (ranks > 1) comm.allreduce_sum(Gout, static_cast<size_t>(2 * b * n), c.stream);
            MSVD_CUDA(cudaMemcpyAsync(ZW, Gout, sizeof(double) * b * n, cudaMemcpyDeviceToDevice, c.stream));
            if (!exfused) {
                if (use_cholqr) launch_trial_cholqr(c, Tall, ml, k, tq, image_gram ? &imgS : nullptr, &imgZ, n);
                launch_tsqr(c, Tall, ml, k, Rparts, st, iter, use_cholqr ? tq.flag : nullptr);
            }
            if (ranks == 1) return {Rparts, np};
            comm.allgather(Rparts, Rall, static_cast<size_t>(np) * k * k, c.stream);
            return {Rall, np * ranks};
        }
        if (csr) csr_apply(c, *M, W, b, aw);
        else fused = launch_apply(c, geom, W, b, aw, fuse ? &fz : nullptr, one_pass ? Gpart : nullptr);
        if (fused) np = geom.grid;
        if (one_pass) {  // ZW = A^T A W summed over CTAs (and ranks)
            launch_reduce_g(c, Gpart, geom.grid, n, b, W, st, 0, ZW, nrm, nblk);
            if (ranks > 1) comm.allreduce_sum(ZW, static_cast<size_t>(n * b), c.stream);
        }
        if (!fused) {
            if (use_cholqr) launch_trial_cholqr(c, Tall, ml, k, tq, image_gram ? &imgS : nullptr, &imgZ, n);
            launch_tsqr(c, Tall, ml, k, Rparts, st, iter, use_cholqr ? tq.flag : nullptr);
        }
        if (ranks == 1) return {Rparts, np};
        comm.allgather(Rparts, Rall, static_cast<size_t>(np) * k * k, c.stream);
        return {Rall, np * ranks};
    };
    auto residual = [&](const double* V) {  // G = A^T Y summed over ranks; R = G - theta^2 V
        if (ranks == 1) {
            launch_reduce_g(c, Gpart, gparts, n, b, V, st, 1, Rres, nrm, nblk);
        } else {
            launch_reduce_g(c, Gpart, gparts, n, b, V, st, 0, Gout, nrm, nblk);
            comm.allreduce_sum(Gout, static_cast<size_t>(n * b), c.stream);
            launch_reduce_g(c, Gout, 1, n, b, V, st, 1, Rres, nrm, nblk);
        }
    };
    // one-pass check iterations: G = A^T (AT C) from the gram pass, summed over
    // CTAs and ranks, becomes the image A^T A V' carried forward
    auto exact_images = [&](double* ZV) {
        launch_reduce_g(c, Gpart, gparts, n, b, nullptr, st, 0, ZV, nrm, nblk);
        if (ranks > 1) comm.allreduce_sum(ZV, static_cast<size_t>(n * b), c.stream);
    };
    // gated checks (opt-in, MSVD_CHECK_GATE = 1; tolerance-only stop, one rank).
    // Off by default: skipping the refresh of A^T A V' far from convergence
    // moves where a run that sits at the roundoff floor happens to dip below
    // tol (C5 shape: 91 iterations instead of the reference's 100).
    const bool gate_checks = one_pass && !o.use_stagnation && ranks == 1 && std::getenv("MSVD_CHECK_GATE") &&
                             std::atoi(std::getenv("MSVD_CHECK_GATE")) != 0;
    // one-pass check refresh (b = 1): a check iteration forms its residual
    // from the images like the others; the NEXT A*W pass also forms the exact
    // A^T (A V') of that iterate (one sweep of A instead of a separate Gram
    // pass), the check row is rewritten with the exact residual and the stop
    // rule runs on it (solver.cpp:439).  A stop returns that iterate; the
    // refreshed image A^T A V' feeds the Rayleigh-Ritz step otherwise.
    bool fused_check = one_pass && b <= 4 && !gate_checks && apply_ex_supported(c, geom, b) &&
                       !(std::getenv("MSVD_FUSED_CHECK") && std::atoi(std::getenv("MSVD_FUSED_CHECK")) == 0);
    // One-pass mode and the check refresh decide which collectives run and
    // their sizes, and each rank derives them from its own geometry (ld
    // parity, pointer alignment, m_local) and environment: the ranks agree on
    // the most conservative choice before the first collective of the loop.
    if (ranks > 1) {
        double h[2] = {one_pass ? 0.0 : 1.0, fused_check ? 0.0 : 1.0};
        MSVD_CUDA(cudaMemcpyAsync(tmp, h, sizeof(h), cudaMemcpyHostToDevice, c.stream));
        comm.allreduce_max(tmp, 2, c.stream);
        MSVD_CUDA(cudaMemcpyAsync(h, tmp, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
        one_pass = one_pass && h[0] == 0.0;
        fused_check = fused_check && one_pass && h[1] == 0.0;
    }
    bool pending = false;  // a check row waits for the next pass
    const int* skip_flag = reinterpret_cast<const int*>(reinterpret_cast<unsigned char*>(st) +
                                                         offsetof(DevState, skip_exact));
    ControlArgs ca{};
    ca.nblk = nblk;
    ca.nrm_part = nrm;
    ca.b = b;
    ca.n = n;
    ca.truth_v = truth ? tv : nullptr;
    ca.truth_sigma = truth ? truth->sigma_min : 0.0;
    ca.st = st;
    ca.rows = rows;
    ca.rh = rh;
    ca.th = th;
    ca.sigma1 = sigma1;
    ca.tol = plan.tol;
    ca.factor = o.stagnation_factor;
    ca.use_stag = o.use_stagnation;
    ca.timing = o.record_timing;

    std::vector<double> host_t, host_v;
    auto emit = [&](int kindv, int iter, std::initializer_list<std::pair<double*, int>> parts) {
        if (!res->iterate_cb) return;
        int cols = 0;
        for (auto& pr : parts) cols += pr.second;
        std::vector<double>& h = kindv == 0 ? host_t : host_v;
        h.resize(static_cast<size_t>(n) * cols);
        int at = 0;
        for (auto& pr : parts) {
            if (pr.second)
                MSVD_CUDA(cudaMemcpyAsync(h.data() + static_cast<size_t>(at) * n, pr.first,
                                          sizeof(double) * n * pr.second, cudaMemcpyDeviceToHost, c.stream));
            at += pr.second;
        }
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
        res->iterate_cb(res->iterate_user, kindv, iter, h.data(), n, cols);
    };

    // ---- initial block and Rayleigh-Ritz (solver.cpp:349-371) ----
    // sketch_and_solve_init: the last b columns of Vt (precond.cpp:50-57)
    if (chol_route) c.paths |= kPathCholPrecond;
    if (chol_route) launch_copy_cols(c, V0b, n, 0, n, b, W);
    else launch_copy_cols(c, Vcol, n, n - b, n, b, W);
    OutCols out{};
    for (int j = 0; j < b; ++j) out.p[j] = AW + static_cast<int64_t>(j) * ml;
    {
        imgS = cols_n({{W, b}});
        imgZ = cols_n({{ZW, b}});
        auto parts = apply_tsqr(Cols{}, 0, out, cols_m({{AW, b}}), b, -1);
        RRArgs ra{};
        ra.Rparts = parts.first;
        ra.nparts = parts.second;
        ra.k = b;
        ra.b = b;
        ra.mode = 0;
        ra.T = cols_n({{W, b}});
        ra.n = n;
        ra.Vout = Vb[0];
        ra.Xout = nullptr;
        ra.Cm = Cm;
        ra.theta_out = theta_dev;
        ra.st = st;
        ra.iter = -1;
        if (use_cholqr) {
            ra.chol_R = tq.R;
            ra.chol_ok = tq.flag;
        }
        if (one_pass) {
            ra.Z = cols_n({{ZW, b}});
            ra.ZVout = ZVb[0];
        }
        launch_rr(c, ra);
        OutCols yo{};
        for (int j = 0; j < b; ++j) yo.p[j] = AVb[0] + static_cast<int64_t>(j) * ml;
        if (one_pass && !std::getenv("MSVD_INIT_GRAM")) {
            // row 0 is not a check row: A^T A V0 = (A^T A W) C from the images
            // the A*W pass just formed -- fresh, nothing carried yet
            {
                ProfScope prof(c, kProfReduce);
                launch_tcombine(c, cols_m({{AW, b}}), b, Cm, b, yo, ml);
            }
            launch_reduce_g(c, ZVb[0], 1, n, b, Vb[0], st, 1, Rres, nrm, nblk);
        } else {
            op_gram(c, *M, geom, cols_m({{AW, b}}), b, Cm, b, b, yo, Gpart);
            if (one_pass) {
                exact_images(ZVb[0]);
                launch_reduce_g(c, ZVb[0], 1, n, b, Vb[0], st, 1, Rres, nrm, nblk);
            } else {
                residual(Vb[0]);
            }
        }
        ca.V = Vb[0];
        ca.row = 0;
        ca.check = 0;
        launch_control(c, ca);
    }
    if (o.store_iterates) emit(1, 0, {{Vb[0], b}});
    MSVD_CUDA(cudaEventRecord(c.ev[3], c.stream));

    // early accept (tolerance-only stop, tol well above the images' drift ~1e-15):
    // MSVD_EARLY_ACCEPT = 0 always confirms on the next pass
    const bool early_accept = !o.use_stagnation && plan.tol >= 1e-13 &&
                              !(std::getenv("MSVD_EARLY_ACCEPT") && std::atoi(std::getenv("MSVD_EARLY_ACCEPT")) == 0);
    int cur = 0;  // index of the current V / X / AV / AX buffers
    int status = 1;
    int last_row = 0;
    int64_t verify_count = 0;
    bool deferred_stop = false;
    for (int i = 0; i < max_iter; ++i) {
        const bool first = (i == 0);
        const int nx = first ? 0 : b;
        const int k = b + nx + b;
        const int nxt = cur ^ 1;
        if (pending) launch_snapshot(c, st);
        launch_precond(c, kind, Vcol, Vrow, sig, dinv, n, Rres, b, tmp, W, st, i);
        launch_cgs2(c, W, n, b, cols_n({{Vb[cur], b}, {Xb[cur], nx}}), b + nx, st, i);
        for (int j = 0; j < b; ++j) out.p[j] = AW + static_cast<int64_t>(j) * ml;
        const Cols Tm = cols_m({{AVb[cur], b}, {AXb[cur], nx}, {AW, b}});
        if (one_pass) {
            imgS = cols_n({{Vb[cur], b}, {Xb[cur], nx}, {W, b}});
            imgZ = cols_n({{ZVb[cur], b}, {ZXb[cur], nx}, {ZW, b}});
        }
        auto parts = apply_tsqr(cols_m({{AVb[cur], b}, {AXb[cur], nx}}), b + nx, out, Tm, k, i,
                                pending ? AVb[cur] : nullptr);
        if (pending) {
            // the deferred check row i: R = A^T (A V') - theta^2 V' exactly,
            // the image refreshed, then the stop rule (row i, loop counter i-1)
            launch_reduce_g(c, Gout + b * n, 1, n, b, Vb[cur], st, 1, Rres, nrm, nblk);
            MSVD_CUDA(cudaMemcpyAsync(ZVb[cur], Gout + b * n, sizeof(double) * b * n, cudaMemcpyDeviceToDevice,
                                      c.stream));
            ca.V = Vb[cur];
            ca.row = i;
            ca.check = 1;
            launch_control(c, ca);
            pending = false;
            const DevState h = read_state_raw(c, st);
            if (h.stop) {
                status = 0;
                deferred_stop = true;
                break;
            }
            if (h.err_code != kErrNone) fail(MSVD_ERR_NUMERICAL, err_message(h));
        }
        RRArgs ra{};
        ra.Rparts = parts.first;
        ra.nparts = parts.second;
        ra.k = k;
        ra.b = b;
        ra.mode = 1;
        ra.T = cols_n({{Vb[cur], b}, {Xb[cur], nx}, {W, b}});
        ra.n = n;
        ra.Vout = Vb[nxt];
        ra.Xout = Xb[nxt];
        ra.Cm = Cm;
        ra.theta_out = theta_dev;
        ra.st = st;
        ra.iter = i;
        if (use_cholqr) {
            ra.chol_R = tq.R;
            ra.chol_ok = tq.flag;
        }
        if (one_pass) {
            ra.Z = cols_n({{ZVb[cur], b}, {ZXb[cur], nx}, {ZW, b}});
            ra.ZVout = ZVb[nxt];
            ra.ZXout = ZXb[nxt];
        }
        launch_rr(c, ra);
        OutCols yo{};
        for (int j = 0; j < b; ++j) {
            yo.p[j] = AVb[nxt] + static_cast<int64_t>(j) * ml;
            yo.p[b + j] = AXb[nxt] + static_cast<int64_t>(j) * ml;
        }
        const bool check_it = (i % o.check_every) == 0;
        const bool defer = fused_check && check_it && i + 1 < max_iter;
        if (one_pass && (!check_it || defer)) {
            {
                ProfScope prof(c, kProfReduce);  // m x k recurrence products: no pass over A
                launch_tcombine(c, Tm, k, Cm, 2 * b, yo, ml);
            }
            launch_reduce_g(c, ZVb[nxt], 1, n, b, Vb[nxt], st, 1, Rres, nrm, nblk);
        } else if (one_pass && gate_checks) {
            // check iteration, tolerance-only stop: the images' residual first;
            // if it is more than 4x above the stop threshold the reference's
            // test cannot pass (the two residuals agree far above the roundoff
            // floor), and the Gram pass, the refresh and the exact residual
            // all exit at once (device flag, no host round trip)
            {
                ProfScope prof(c, kProfReduce);
                launch_tcombine(c, Tm, k, Cm, 2 * b, yo, ml);
            }
            launch_reduce_g(c, ZVb[nxt], 1, n, b, Vb[nxt], st, 1, Rres, nrm, nblk);
            launch_gate(c, nrm, nblk, b, st, 4.0 * sigma1 * sigma1 * plan.tol);
            launch_gram(c, geom, Tm, k, Cm, 2 * b, b, yo, false, Gpart, skip_flag);
            launch_reduce_g(c, Gpart, geom.grid, n, b, nullptr, st, 0, ZVb[nxt], nrm, nblk, skip_flag);
            launch_reduce_g(c, ZVb[nxt], 1, n, b, Vb[nxt], st, 1, Rres, nrm, nblk, skip_flag);
        } else {
            op_gram(c, *M, geom, Tm, k, Cm, 2 * b, b, yo, Gpart);
            if (one_pass) {  // check iteration: the reference's residual, and a fresh A^T A V'
                exact_images(ZVb[nxt]);
                launch_reduce_g(c, ZVb[nxt], 1, n, b, Vb[nxt], st, 1, Rres, nrm, nblk);
            } else {
                residual(Vb[nxt]);
            }
        }
        ca.V = Vb[nxt];
        ca.row = i + 1;
        // a deferred check row whose image-based residual is already far under the
        // tolerance stops here (control_kernel, check = 2): the speculative pass that
        // would only confirm it is not launched (one pass of A per solve)
        ca.check = check_it && !defer ? 1 : (defer && early_accept ? 2 : 0);
        launch_control(c, ca);
        last_row = i + 1;
        pending = defer;
        if (o.store_iterates) {
            emit(0, i, {{Vb[cur], b}, {Xb[cur], nx}, {W, b}});
            emit(1, i + 1, {{Vb[nxt], b}});
        }
        if (o.verify_cached_products && (i + 1) % 25 == 0) {  // solver.cpp:430-436
            OutCols fo{};
            for (int j = 0; j < b; ++j) fo.p[j] = fresh + static_cast<int64_t>(j) * ml;
            op_apply(c, *M, Vb[nxt], b, fo);
            launch_drift(c, fresh, AVb[nxt], ml * b, st, 1e-10 * sigma1, i);
            if (ranks > 1) {
                double* dm = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(st) +
                                                       offsetof(DevState, max_drift));
                comm.allreduce_max(dm, 1, c.stream);
                launch_drift(c, fresh, fresh, 0, st, 1e-10 * sigma1, i);
            }
            verify_count += b;
        }
        cur = nxt;
        if (ca.check) {
            const DevState h = read_state(c, st);
            if (h.stop) {
                status = 0;
                pending = false;
                break;
            }
        }
    }
    MSVD_CUDA(cudaEventRecord(c.ev[4], c.stream));
    const DevState fin = deferred_stop ? stopped_state(read_state_raw(c, st)) : read_state(c, st);

    // ---- results (solver.cpp:469-476): ascending from the smallest ----
    std::vector<double> V(static_cast<size_t>(n) * b);
    MSVD_CUDA(cudaMemcpyAsync(V.data(), Vb[cur], sizeof(double) * n * b, cudaMemcpyDeviceToHost, c.stream));
    const int nrows = last_row + 1;
    std::vector<msvd_record_row> hrows(nrows);
    MSVD_CUDA(cudaMemcpyAsync(hrows.data(), rows, sizeof(msvd_record_row) * nrows, cudaMemcpyDeviceToHost, c.stream));
    if (res->vtilde)
        MSVD_CUDA(cudaMemcpyAsync(res->vtilde, Vcol, sizeof(double) * n * n, cudaMemcpyDeviceToHost, c.stream));
    if (res->sigma_tilde)
        MSVD_CUDA(cudaMemcpyAsync(res->sigma_tilde, sig, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
    MSVD_CUDA(cudaEventRecord(c.ev[5], c.stream));
    MSVD_CUDA(cudaStreamSynchronize(c.stream));
    for (int j = 0; j < b; ++j) {
        res->sigma[j] = fin.theta[b - 1 - j];
        std::memcpy(res->v + static_cast<size_t>(j) * n, V.data() + static_cast<size_t>(b - 1 - j) * n,
                    sizeof(double) * n);
    }
    res->rows_count = nrows;
    res->iterations = nrows - 1;
    for (int r = 0; r < nrows && r < res->rows_capacity; ++r) res->rows[r] = hrows[r];
    res->status = status;
    res->sigma_max_estimate = sigma1;
    res->floored = nfloor > 0;
    res->floor_count = nfloor;
    res->sketch_skipped = plan.skip;
    res->sketch_dim = plan.skip ? 0 : plan.d;
    res->zeta = plan.skip ? 0 : o.zeta;
    res->verify_count = verify_count;
    res->max_cache_drift = fin.max_drift;
    res->degenerate_replacements = fin.replacements;
    res->t_sketch_ms = ev_ms(c.ev[0], c.ev[1]);
    res->t_svd_ms = ev_ms(c.ev[1], c.ev[2]);
    res->t_init_ms = ev_ms(c.ev[2], c.ev[3]);
    res->t_loop_ms = ev_ms(c.ev[3], c.ev[4]);
    res->t_total_ms = ev_ms(c.ev[0], c.ev[5]);
}

DevState* prim_state(Ctx& c) {
    if (!c.pstate) {
        MSVD_CUDA(cudaMalloc(&c.pstate, sizeof(DevState)));
        MSVD_CUDA(cudaMemsetAsync(c.pstate, 0, sizeof(DevState), c.stream));
    }
    return c.pstate;
}

void need(const void* p, const char* what) {
    if (!p) fail(MSVD_ERR_INVALID, std::string("msvd: null ") + what);
}

}  // namespace
}  // namespace msvd

using namespace msvd;

extern "C" {

int32_t msvd_abi_version(void) { return MSVD_ABI_VERSION; }
const char* msvd_last_error(void) { return g_last_error.c_str(); }

const char* msvd_status_name(int32_t s) {
    switch (s) {
        case MSVD_OK: return "ok";
        case MSVD_ERR_DIMENSION: return "DimensionError";
        case MSVD_ERR_IO: return "IoError";
        case MSVD_ERR_NUMERICAL: return "NumericalError";
        case MSVD_ERR_CONVERGENCE: return "ConvergenceError";
        case MSVD_ERR_CUDA: return "CudaError";
        case MSVD_ERR_COMM: return "CommError";
        default: return "Error";
    }
}

void msvd_options_default(msvd_options* o) {
    if (!o) return;
    o->tol = -1.0;
    o->max_iter = -1;
    o->check_every = 5;
    o->stagnation_factor = 1.1;
    o->block_size = 1;
    o->seed = 0;
    o->sketch_dim = -1;
    o->zeta = 4;
    o->use_stagnation = 1;
    o->record_timing = 1;
    o->verify_cached_products = 0;
    o->store_iterates = 0;
    o->precond_kind = MSVD_PRECOND_RANDOMIZED;
}

double msvd_default_tolerance(int64_t n) { return default_tol(n); }

int32_t msvd_validate_options(int64_t m, int64_t n, const msvd_options* o, const msvd_truth* truth) {
    return guard([&] {
        need(o, "options");
        validate(m, n, *o);
        if (truth && !truth->v_min) fail(MSVD_ERR_DIMENSION, "solver: ground-truth vector length mismatch");
    });
}

void msvd_shard_rows(int64_t m, int32_t nranks, int32_t rank, int64_t* row0, int64_t* rows) {
    const int64_t a = (m * rank) / nranks, b = (m * (rank + 1)) / nranks;
    if (row0) *row0 = a;
    if (rows) *rows = b - a;
}

int32_t msvd_get_nccl_unique_id(uint8_t out[128]) {
    return guard([&] { nccl_unique_id(out); });
}

int32_t msvd_fake_group_create(int32_t nranks, void** group) {
    return guard([&] {
        need(group, "group");
        if (nranks < 1) fail(MSVD_ERR_INVALID, "msvd: nranks must be positive");
        *group = fake_group_create(nranks);
    });
}
int32_t msvd_fake_group_destroy(void* group) {
    return guard([&] {
        if (group) fake_group_destroy(group);
    });
}

int32_t msvd_ctx_create(const msvd_ctx_desc* desc, msvd_ctx** out) {
    return guard([&] {
        need(desc, "descriptor");
        need(out, "output handle");
        *out = nullptr;
        int count = 0;
        MSVD_CUDA(cudaGetDeviceCount(&count));
        if (desc->device < 0 || desc->device >= count) fail(MSVD_ERR_INVALID, "msvd: no such CUDA device");
        auto* h = new msvd_ctx();
        Ctx& c = h->c;
        try {
            c.device = desc->device;
            MSVD_CUDA(cudaSetDevice(c.device));
            int major = 0;
            MSVD_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, c.device));
            if (major != 10) fail(MSVD_ERR_CUDA, "msvd: this build targets sm_100a (B200) only");
            MSVD_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, c.device));
            int optin = 0;
            MSVD_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
            c.smem_optin = static_cast<size_t>(optin);
            if (desc->stream) {
                c.stream = static_cast<cudaStream_t>(desc->stream);
            } else {
                MSVD_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
                c.own_stream = true;
            }
            c.comm = make_comm(*desc, c.stream);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int32_t msvd_ctx_destroy(msvd_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        Ctx& c = ctx->c;
        cudaSetDevice(c.device);
        cudaStreamSynchronize(c.stream);
        delete c.comm;
        if (c.solver) cusolverDnDestroy(c.solver);
        if (c.blas) cublasDestroy(c.blas);
        if (c.scratch) cudaFree(c.scratch);
        if (c.pstate) cudaFree(c.pstate);
        if (c.svd_ws) cudaFree(c.svd_ws);
        if (c.arena) cudaFree(c.arena);
        if (c.hostA) cudaFree(c.hostA);
        if (c.copy_stream) cudaStreamDestroy(c.copy_stream);
        if (c.copy_ev) cudaEventDestroy(c.copy_ev);
        if (c.sa) cudaFree(c.sa);
        if (c.sar) cudaFree(c.sar);
        if (c.svd_lw) cudaFree(c.svd_lw);
        for (auto& e : c.ev)
            if (e) cudaEventDestroy(e);
        for (auto& v : c.prof_ev)
            for (auto& e : v) {
                cudaEventDestroy(e.first);
                cudaEventDestroy(e.second);
            }
        if (c.own_stream) cudaStreamDestroy(c.stream);
        delete ctx;
    });
}

int32_t msvd_ctx_synchronize(msvd_ctx* ctx) {
    return guard([&] {
        need(ctx, "context");
        set_device(ctx->c);
        MSVD_CUDA(cudaStreamSynchronize(ctx->c.stream));
    });
}

int64_t msvd_launch_count(msvd_ctx* ctx) { return ctx ? ctx->c.launches : -1; }

int64_t msvd_ctx_kernel_paths(msvd_ctx* ctx, int32_t reset) {
    if (!ctx) return -1;
    const int64_t p = ctx->c.paths;
    if (reset) ctx->c.paths = 0;
    return p;
}

int32_t msvd_ctx_profile(msvd_ctx* ctx, int32_t enable) {
    return guard([&] {
        need(ctx, "context");
        Ctx& c = ctx->c;
        c.profiling = enable < 0 ? 0 : (enable > 2 ? 2 : enable);
        for (auto& u : c.prof_used) u = 0;
    });
}

int32_t msvd_ctx_profile_read(msvd_ctx* ctx, double* ms, int64_t* counts, int32_t nslots) {
    return guard([&] {
        need(ctx, "context");
        Ctx& c = ctx->c;
        set_device(c);
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
        for (int s = 0; s < nslots && s < kProfSlots; ++s) {
            double tot = 0.0;
            for (size_t i = 0; i < c.prof_used[s]; ++i) tot += ev_ms(c.prof_ev[s][i].first, c.prof_ev[s][i].second);
            if (ms) ms[s] = tot;
            if (counts) counts[s] = static_cast<int64_t>(c.prof_used[s]);
        }
    });
}

void msvd_abi_sizes(int64_t* out, int32_t n) {
    const int64_t s[6] = {sizeof(msvd_options), sizeof(msvd_record_row), sizeof(msvd_truth), sizeof(msvd_result),
                          sizeof(msvd_ctx_desc), sizeof(msvd_lanczos_result)};
    for (int i = 0; i < n && i < 6; ++i) out[i] = s[i];
}

int32_t msvd_matrix_attach(msvd_ctx* ctx, const double* dA, int64_t m_local, int64_t n, int64_t ld, int64_t row0,
                           int64_t m_global, msvd_matrix** out) {
    return guard([&] {
        need(ctx, "context");
        need(out, "output handle");
        if (m_local > 0) need(dA, "matrix pointer");
        if (m_local < 0 || n < 0) fail(MSVD_ERR_DIMENSION, "DenseMatrix: negative dimension");
        if (ld < n) fail(MSVD_ERR_DIMENSION, "msvd: leading dimension below column count");
        if (row0 < 0 || row0 + m_local > m_global) fail(MSVD_ERR_DIMENSION, "msvd: local rows outside the global range");
        auto* M = new msvd_matrix{ctx, dA, m_local, n, ld, row0, m_global};
        *out = M;
    });
}

int32_t msvd_matrix_detach(msvd_matrix* mat) {
    return guard([&] {
        if (mat) {
            set_device(mat->ctx->c);
            csr_release(*mat);
        }
        delete mat;
    });
}

int32_t msvd_csr_attach(msvd_ctx* ctx, const int64_t* dRowOffsets, const void* dColIndices, int32_t index_bytes,
                        const double* dValues, int64_t m_local, int64_t n, int64_t nnz, int64_t row0, int64_t m_global,
                        msvd_matrix** out) {
    return guard([&] {
        need(ctx, "context");
        need(out, "output handle");
        need(dRowOffsets, "row offsets");
        if (nnz > 0) {
            need(dColIndices, "column indices");
            need(dValues, "values");
        }
        if (index_bytes != 4 && index_bytes != 8) fail(MSVD_ERR_INVALID, "msvd: CSR column indices must be 4 or 8 bytes");
        if (m_local < 0 || n < 0) fail(MSVD_ERR_DIMENSION, "CsrMatrix: negative dimension");
        if (row0 < 0 || row0 + m_local > m_global) fail(MSVD_ERR_DIMENSION, "msvd: local rows outside the global range");
        if (n < 1 || n > kMaxCols) fail(MSVD_ERR_DIMENSION, "msvd: column count outside the supported range [1, 2^20]");
        Ctx& c = ctx->c;
        set_device(c);
        auto* M = new msvd_matrix{ctx, nullptr, m_local, n, n, row0, m_global};
        M->kind = kMatCsr;
        M->csr_rp = dRowOffsets;
        M->csr_ci = dColIndices;
        M->csr_idx64 = index_bytes == 8;
        M->csr_v = dValues;
        M->csr_nnz = nnz;
        try {
            csr_prepare(c, *M);
        } catch (...) {
            csr_release(*M);
            delete M;
            throw;
        }
        *out = M;
    });
}

int32_t msvd_apply(msvd_matrix* M, const double* dX, int64_t b, double* dY) {
    return guard([&] {
        need(M, "matrix");
        Ctx& c = M->ctx->c;
        set_device(c);
        if (b < 1 || b > kMaxB) fail(MSVD_ERR_DIMENSION, "msvd: block size must lie in [1, 8]");
        OutCols out{};
        for (int j = 0; j < b; ++j) out.p[j] = dY + j * M->m_local;
        op_apply(c, *M, dX, static_cast<int>(b), out);
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int32_t msvd_apply_adjoint(msvd_matrix* M, const double* dY, int64_t b, double* dX) {
    return guard([&] {
        need(M, "matrix");
        Ctx& c = M->ctx->c;
        set_device(c);
        if (b < 1 || b > kMaxB) fail(MSVD_ERR_DIMENSION, "msvd: block size must lie in [1, 8]");
        const int64_t n = M->n;
        const int nblk = static_cast<int>(ceil_div(n, 64));  // reduce_g column blocks
        const size_t gp = static_cast<size_t>(op_parts(c, *M)) * b * n;
        double* s = static_cast<double*>(c.ensure_scratch(sizeof(double) * (gp + static_cast<size_t>(b) * nblk)));
        Cols T{};
        for (int j = 0; j < b; ++j) T.p[j] = dY + j * M->m_local;
        const int np = op_adjoint(c, *M, T, static_cast<int>(b), s);
        launch_reduce_g(c, s, np, n, static_cast<int>(b), nullptr, nullptr, 0, dX, s + gp, nblk);
        c.comm->allreduce_sum(dX, static_cast<size_t>(n * b), c.stream);
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int32_t msvd_column_norms(msvd_matrix* M, double* dNorms) {
    return guard([&] {
        need(M, "matrix");
        Ctx& c = M->ctx->c;
        set_device(c);
        if (M->kind == kMatCsr) {
            csr_colsq(c, *M, dNorms);
        } else {
            const StreamGeom g = geom_of(c, *M);
            double* part = static_cast<double*>(c.ensure_scratch(sizeof(double) * c.num_sms * M->n));
            launch_colnorms(c, g, part, dNorms);
        }
        c.comm->allreduce_sum(dNorms, static_cast<size_t>(M->n), c.stream);
        std::vector<double> h(M->n);
        MSVD_CUDA(cudaMemcpyAsync(h.data(), dNorms, sizeof(double) * M->n, cudaMemcpyDeviceToHost, c.stream));
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
        for (double& v : h) v = std::sqrt(v);
        MSVD_CUDA(cudaMemcpy(dNorms, h.data(), sizeof(double) * M->n, cudaMemcpyHostToDevice));
    });
}

int32_t msvd_build_sparsestack(msvd_ctx* ctx, int64_t d, int64_t m, int32_t zeta, uint64_t seed,
                               uint32_t* dPositions, int8_t* dSigns) {
    return guard([&] {
        need(ctx, "context");
        Ctx& c = ctx->c;
        set_device(c);
        if (d <= 0 || m <= 0) fail(MSVD_ERR_DIMENSION, "build_sparsestack: dimensions must be positive");
        if (zeta <= 0 || zeta > d) fail(MSVD_ERR_DIMENSION, "build_sparsestack: zeta must be in [1, d]");
        if (d % zeta != 0)
            fail(MSVD_ERR_DIMENSION, "build_sparsestack: zeta must divide d; use round_up_to_multiple(d, zeta) = " +
                                         std::to_string(d + (zeta - d % zeta)));
        build_sparsestack_dev(c, d, m, zeta, seed, dPositions, dSigns);
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int32_t msvd_sketch(msvd_matrix* M, int64_t d, int32_t zeta, uint64_t seed, double* dSA) {
    return guard([&] {
        need(M, "matrix");
        Ctx& c = M->ctx->c;
        set_device(c);
        if (d <= 0 || M->m_global <= 0) fail(MSVD_ERR_DIMENSION, "build_sparsestack: dimensions must be positive");
        if (zeta <= 0 || zeta > d) fail(MSVD_ERR_DIMENSION, "build_sparsestack: zeta must be in [1, d]");
        if (d % zeta != 0)
            fail(MSVD_ERR_DIMENSION, "build_sparsestack: zeta must divide d; use round_up_to_multiple(d, zeta) = " +
                                         std::to_string(d + (zeta - d % zeta)));
        const StreamGeom g = make_geom(c, M->A, M->m_local, static_cast<int32_t>(M->n), M->ld);
        DevState* st = prim_state(c);
        MSVD_CUDA(cudaMemsetAsync(st, 0, sizeof(DevState), c.stream));
        if (M->kind == kMatCsr) csr_sketch(c, *M, d, zeta, seed, dSA);
        else sketch_dev(c, g, M->row0, d, zeta, seed, dSA, st);
        c.comm->allreduce_sum(dSA, static_cast<size_t>(d * M->n), c.stream);
        read_state(c, st);
    });
}

int32_t msvd_precond_build(msvd_ctx* ctx, const double* dSA, int64_t rows, int64_t n, double* dVt, double* dSig,
                           double* sigma_max_estimate, int64_t* floor_count) {
    return guard([&] {
        need(ctx, "context");
        Ctx& c = ctx->c;
        set_device(c);
        double* Vrow = nullptr;
        MSVD_CUDA(cudaMalloc(&Vrow, sizeof(double) * std::max<int64_t>(n * n, 1)));
        double smax = 0.0;
        int64_t nf = 0;
        try {
            precond_build_dev(c, dSA, rows, n, dVt, Vrow, dSig, &smax, &nf);
        } catch (...) {
            cudaFree(Vrow);
            throw;
        }
        cudaFree(Vrow);
        if (sigma_max_estimate) *sigma_max_estimate = smax;
        if (floor_count) *floor_count = nf;
    });
}

int32_t msvd_precond_apply(msvd_ctx* ctx, const double* dVt, const double* dSig, int64_t n, const double* dR,
                           int64_t b, double* dW) {
    return guard([&] {
        need(ctx, "context");
        Ctx& c = ctx->c;
        set_device(c);
        if (b < 1 || b > kMaxB) fail(MSVD_ERR_DIMENSION, "msvd: block size must lie in [1, 8]");
        double* s = static_cast<double*>(c.ensure_scratch(sizeof(double) * (n * n + n * b)));
        launch_transpose_rm_to_cm(c, dVt, n, n, n, s);  // column-major Vt -> row-major copy
        DevState* st = prim_state(c);
        launch_precond(c, MSVD_PRECOND_RANDOMIZED, dVt, s, dSig, nullptr, n, dR, static_cast<int>(b), s + n * n, dW,
                       st, 0);
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int32_t msvd_tsqr_r(msvd_ctx* ctx, const double* dT, int64_t rows, int64_t k, double* dR) {
    return guard([&] {
        need(ctx, "context");
        Ctx& c = ctx->c;
        set_device(c);
        if (k < 1 || k > kMaxK) fail(MSVD_ERR_DIMENSION, "msvd: tsqr width must lie in [1, 24]");
        if (rows < k) fail(MSVD_ERR_DIMENSION, "householder_qr: requires rows >= cols");
        const int np = tsqr_parts(c);
        double* parts = static_cast<double*>(c.ensure_scratch(sizeof(double) * np * k * k));
        DevState* st = prim_state(c);
        MSVD_CUDA(cudaMemsetAsync(st, 0, sizeof(DevState), c.stream));
        Cols T{};
        for (int l = 0; l < k; ++l) T.p[l] = dT + l * rows;
        launch_tsqr(c, T, rows, static_cast<int>(k), parts, st, 0);
        RRArgs ra{};
        ra.Rparts = parts;
        ra.nparts = np;
        ra.k = static_cast<int>(k);
        ra.b = 1;
        ra.mode = 2;
        ra.R_out = dR;
        ra.st = st;
        launch_rr(c, ra);
        const DevState h = read_state(c, st);
        (void)h;
    });
}

int32_t msvd_gram_apply(msvd_matrix* M, const double* dT, int64_t k, const double* dC, int64_t q, int64_t b,
                        double* dG, double* dY) {
    return guard([&] {
        need(M, "matrix");
        Ctx& c = M->ctx->c;
        set_device(c);
        if (b < 1 || b > kMaxB) fail(MSVD_ERR_DIMENSION, "msvd: block size must lie in [1, 8]");
        if (k < 1 || k > kMaxK) fail(MSVD_ERR_DIMENSION, "msvd: trial width must lie in [1, 24]");
        const bool direct = dC == nullptr;
        if (direct && (k != b || q != b)) fail(MSVD_ERR_DIMENSION, "msvd_gram_apply: Y = T needs q == k == b");
        if (!direct && (q < b || q > 2 * b)) fail(MSVD_ERR_DIMENSION, "msvd_gram_apply: q must lie in [b, 2b]");
        if (!direct && !dY) fail(MSVD_ERR_INVALID, "msvd_gram_apply: dY missing");
        const int64_t n = M->n, ml = M->m_local;
        const StreamGeom g = geom_of(c, *M);
        const int nblk = static_cast<int>(ceil_div(n, 64));  // reduce_g column blocks
        const size_t gp = static_cast<size_t>(std::max(g.grid, op_parts(c, *M))) * b * n;
        double* s = static_cast<double*>(c.ensure_scratch(sizeof(double) * (gp + static_cast<size_t>(b) * nblk +
                                                                            kMaxK * 2 * kMaxB)));
        double* Cs = s + gp + static_cast<size_t>(b) * nblk;
        Cols T{};
        for (int l = 0; l < k; ++l) T.p[l] = dT + l * ml;
        OutCols out{};
        if (!direct) {
            for (int j = 0; j < q; ++j) out.p[j] = dY + j * ml;
            MSVD_CUDA(cudaMemcpyAsync(Cs, dC, sizeof(double) * k * q, cudaMemcpyDeviceToDevice, c.stream));
        }
        int np = g.grid;
        if (direct) np = op_adjoint(c, *M, T, static_cast<int>(b), s);
        else np = op_gram(c, *M, g, T, static_cast<int>(k), Cs, static_cast<int>(q), static_cast<int>(b), out, s);
        launch_reduce_g(c, s, np, n, static_cast<int>(b), nullptr, nullptr, 0, dG, s + gp, nblk);
        c.comm->allreduce_sum(dG, static_cast<size_t>(n * b), c.stream);
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int32_t msvd_aw_tsqr(msvd_matrix* M, const double* dW, int64_t b, const double* dLead, int64_t kl, double* dAW,
                     double* dR) {
    return guard([&] {
        need(M, "matrix");
        Ctx& c = M->ctx->c;
        set_device(c);
        if (b < 1 || b > kMaxB) fail(MSVD_ERR_DIMENSION, "msvd: block size must lie in [1, 8]");
        const int64_t k = kl + b, ml = M->m_local, n = M->n;
        if (kl < 0 || k > kMaxK) fail(MSVD_ERR_DIMENSION, "msvd: trial width must lie in [1, 24]");
        if (M->m_global < k) fail(MSVD_ERR_DIMENSION, "householder_qr: requires rows >= cols");
        const StreamGeom g = geom_of(c, *M);
        const int np_max = std::max(tsqr_parts(c), g.grid);
        const int ranks = c.comm->nranks();
        const size_t pk = static_cast<size_t>(np_max) * k * k;
        double* parts = static_cast<double*>(c.ensure_scratch(sizeof(double) * pk * (1 + ranks)));
        double* all = parts + pk;
        DevState* st = prim_state(c);
        MSVD_CUDA(cudaMemsetAsync(st, 0, sizeof(DevState), c.stream));
        OutCols out{};
        for (int j = 0; j < b; ++j) out.p[j] = dAW + j * ml;
        TsqrFuse fz{};
        for (int l = 0; l < kl; ++l) fz.T.p[l] = dLead + l * ml;
        fz.k = static_cast<int>(k);
        fz.Rparts = parts;
        fz.st = st;
        int np = tsqr_parts(c);
        bool fused = false;
        if (M->kind == kMatCsr) csr_apply(c, *M, dW, static_cast<int>(b), out);
        else fused = launch_apply(c, g, dW, static_cast<int>(b), out, &fz);
        if (fused) {
            np = g.grid;
        } else {
            Cols T{};
            for (int l = 0; l < kl; ++l) T.p[l] = dLead + l * ml;
            for (int j = 0; j < b; ++j) T.p[kl + j] = dAW + j * ml;
            launch_tsqr(c, T, ml, static_cast<int>(k), parts, st, 0);
        }
        const double* src = parts;
        if (ranks > 1) {
            c.comm->allgather(parts, all, static_cast<size_t>(np) * k * k, c.stream);
            src = all;
        }
        RRArgs ra{};
        ra.Rparts = src;
        ra.nparts = np * ranks;
        ra.k = static_cast<int>(k);
        ra.b = 1;
        ra.mode = 2;
        ra.R_out = dR;
        ra.st = st;
        launch_rr(c, ra);
        read_state(c, st);
    });
}

int32_t msvd_aw_gram(msvd_matrix* M, const double* dW, int64_t b, double* dAW, double* dZ) {
    return guard([&] {
        need(M, "matrix");
        Ctx& c = M->ctx->c;
        set_device(c);
        if (b < 1 || b > kMaxB) fail(MSVD_ERR_DIMENSION, "msvd: block size must lie in [1, 8]");
        const int64_t n = M->n, ml = M->m_local;
        const StreamGeom g = geom_of(c, *M);
        const int nblk = static_cast<int>(ceil_div(n, 64));  // reduce_g column blocks
        const size_t gp = static_cast<size_t>(std::max(g.grid, op_parts(c, *M))) * b * n;
        double* s = static_cast<double*>(c.ensure_scratch(sizeof(double) * (gp + static_cast<size_t>(b) * nblk)));
        OutCols out{};
        for (int j = 0; j < b; ++j) out.p[j] = dAW + j * ml;
        int np = g.grid;
        if (M->kind == kMatDense && apply_gram_supported(c, g, static_cast<int>(b), nullptr)) {
            launch_apply(c, g, dW, static_cast<int>(b), out, nullptr, s);
        } else {  // two passes
            op_apply(c, *M, dW, static_cast<int>(b), out);
            Cols T{};
            for (int j = 0; j < b; ++j) T.p[j] = dAW + j * ml;
            np = op_adjoint(c, *M, T, static_cast<int>(b), s);
        }
        launch_reduce_g(c, s, np, n, static_cast<int>(b), nullptr, nullptr, 0, dZ, s + gp, nblk);
        c.comm->allreduce_sum(dZ, static_cast<size_t>(n * b), c.stream);
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int32_t msvd_aw_gram_ex(msvd_matrix* M, const double* dW, int64_t b, const double* dE, double* dAW, double* dZ,
                        double* dZE) {
    return guard([&] {
        need(M, "matrix");
        Ctx& c = M->ctx->c;
        set_device(c);
        if (b < 1 || b > kMaxB) fail(MSVD_ERR_DIMENSION, "msvd: block size must lie in [1, 8]");
        const int64_t n = M->n, ml = M->m_local;
        const StreamGeom g = geom_of(c, *M);
        if (M->kind != kMatDense || b > 4 || !apply_ex_supported(c, g, static_cast<int>(b)))
            fail(MSVD_ERR_INVALID, "msvd: A*W + A^T e pass on an unsupported shape");
        const int nblk = static_cast<int>(ceil_div(n, 64));  // reduce_g column blocks
        const size_t gp = static_cast<size_t>(g.grid) * 2 * b * n;
        double* s = static_cast<double*>(c.ensure_scratch(sizeof(double) * (gp + 2 * b * n + static_cast<size_t>(2 * b) * nblk)));
        double* gout = s + gp;
        OutCols out{};
        for (int j = 0; j < b; ++j) out.p[j] = dAW + j * ml;
        launch_apply_ex(c, g, dW, static_cast<int>(b), out, dE, ml, s, nullptr);
        launch_reduce_g(c, s, g.grid, n, static_cast<int>(2 * b), nullptr, nullptr, 0, gout, gout + 2 * b * n, nblk);
        c.comm->allreduce_sum(gout, static_cast<size_t>(2 * b * n), c.stream);
        MSVD_CUDA(cudaMemcpyAsync(dZ, gout, sizeof(double) * b * n, cudaMemcpyDeviceToDevice, c.stream));
        MSVD_CUDA(cudaMemcpyAsync(dZE, gout + b * n, sizeof(double) * b * n, cudaMemcpyDeviceToDevice, c.stream));
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int32_t msvd_small_svd(msvd_ctx* ctx, const double* dB, int64_t k, double* dSigma, double* dV) {
    return guard([&] {
        need(ctx, "context");
        Ctx& c = ctx->c;
        set_device(c);
        if (k < 1 || k > kMaxK) fail(MSVD_ERR_DIMENSION, "msvd: small svd size must lie in [1, 24]");
        DevState* st = prim_state(c);
        MSVD_CUDA(cudaMemsetAsync(st, 0, sizeof(DevState), c.stream));
        launch_small_svd(c, dB, static_cast<int>(k), dSigma, dV, st);
        const DevState h = read_state(c, st);
        if (std::getenv("MSVD_DEBUG_JACOBI")) std::fprintf(stderr, "msvd_small_svd: k=%lld sweeps=%g\n",
                                                         static_cast<long long>(k), h.worst_jacobi);
    });
}

int32_t msvd_check_convergence(msvd_ctx* ctx, const double* resid_hist, const double* theta_hist, int64_t len,
                               int32_t i, double sigma1_estimate, double tol, double factor, int32_t use_stagnation,
                               int32_t* flags) {
    return guard([&] {
        need(ctx, "context");
        need(flags, "flags");
        if (i + 1 >= len || i < 0)  // solver.cpp:181-183
            fail(MSVD_ERR_DIMENSION, "check_convergence: history shorter than the loop counter");
        need(resid_hist, "resid_hist");
        need(theta_hist, "theta_hist");
        Ctx& c = ctx->c;
        set_device(c);
        double* d = nullptr;
        MSVD_CUDA(cudaMalloc(&d, sizeof(double) * 2 * len + sizeof(int) * 4));
        MSVD_CUDA(cudaMemcpyAsync(d, resid_hist, sizeof(double) * len, cudaMemcpyHostToDevice, c.stream));
        MSVD_CUDA(cudaMemcpyAsync(d + len, theta_hist, sizeof(double) * len, cudaMemcpyHostToDevice, c.stream));
        int* df = reinterpret_cast<int*>(d + 2 * len);
        launch_stop_rule(c, d, d + len, i, sigma1_estimate, tol, factor, use_stagnation, df);
        int hf[4];
        MSVD_CUDA(cudaMemcpyAsync(hf, df, sizeof(hf), cudaMemcpyDeviceToHost, c.stream));
        MSVD_CUDA(cudaStreamSynchronize(c.stream));
        MSVD_CUDA(cudaFree(d));
        for (int k = 0; k < 4; ++k) flags[k] = hf[k];
    });
}

int32_t msvd_raw_write(const char* path, const double* hA, int64_t m, int64_t n, int64_t ld) {
    return guard([&] {
        need(path, "path");
        if (m * n > 0) need(hA, "matrix");
        raw_write(path, hA, m, n, ld);
    });
}

int32_t msvd_raw_info(const char* path, int64_t* m, int64_t* n) {
    return guard([&] {
        need(path, "path");
        need(m, "rows");
        need(n, "cols");
        raw_info(path, m, n);
    });
}

int32_t msvd_raw_read_rows(const char* path, int64_t row0, int64_t rows, double* hA, int64_t ld) {
    return guard([&] {
        need(path, "path");
        if (rows > 0) need(hA, "matrix");
        raw_read_rows(path, row0, rows, hA, ld);
    });
}

int32_t msvd_raw_load_device(msvd_ctx* ctx, const char* path, int64_t row0, int64_t rows, double* dA, int64_t ld) {
    return guard([&] {
        need(ctx, "context");
        need(path, "path");
        if (rows > 0) need(dA, "matrix");
        set_device(ctx->c);
        raw_load_device(ctx->c, path, row0, rows, dA, ld);
    });
}

int32_t msvd_lanczos_gk(msvd_matrix* mat, int32_t iters, const double* v0, const msvd_truth* truth,
                        int32_t record_timing, msvd_lanczos_result* res) {
    return guard([&] {
        need(mat, "matrix");
        need(v0, "starting vector");
        need(res, "result");
        need(res->v, "result vector");
        Ctx& c = mat->ctx->c;
        set_device(c);
        lanczos_run(c, *mat, iters, v0, truth, record_timing != 0, res);
    });
}

int32_t msvd_lobpcg_solve(msvd_matrix* mat, const msvd_options* opts, const msvd_truth* truth, msvd_result* res) {
    return guard([&] {
        need(mat, "matrix");
        need(opts, "options");
        solve(mat, *opts, truth, res);
    });
}

int32_t msvd_rlobpcg_single(msvd_matrix* mat, const msvd_options* opts, const msvd_truth* truth, msvd_result* res) {
    return guard([&] {
        need(mat, "matrix");
        need(opts, "options");
        msvd_options o = *opts;
        o.block_size = 1;
        o.precond_kind = MSVD_PRECOND_RANDOMIZED;
        solve(mat, o, truth, res);
    });
}

int32_t msvd_rlobpcg_block(msvd_matrix* mat, const msvd_options* opts, const msvd_truth* truth, msvd_result* res) {
    return guard([&] {
        need(mat, "matrix");
        need(opts, "options");
        msvd_options o = *opts;
        o.precond_kind = MSVD_PRECOND_RANDOMIZED;
        solve(mat, o, truth, res);
    });
}

int32_t msvd_solve_host(msvd_ctx* ctx, const double* hA, int64_t m_local, int64_t n, int64_t ld, int64_t row0,
                        int64_t m_global, const msvd_options* opts, const msvd_truth* truth, msvd_result* res) {
    return guard([&] {
        need(ctx, "context");
        need(opts, "options");
        Ctx& c = ctx->c;
        set_device(c);
        if (m_local > 0) need(hA, "host matrix");
        if (ld < n) fail(MSVD_ERR_DIMENSION, "msvd: leading dimension below column count");
        if (m_local < 0 || n < 0) fail(MSVD_ERR_DIMENSION, "DenseMatrix: negative dimension");
        const int64_t ldd = (n % 2 == 0) ? n : n + 1;  // even pitch keeps the TMA path
        const size_t bytes = sizeof(double) * static_cast<size_t>(std::max<int64_t>(m_local * ldd, 1));
        if (bytes > c.hostA_bytes) {  // device copy of A, reused across calls
            if (c.hostA) MSVD_CUDA(cudaFree(c.hostA));
            c.hostA = nullptr;
            MSVD_CUDA(cudaMalloc(&c.hostA, bytes));
            c.hostA_bytes = bytes;
        }
        msvd_matrix M{ctx, static_cast<double*>(c.hostA), m_local, n, ldd, row0, m_global};
        HostSource hs{hA, ld};
        solve(&M, *opts, truth, res, &hs);
    });
}

}  // extern "C"
