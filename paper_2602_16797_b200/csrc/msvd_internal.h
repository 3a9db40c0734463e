// Internal declarations shared by the msvd CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "msvd.h"

namespace msvd {

constexpr int kMaxB = 8;              // block size limit of the register-tiled kernels
constexpr int kMaxK = 3 * kMaxB;      // trial width limit
constexpr int kMaxPairs = 4;          // column pairs per consumer thread (n <= 2048 per panel)
constexpr int kConsumers = 256;       // consumer threads per stream CTA
constexpr int kMaxN = 2 * kMaxPairs * kConsumers;  // widest column panel of one streaming launch
// wider A (the paper's own 2e6 x 4e3 example) streams in column panels of
// <= kMaxN columns, one launch per panel (stream.cu); the n x n
// preconditioner bounds n in practice -- this cap only keeps 8 n^2 in int64
constexpr int64_t kMaxCols = 1 << 20;

// thrown inside the library; converted to a status at the C boundary
struct Fail : std::runtime_error {
    int code;
    Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define MSVD_CUDA(x) ::msvd::cuda_check((x), #x)

// ---- device-side solver state (one per solve, in device memory) ----------
enum DevErr : int32_t {
    kErrNone = 0,
    kErrNonfiniteW = 1,      // solver.cpp:407
    kErrNonfiniteAT = 2,     // solver.cpp:414
    kErrJacobi = 3,          // svd.cpp:147-149
    kErrCgs2 = 4,            // solver.cpp:254
    kErrOrth = 5,            // solver.cpp:112
    kErrDrift = 6,           // solver.cpp:435
    kErrNonfiniteA = 7,      // operator.cpp:35-37 (DenseOperator ctor)
};

struct DevState {
    int32_t stop;
    int32_t err_code;
    int32_t err_iter;
    int32_t have_spare;     // SplitMix64 Box-Muller spare (rng.hpp:40-52)
    uint64_t rng_state;
    double spare;
    int64_t replacements;   // SolveResult::degenerate_replacements
    unsigned long long t0_ns;
    double theta[kMaxB];    // Ritz values of the current target block (descending)
    double max_drift;
    double worst_jacobi;
    int32_t skip_exact;     // one-pass check gate: 1 = the images' residual decides (far from tol)
    int32_t pad_;
    // taken before the speculative work a deferred check row runs ahead of its
    // stop test (precond, cgs2 and the next pass of iteration i + 1): a stop
    // there reports the state the reference stops with
    int32_t snap_err_code;
    int32_t snap_err_iter;
    int64_t snap_replacements;
};

// column-pointer bundles passed by value to kernels
struct Cols {
    const double* p[kMaxK];
};
struct DevState;
struct TsqrFuse {
    Cols T;           // the k - b leading trial columns (AV, AX), length m
    int k;            // trial width; the A*W output supplies the last b columns
    double* Rparts;   // [grid][k][k]
    DevState* st;
    int iter;
};
struct OutCols {
    double* p[2 * kMaxB];
};

// ---- stream geometry of a row-major A on one rank -------------------------
struct StreamGeom {
    const double* A;
    int64_t m;       // local rows
    int32_t n;       // columns
    int64_t ld;      // leading dimension (elements)
    int32_t ld_s;    // shared-memory row stride (elements, even)
    int32_t rc;      // rows per chunk
    int32_t stages;  // pipeline depth
    int32_t tma;     // 1: cp.async.bulk producer, 0: LDG producer
    int32_t grid;    // persistent CTAs
    size_t stage_bytes;
    int32_t rowcopy; // column panel of a wider A: one bulk copy per row (ld_s of the ld-pitched row)
};

struct Ctx;

enum KernelPath : int64_t { kPathRows = 1, kPathSelf = 2, kPathPair = 4, kPathPairEx = 8, kPathTeamEx = 16,
                            kPathTicket = 32, kPathGram = 64, kPathTsqr = 128, kPathCholPrecond = 256,
                            kPathTeam = 512, kPathSplit = 1024, kPathSplitEx = 2048 };

enum ProfSlot { kProfApply = 0, kProfGram, kProfTsqr, kProfRR, kProfSketch, kProfSvd, kProfPrecond, kProfCgs2,
                kProfReduce, kProfControl, kProfSlots };

// ---- launchers (kernels.cu) -----------------------------------------------
StreamGeom make_geom(const Ctx& c, const double* A, int64_t m, int32_t n, int64_t ld);
// Y (m x b, out cols) = A W (W n x b col-major).  With `fuse`, the pass may
// also fold [T | Y] into per-CTA R factors (returns true if it did; the
// caller then skips launch_tsqr)
struct TsqrFuse;
// gpart != nullptr (one-pass mode): the same pass also writes the per-CTA
// partials [grid][b][n] of A^T (A W); only where apply_gram_supported()
bool launch_apply(Ctx& c, const StreamGeom& g, const double* W, int b, OutCols out,
                  const TsqrFuse* fuse = nullptr, double* gpart = nullptr);
bool apply_gram_supported(const Ctx& c, const StreamGeom& g, int b, const TsqrFuse* fuse);
// b = 1: Y = A w and gpart[grid][2][n] = [A^T (A w), A^T e] in one pass (the
// one-pass solver's check refresh of A^T A V', e = A V');
// b = 2..4: Y = A W and gpart[grid][2b][n] = [A^T (A W), A^T E] for E (m x b, ld ld_ex)
bool apply_ex_supported(const Ctx& c, const StreamGeom& g, int b);
// (b = 1 with `fuse` and e its first trial column: the TSQR is folded in too, returns true)
bool launch_apply_ex(Ctx& c, const StreamGeom& g, const double* W, int b, OutCols out, const double* ex,
                     int64_t ld_ex, double* gpart, const TsqrFuse* fuse = nullptr);
// out[j] = T Cm[:, j] for j < q (m-side recurrence products without A)
void launch_tcombine(Ctx& c, Cols T, int k, const double* Cm, int q, OutCols out, int64_t m);
// Gpart[grid][b][n]: A^T Y with Y = T C (gram mode, writes Y cols + extra cols)
// or Y = T (direct mode, q == b, no writes)
void launch_gram(Ctx& c, const StreamGeom& g, Cols T, int k, const double* Cm, int q, int b,
                 OutCols out, bool direct, double* Gpart, const int* skip = nullptr);
// per-CTA Householder R of the m x k column block T, Rparts[nparts][k][k]
int tsqr_parts(const Ctx& c);  // number of partial R factors launch_tsqr produces
// skip: device flag; nonzero = the Cholesky QR2 of the block succeeded, the
// TSQR kernels return at once (trial_qr.cu)
void launch_tsqr(Ctx& c, Cols T, int64_t m, int k, double* Rparts, DevState* st, int iter,
                 const int* skip = nullptr);
// Cholesky QR2 of the m x k trial block (trial_qr.cu): R (k x k upper) and a
// device flag (1 = usable; else the TSQR path runs)
struct TrialQr {
    double* gpart;   // [4 num_sms][k][k] partial Grams
    double* R1;      // k x k
    double* R1inv;   // k x k
    double* R2inv;   // k x k
    double* R;       // k x k: R2 R1, the block's R factor
    int* flag;
    int* disabled;   // sticky: set when a block failed; zeroed at solve start
};
// S, Z (n-side trial basis and its images A^T A S, k columns each): pass 1's Gram from
// S^T Z instead of a sweep of the block (one-pass mode); nullptr: two sweeps
void launch_trial_cholqr(Ctx& c, Cols T, int64_t m, int k, TrialQr& q, const Cols* S = nullptr,
                         const Cols* Z = nullptr, int64_t n = 0);

// single-CTA Rayleigh-Ritz: merge R parts, Jacobi SVD, C / theta / mix, V' = T C, X' = T mix
struct RRArgs {
    const double* Rparts;
    int nparts;
    int k, b;
    int mode;            // 0 init (C = all of V, theta = all sigma), 1 iteration, 2 merge only
    Cols T;              // n-side trial basis columns [V X W]
    int64_t n;
    double* Vout;        // n x b
    double* Xout;        // n x b (mode 1)
    double* Cm;          // k x 2b (C | mix), ld k
    double* theta_out;   // b, descending (theta_next)
    double* sig_out;     // optional k: all Ritz sigma (tests)
    double* Vfull_out;   // optional k x k sorted, sign-fixed V (tests)
    double* R_out;       // optional k x k merged R factor (tests / msvd_tsqr_r)
    Cols Z;              // one-pass mode: n-side A^T A images of T ([ZV ZX ZW]), or Z.p[0] == nullptr
    double* ZVout;       // n x b: A^T A V' = Z C
    double* ZXout;       // n x b (mode 1): A^T A X' = Z mix
    DevState* st;
    int iter;
    const double* chol_R = nullptr;  // k x k R from launch_trial_cholqr, used when *chol_ok != 0
    const int* chol_ok = nullptr;
};
void launch_rr(Ctx& c, const RRArgs& a);

void launch_reduce_g(Ctx& c, const double* Gpart, int nparts, int64_t n, int b, const double* V,
                     const DevState* st, int residual, double* Gout, double* nrm_part, int nblk,
                     const int* skip = nullptr);
// st->skip_exact = (max_j ||R_j|| > thresh): the gate of a one-pass check iteration
void launch_gate(Ctx& c, const double* nrm_part, int nblk, int b, DevState* st, double thresh);
struct ControlArgs {
    const double* nrm_part;  // b x nblk partial sums of squares
    int nblk;
    int b;
    int64_t n;
    const double* V;         // n x b current target block
    const double* truth_v;   // n or null
    double truth_sigma;
    DevState* st;
    msvd_record_row* rows;
    double* rh;
    double* th;
    int row;                 // record row index (= iteration + 1, or 0)
    int check;               // evaluate stop rule at loop counter row-1
    double sigma1, tol, factor;
    int use_stag;
    int timing;
};
void launch_control(Ctx& c, const ControlArgs& a);

void launch_precond(Ctx& c, int kind, const double* Vcol, const double* Vrow, const double* sig,
                    const double* dinv, int64_t n, const double* R, int b, double* tmp, double* W,
                    DevState* st, int iter);
void launch_cgs2(Ctx& c, double* W, int64_t n, int b, Cols basis, int nb, DevState* st, int iter);
void launch_state_init(Ctx& c, DevState* st, uint64_t seed);
void launch_snapshot(Ctx& c, DevState* st);
// the control kernel's stop rule on a given history (flags: tol_ok,
// resid_stalled, progress_stalled, stop; device memory)
void launch_stop_rule(Ctx& c, const double* rh, const double* th, int i, double sigma1, double tol, double factor,
                      int use_stag, int* flags);  // snap_* <- err_code, err_iter, replacements
void launch_drift(Ctx& c, const double* fresh, const double* cached, int64_t count, DevState* st,
                  double limit, int iter);
void launch_colnorms(Ctx& c, const StreamGeom& g, double* part, double* out);
void launch_transpose_rm_to_cm(Ctx& c, const double* A, int64_t m, int64_t n, int64_t ld,
                               double* out);
void launch_copy_cols(Ctx& c, const double* src, int64_t ld_src, int64_t col0, int64_t rows,
                      int64_t cols, double* dst);
void launch_small_svd(Ctx& c, const double* B, int k, double* sigma, double* V, DevState* st);

// ---- sketch (sketch.cu) ---------------------------------------------------
void build_sparsestack_dev(Ctx& c, int64_t d, int64_t m, int zeta, uint64_t seed, uint32_t* pos,
                           int8_t* sgn);
void sketch_dev(Ctx& c, const StreamGeom& g, int64_t row0, int64_t d, int zeta, uint64_t seed,
                double* SA, DevState* st);
// chunked form: sort the (sketch row, source row) lists once, then add row
// chunks in order (bit-identical to one pass); used to overlap H2D copies
struct SketchLists {
    int64_t d = 0, m = 0;
    double val = 0.0;
    const int64_t* offs = nullptr;
    const uint32_t* vals = nullptr;
    const int64_t* bounds = nullptr;  // [chunk][sketch row] segment starts
    int64_t step = 0;                 // source rows per chunk
};
SketchLists sketch_prepare(Ctx& c, int64_t m, int64_t row0, int64_t d, int zeta, uint64_t seed, int64_t step);
void sketch_rows(Ctx& c, const SketchLists& L, const double* A, int64_t ld, int n, int vec, int64_t chunk,
                 double* SA, DevState* st);
int64_t sketch_chunk_rows(int64_t ld);
double* sketch_begin(Ctx& c, int64_t d, int64_t n);  // zeroed row-major running sums
void sketch_finish(Ctx& c, const double* SAr, int64_t d, int64_t n, double* SA);

// ---- preconditioner factorization (svd.cu) --------------------------------
// tail_hint: number of smallest singular triplets refined to Jacobi accuracy
// when the fast polar SVD is used (the solver passes b + 8)
void precond_build_dev(Ctx& c, const double* SA, int64_t rows, int64_t n, double* Vcol,
                       double* Vrow, double* sig, double* sigma_max, int64_t* nfloor, int tail_hint = 8);
// Cholesky-QR route (precond_chol.cu): Vcol / Vrow = R^-1 of the sketch, sig = 1,
// V0 (n x b) = the b smallest right singular vectors (Vt's last b columns),
// sigma_max = sigma~_1.  false (nothing usable written): take the SVD route
bool precond_build_chol(Ctx& c, const double* SA, int64_t rows, int64_t n, int b, double* Vcol, double* Vrow,
                        double* sig, double* V0, double* sigma_max, uint64_t seed);

// ---- operator kinds --------------------------------------------------------
enum MatKind { kMatDense = 0, kMatCsr = 1 };
// CSR operator (csr.cu): validate + build the transpose at attach
void csr_prepare(Ctx& c, msvd_matrix& M);
void csr_release(msvd_matrix& M);
void csr_apply(Ctx& c, const msvd_matrix& M, const double* W, int b, OutCols out);
int csr_parts(const Ctx& c, const msvd_matrix& M);
int csr_adjoint_parts(Ctx& c, const msvd_matrix& M, Cols Y, int b, double* Gpart);
void csr_colsq(Ctx& c, const msvd_matrix& M, double* out);
void csr_sketch(Ctx& c, const msvd_matrix& M, int64_t d, int zeta, uint64_t seed, double* SA);
void csr_scatter_dense(Ctx& c, const msvd_matrix& M, double* out_rows);
// operator-generic passes (api.cu): dense -> the streaming kernels, CSR -> csr.cu
void op_apply(Ctx& c, const msvd_matrix& M, const double* W, int b, OutCols out);
int op_parts(const Ctx& c, const msvd_matrix& M);
int op_adjoint(Ctx& c, const msvd_matrix& M, Cols Y, int b, double* Gpart);  // returns the partial count
int op_gram(Ctx& c, const msvd_matrix& M, const StreamGeom& g, Cols T, int k, const double* Cm, int q, int b,
            OutCols out, double* Gpart);

// ---- Golub-Kahan-Lanczos baseline (lanczos.cu) ---------------------------
void lanczos_run(Ctx& c, const msvd_matrix& M, int iters, const double* v0h, const msvd_truth* truth, bool timing,
                 msvd_lanczos_result* res);

// ---- communicator (comm.cu) ----------------------------------------------
struct Comm {
    virtual ~Comm() = default;
    virtual int nranks() const = 0;
    virtual int rank() const = 0;
    virtual void allreduce_sum(double* d, size_t count, cudaStream_t s) = 0;
    virtual void allgather(const double* send, double* recv, size_t count, cudaStream_t s) = 0;
    virtual void bcast(double* d, size_t count, int root, cudaStream_t s) = 0;
    virtual void allreduce_max(double* d, size_t count, cudaStream_t s) = 0;
};
Comm* make_comm(const msvd_ctx_desc& desc, cudaStream_t s);

// ---- context ---------------------------------------------------------------
struct Ctx {
    int device = 0;
    int num_sms = 148;
    size_t smem_optin = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    Comm* comm = nullptr;
    cusolverDnHandle_t solver = nullptr;
    cublasHandle_t blas = nullptr;
    int64_t launches = 0;
    cudaEvent_t ev[8] = {};
    // reusable device scratch
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    void* ensure_scratch(size_t bytes);
    DevState* pstate = nullptr;  // error word for primitive entry points
    void* arena = nullptr;       // per-solve buffers (reused)
    size_t arena_bytes = 0;
    void* hostA = nullptr;       // device copy of A for msvd_solve_host
    size_t hostA_bytes = 0;
    cudaStream_t copy_stream = nullptr;  // H2D chunks overlapped with the sketch
    cudaEvent_t copy_ev = nullptr;
    void* sa = nullptr;          // sketch d x n
    size_t sa_bytes = 0;
    void* ensure_sa(size_t bytes);
    void* sar = nullptr;         // row-major sketch accumulator
    size_t sar_bytes = 0;
    void* ensure_sar(size_t bytes);
    void* svd_ws = nullptr;      // preconditioner factorization workspace
    size_t svd_ws_bytes = 0;
    void* svd_lw = nullptr;      // cuSOLVER work buffer
    size_t svd_lw_bytes = 0;
    // optional per-kernel-class timing (bench evidence): event pairs per slot
    int profiling = 0;  // 1: the A-pass classes (apply, gram) only; 2: every class
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev[kProfSlots];
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_pool;
    size_t prof_used[kProfSlots] = {};
    // A-pass kernel variants launched (msvd_ctx_kernel_paths bits)
    int64_t paths = 0;
    // kernels already opted in to the device's full dynamic shared memory
    std::unordered_set<const void*> smem_attr;
};

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device-context setting:
// opt each kernel in once per Ctx (a Ctx is bound to one device), never
// through process-wide flags (several devices / FakeComm threads per process)
template <class K>
inline void optin_smem(Ctx& c, K* kernel) {
    if (c.smem_attr.insert(reinterpret_cast<const void*>(kernel)).second)
        MSVD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(c.smem_optin)));
}

// RAII: events around the launches of one kernel class when profiling
struct ProfScope {
    Ctx& c;
    int slot;
    cudaEvent_t stop = nullptr;
    ProfScope(Ctx& ctx, int s);
    ~ProfScope();
};

void* fake_group_create(int n);
void fake_group_destroy(void* g);
int nccl_unique_id(uint8_t out[128]);

#ifdef __CUDACC__
__host__ __device__
#endif
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace msvd

struct msvd_ctx {
    msvd::Ctx c;
};
struct msvd_matrix {
    msvd_ctx* ctx;
    const double* A;  // dense: row-major rows (kind 0)
    int64_t m_local, n, ld, row0, m_global;
    int kind = msvd::kMatDense;
    // CSR (kind 1): borrowed arrays, local rows; owned transpose (CSC)
    const int64_t* csr_rp = nullptr;
    const void* csr_ci = nullptr;
    int csr_idx64 = 1;
    const double* csr_v = nullptr;
    int64_t csr_nnz = 0;
    int csr_lanes = 1;
    void* csr_owned = nullptr;
    int64_t* csc_cp = nullptr;
    uint32_t* csc_ri = nullptr;
    double* csc_cv = nullptr;
};
