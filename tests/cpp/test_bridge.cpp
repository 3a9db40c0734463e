// The device path behind the reference's own types (include/minsvd_bridge.hpp),
// checked the way the reference's test_solver.cpp checks its solver:
//   1. the reference's CPU lobpcg_solve drives a CountingOperator over the
//      DeviceDenseOperatorAdapter: every product runs on the GPU, the
//      counts are the reference's (test_solver.cpp:237-265);
//   2. gpu_rlobpcg_single / gpu_rlobpcg_block return a minsvd::SolveResult
//      that matches the reference's own solve on the same matrix (sigma,
//      v, record rows, to_csv columns, Preconditioner fields);
//   3. the device stop rule on the reference's synthetic histories
//      (test_solver.cpp:84-145) gives the reference's decisions;
//   4. no CPU fallback: any other operator is a DimensionError.
// Built by oracle/Makefile (`make bridge`) against /root/reference/proj/include
// and the reference library; run by tests/test_bridge.py on the GPU.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "minsvd/matgen.hpp"
#include "minsvd/svd.hpp"
#include "minsvd_bridge.hpp"

using namespace minsvd;

static int failures = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (!(cond)) {                                                         \
            std::printf("CHECK failed at %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                        \
        }                                                                      \
    } while (0)

namespace {

DenseMatrix random_matrix(index_t m, index_t n, std::uint64_t seed) {
    SplitMix64 rng(seed);
    DenseMatrix a(m, n);
    for (index_t j = 0; j < n; ++j)
        for (index_t i = 0; i < m; ++i) a(i, j) = rng.next_gaussian();
    return a;
}

struct Instance {
    DenseMatrix a;
    Vector sigma;
    DenseMatrix vfull;
    GroundTruth truth() const { return {sigma.back(), vfull.col_copy(vfull.cols() - 1)}; }
};

// test_solver.cpp:50-62 make_instance
Instance make_instance(index_t m, index_t n, Vector sigma_desc, std::uint64_t seed) {
    Instance inst;
    DenseMatrix u = qr_q_economy(householder_qr(random_matrix(m, n, seed)));
    inst.vfull = qr_q_economy(householder_qr(random_matrix(n, n, seed ^ 0xabcdef123456ull)));
    for (index_t j = 0; j < n; ++j) {
        double* c = u.col(j);
        for (index_t i = 0; i < m; ++i) c[i] *= sigma_desc[static_cast<std::size_t>(j)];
    }
    inst.a = matmul(u, transpose(inst.vfull));
    inst.sigma = std::move(sigma_desc);
    return inst;
}

Vector geometric_spectrum(index_t n, double last) {
    Vector s(static_cast<std::size_t>(n));
    for (index_t i = 0; i < n; ++i)
        s[static_cast<std::size_t>(i)] = std::pow(last, static_cast<double>(i) / static_cast<double>(n - 1));
    return s;
}

double sin_between(const Vector& ref, const DenseMatrix& v, index_t col) {
    // || ref - v (v^T ref) ||, both unit
    double c = 0.0;
    for (index_t i = 0; i < v.rows(); ++i) c += v(i, col) * ref[static_cast<std::size_t>(i)];
    double s = 0.0;
    for (index_t i = 0; i < v.rows(); ++i) {
        const double d = ref[static_cast<std::size_t>(i)] - v(i, col) * c;
        s += d * d;
    }
    return std::sqrt(s);
}

msvd_ctx* make_ctx() {
    msvd_ctx_desc desc{};
    desc.device = 0;
    msvd_ctx* ctx = nullptr;
    if (msvd_ctx_create(&desc, &ctx) != MSVD_OK) {
        std::printf("msvd_ctx_create: %s\n", msvd_last_error());
        std::exit(2);
    }
    return ctx;
}

std::string csv_header(const std::string& csv) { return csv.substr(0, csv.find('\n')); }

}  // namespace

int main() {
    msvd_ctx* ctx = make_ctx();

    // ---- 1. the reference solver drives the device operator -------------
    {
        Instance inst = make_instance(120, 12, geometric_spectrum(12, 1e-5), 77);
        SolverOptions opts;
        opts.seed = 3;
        opts.max_iter = 37;
        opts.tol = 0.0;
        opts.record_timing = false;
        DeviceDenseOperatorAdapter dev(ctx, inst.a);
        CountingOperator counted(dev);
        SolveResult plain = rlobpcg_single(counted, opts);  // the REFERENCE's solver
        CHECK(plain.status == SolveStatus::max_iter_reached);
        CHECK(plain.iterations() == 37);
        CHECK(counted.applies() == 38);
        CHECK(counted.adjoints() == 38);
        CHECK(plain.record.rows.back().matvecs_a == 38);
        DenseOperator cpu(inst.a);
        SolveResult host = rlobpcg_single(cpu, opts);
        CHECK(std::fabs(plain.sigma[0] - host.sigma[0]) <= 1e-10 * host.sigma_max_estimate);
        CHECK(sin_between(host.v.col_copy(0), plain.v, 0) <= 1e-8);
        // block products in one device pass equal the column-by-column ones
        DenseMatrix x = random_matrix(12, 3, 5);
        DenseMatrix y = dev.apply_block(x);
        DenseMatrix yh = cpu.apply_block(x);
        double worst = 0.0;
        for (index_t j = 0; j < 3; ++j)
            for (index_t i = 0; i < 120; ++i) worst = std::fmax(worst, std::fabs(y(i, j) - yh(i, j)));
        CHECK(worst <= 1e-13);
        Vector nd = dev.column_norms(), nh = cpu.column_norms();
        for (std::size_t j = 0; j < nd.size(); ++j) CHECK(nd[j] == nh[j]);
        DenseMatrix back = dev.to_dense();
        CHECK(back(7, 3) == inst.a(7, 3) && back(119, 11) == inst.a(119, 11));
        std::printf("reference solver over the device operator: %ld applies, %ld adjoints\n", counted.applies(),
                    counted.adjoints());
    }

    // ---- 2. the whole solve on the device, reference result types --------
    {
        Vector spec(100);
        for (index_t i = 0; i + 1 < 100; ++i)
            spec[static_cast<std::size_t>(i)] = std::pow(10.0, -static_cast<double>(i) / 98.0);
        spec[99] = 1e-7;
        Instance inst = make_instance(2000, 100, spec, 3);
        GroundTruth truth = inst.truth();
        SolverOptions opts;
        opts.seed = 12;
        opts.use_stagnation = false;
        opts.tol = 1e-12;
        opts.record_timing = false;
        DenseOperator cpu(inst.a);
        SolveResult ref = rlobpcg_single(cpu, opts, &truth);
        DeviceDenseOperatorAdapter dev(ctx, inst.a);
        SolveResult got = gpu_rlobpcg_single(dev, opts, &truth);
        CHECK(got.status == ref.status);
        CHECK(std::abs(static_cast<long>(got.iterations()) - static_cast<long>(ref.iterations())) <= 1);
        CHECK(std::fabs(got.sigma[0] - ref.sigma[0]) <= 1e-10 * ref.sigma_max_estimate);
        CHECK(sin_between(ref.v.col_copy(0), got.v, 0) <= 1e-8);
        CHECK(got.v.rows() == 100 && got.v.cols() == 1);
        CHECK(std::fabs(got.sigma_max_estimate - ref.sigma_max_estimate) <= 1e-12 * ref.sigma_max_estimate);
        CHECK(got.precond.vtilde.rows() == 100 && got.precond.vtilde.cols() == 100);
        CHECK(got.precond.sigma_tilde.size() == 100);
        CHECK(std::fabs(got.precond.sigma_tilde[0] - ref.precond.sigma_tilde[0]) <= 1e-12 * ref.sigma_max_estimate);
        CHECK(got.precond.floor_count == ref.precond.floor_count);
        CHECK(got.sketch_dim == ref.sketch_dim && got.zeta == ref.zeta && got.sketch_skipped == ref.sketch_skipped);
        // sketch_and_solve_init (precond.cpp:50-57) on the returned preconditioner
        DenseMatrix v0 = sketch_and_solve_init(got.precond, 1);
        DenseMatrix v0r = sketch_and_solve_init(ref.precond, 1);
        CHECK(sin_between(v0r.col_copy(0), v0, 0) <= 1e-8);
        // the record is the reference's type: to_csv() (solver.cpp:149-171)
        const std::string csv = got.record.to_csv(), csv_ref = ref.record.to_csv();
        CHECK(csv_header(csv) == csv_header(csv_ref));
        CHECK(got.record.has_truth);
        for (std::size_t r = 0; r < got.record.rows.size() && r < ref.record.rows.size(); ++r) {
            CHECK(got.record.rows[r].iter == ref.record.rows[r].iter);
            CHECK(got.record.rows[r].matvecs_a == ref.record.rows[r].matvecs_a);
            CHECK(got.record.rows[r].matvecs_at == ref.record.rows[r].matvecs_at);
            CHECK(std::fabs(got.record.rows[r].theta - ref.record.rows[r].theta) <= 1e-10 * ref.sigma_max_estimate);
        }
        // product counters of the device solve: b (1 + iterations) per side
        CHECK(got.record.rows.back().matvecs_a == 1 + got.iterations());
        // store_iterates fills the reference's trail vectors
        SolverOptions so = opts;
        so.store_iterates = true;
        so.max_iter = 8;
        SolveResult tr = gpu_rlobpcg_single(dev, so);
        CHECK(tr.trail_t.size() == 8 && tr.trail_v.size() == 9);
        CHECK(tr.trail_t[2].rows() == 100 && tr.trail_t[2].cols() == 3);
        // a CountingOperator over the adapter is unwrapped (sketch.cpp:121)
        CountingOperator counted(dev);
        SolveResult viac = gpu_rlobpcg_single(counted, opts, &truth);
        CHECK(viac.sigma[0] == got.sigma[0]);
        // block mode (test_solver.cpp:167-187 shape)
        DenseMatrix diag(50, 6);
        for (index_t j = 0; j < 6; ++j) diag(j, j) = 6.0 - static_cast<double>(j);
        DeviceDenseOperatorAdapter dd(ctx, diag);
        SolverOptions bo;
        bo.block_size = 2;
        bo.seed = 11;
        SolveResult blk = gpu_rlobpcg_block(dd, bo);
        CHECK(blk.status == SolveStatus::converged);
        CHECK(blk.sigma[0] < blk.sigma[1]);
        CHECK(std::fabs(blk.sigma[0] - 1.0) <= 1e-10 && std::fabs(blk.sigma[1] - 2.0) <= 1e-10);
        std::printf("device solve: %ld iterations (reference %ld), sigma %.17g (reference %.17g)\n",
                    static_cast<long>(got.iterations()), static_cast<long>(ref.iterations()), got.sigma[0],
                    ref.sigma[0]);
    }

    // ---- 3. the device stop rule on the reference's synthetic histories --
    {
        const double s1 = 1.0, tol = 1e-10;
        std::vector<double> resid, theta;
        for (int j = 0; j <= 11; ++j) {
            resid.push_back(1e-8 * std::pow(0.5, j));
            theta.push_back(1.0 + std::pow(0.25, j));
        }
        for (int i : {10, 5, 0}) {
            for (bool stag : {true, false}) {
                StopDecision g = gpu_check_convergence(resid, theta, i, s1, tol, 1.1, stag);
                StopDecision r = check_convergence(resid, theta, i, s1, tol, 1.1, stag);
                CHECK(g.tol_ok == r.tol_ok && g.resid_stalled == r.resid_stalled &&
                      g.progress_stalled == r.progress_stalled && g.stop == r.stop);
            }
        }
        std::vector<double> flat(12, 1e-20), one(12, 1.0), zero(12, 0.0), high(12, 1e-3);
        StopDecision d10 = gpu_check_convergence(flat, one, 10, s1, tol, 1.1, true);
        CHECK(d10.tol_ok && d10.resid_stalled && d10.progress_stalled && d10.stop);
        StopDecision d5 = gpu_check_convergence(flat, one, 5, s1, tol, 1.1, true);
        CHECK(d5.tol_ok && d5.resid_stalled && !d5.progress_stalled && !d5.stop);
        CHECK(!gpu_check_convergence(flat, one, 0, s1, tol, 1.1, true).stop);
        StopDecision st = gpu_check_convergence(high, one, 10, s1, tol, 1.1, true);
        CHECK(!st.tol_ok && st.resid_stalled && !st.stop);
        CHECK(gpu_check_convergence(flat, zero, 10, s1, tol, 1.1, true).stop);
        StopDecision to = gpu_check_convergence({1e-3, 1e-20}, {1.0, 1.0}, 0, s1, tol, 1.1, false);
        CHECK(to.tol_ok && to.stop);
        bool threw = false;
        try {
            gpu_check_convergence({1.0, 0.5}, {1.0, 1.0}, 5, s1, tol, 1.1, true);
        } catch (const DimensionError&) {
            threw = true;
        }
        CHECK(threw);
    }

    // ---- 4. no CPU fallback ---------------------------------------------
    {
        Instance inst = make_instance(60, 6, geometric_spectrum(6, 1e-2), 9);
        DenseOperator cpu(inst.a);
        bool threw = false;
        try {
            gpu_rlobpcg_single(cpu, SolverOptions{});
        } catch (const DimensionError&) {
            threw = true;
        }
        CHECK(threw);
        // the reference's validation order and classes through the device path
        DeviceDenseOperatorAdapter dev(ctx, inst.a);
        SolverOptions bad;
        bad.tol = 1.5;
        threw = false;
        try {
            gpu_rlobpcg_single(dev, bad);
        } catch (const NumericalError&) {
            threw = true;
        }
        CHECK(threw);
    }

    msvd_ctx_destroy(ctx);
    if (failures) {
        std::printf("bridge: %d check(s) FAILED\n", failures);
        return 1;
    }
    std::printf("bridge: OK\n");
    return 0;
}
