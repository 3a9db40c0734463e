// C++ API over the C ABI, exercised like the reference's own solver tests
// (test_solver.cpp:147-187, :446-477).  Built and run by tests/test_cpp_api.py.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "minsvd_gpu.hpp"

using namespace minsvd::gpu;

static int failures = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::printf("CHECK failed line %d: %s\n", __LINE__, #c);          \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static double* upload(const std::vector<double>& h) {
    double* d = nullptr;
    cudaMalloc(&d, h.size() * sizeof(double));
    cudaMemcpy(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice);
    return d;
}

int main() {
    Context ctx(0);
    {   // tiny diagonal instance (test_solver.cpp:147-165), row-major 50 x 5
        std::vector<double> a(50 * 5, 0.0);
        for (int j = 0; j < 5; ++j) a[j * 5 + j] = 5.0 - j;
        double* d = upload(a);
        DeviceDenseOperator op(ctx, d, 50, 5, 5);
        SolverOptions o;
        o.seed = 7;
        GroundTruth t{1.0, {0, 0, 0, 0, 1.0}};
        SolveResult r = rlobpcg_single(op, o, &t);
        CHECK(r.status == SolveStatus::converged);
        CHECK(std::fabs(r.sigma[0] - 1.0) <= 1e-12);
        CHECK(r.record.rows.back().sin_angle <= 1e-8);
        CHECK(!r.sketch_skipped && r.sketch_dim == 20);
        cudaFree(d);
    }
    {   // block solve ascending (test_solver.cpp:167-187)
        std::vector<double> a(50 * 6, 0.0);
        for (int j = 0; j < 6; ++j) a[j * 6 + j] = 6.0 - j;
        double* d = upload(a);
        DeviceDenseOperator op(ctx, d, 50, 6, 6);
        SolverOptions o;
        o.block_size = 2;
        o.seed = 11;
        SolveResult r = rlobpcg_block(op, o);
        CHECK(r.status == SolveStatus::converged);
        CHECK(r.sigma.size() == 2 && r.sigma[0] < r.sigma[1]);
        CHECK(std::fabs(r.sigma[0] - 1.0) <= 1e-10 && std::fabs(r.sigma[1] - 2.0) <= 1e-10);
        CHECK(std::fabs(std::fabs(r.v[5]) - 1.0) <= 1e-12);      // column 0 ~ e5
        CHECK(std::fabs(std::fabs(r.v[6 + 4]) - 1.0) <= 1e-12);  // column 1 ~ e4
        cudaFree(d);
    }
    {   // validation (test_solver.cpp:446-477)
        std::vector<double> wide(3 * 5, 1.0);
        double* dw = upload(wide);
        DeviceDenseOperator w(ctx, dw, 3, 5, 5);
        SolverOptions o;
        CHECK(throws<DimensionError>([&] { rlobpcg_single(w, o); }));
        std::vector<double> a(40 * 8);
        for (size_t i = 0; i < a.size(); ++i) a[i] = std::sin(0.37 * i) + (i % 9 == 0 ? 2.0 : 0.0);
        double* d = upload(a);
        DeviceDenseOperator op(ctx, d, 40, 8, 8);
        SolverOptions big;
        big.block_size = 3;
        CHECK(throws<DimensionError>([&] { rlobpcg_block(op, big); }));
        SolverOptions bt;
        bt.tol = 1.5;
        CHECK(throws<NumericalError>([&] { rlobpcg_single(op, bt); }));
        SolverOptions bc;
        bc.check_every = 0;
        CHECK(throws<NumericalError>([&] { rlobpcg_single(op, bc); }));
        SolverOptions bs;
        bs.sketch_dim = 30;
        CHECK(throws<DimensionError>([&] { rlobpcg_single(op, bs); }));
        GroundTruth bad{1.0, Vector(3, 0.0)};
        CHECK(throws<DimensionError>([&] { rlobpcg_single(op, SolverOptions{}, &bad); }));
        // products through the operator (apply / apply_adjoint)
        std::vector<double> x(8, 1.0), y(40);
        double* dx = upload(x);
        double* dy = nullptr;
        cudaMalloc(&dy, 40 * sizeof(double));
        op.apply_block(dx, 1, dy);
        cudaMemcpy(y.data(), dy, 40 * sizeof(double), cudaMemcpyDeviceToHost);
        double err = 0.0;
        for (int i = 0; i < 40; ++i) {
            double s = 0.0;
            for (int j = 0; j < 8; ++j) s += a[i * 8 + j];
            err = std::fmax(err, std::fabs(s - y[i]));
        }
        CHECK(err <= 1e-13);
        cudaFree(dx);
        cudaFree(dy);
        cudaFree(d);
        cudaFree(dw);
    }
    {   // CsrOperator (operator.hpp:58-74): the same diagonal instance as CSR,
        // a solve, the column norms, and the reference's validation errors
        const int m = 60, n = 6;
        std::vector<int64_t> rp(m + 1, 0), ci;
        std::vector<double> v;
        for (int i = 0; i < m; ++i) {
            if (i < n) {
                ci.push_back(i);
                v.push_back(6.0 - i);
            }
            rp[i + 1] = static_cast<int64_t>(ci.size());
        }
        int64_t *drp = nullptr, *dci = nullptr;
        cudaMalloc(&drp, rp.size() * sizeof(int64_t));
        cudaMalloc(&dci, ci.size() * sizeof(int64_t));
        cudaMemcpy(drp, rp.data(), rp.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
        cudaMemcpy(dci, ci.data(), ci.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
        double* dv = upload(v);
        DeviceCsrOperator op(ctx, drp, dci, 8, dv, m, n, static_cast<index_t>(v.size()));
        CHECK(op.nnz() == n && op.rows() == m && op.cols() == n);
        SolverOptions o;
        o.seed = 3;
        GroundTruth t{1.0, {0, 0, 0, 0, 0, 1.0}};
        SolveResult r = rlobpcg_single(op, o, &t);
        CHECK(r.status == SolveStatus::converged);
        CHECK(std::fabs(r.sigma[0] - 1.0) <= 1e-12);
        double* dn = nullptr;
        cudaMalloc(&dn, n * sizeof(double));
        op.column_norms(dn);
        std::vector<double> hn(n);
        cudaMemcpy(hn.data(), dn, n * sizeof(double), cudaMemcpyDeviceToHost);
        for (int j = 0; j < n; ++j) CHECK(hn[j] == 6.0 - j);  // operator.cpp:98-104
        // lanczos_gk over the CSR operator (baselines.cpp:51-166): n steps end
        // in an invariant subspace with the exact smallest sigma
        LanczosResult lz = lanczos_gk(op, n, Vector(n, 1.0), &t, false, m);
        CHECK(std::fabs(lz.sigma_min - 1.0) <= 1e-12);
        CHECK(lz.steps >= 1 && lz.steps <= n);
        CHECK(lz.v_basis.size() == static_cast<size_t>(n) * lz.steps);
        // csr.cpp:9-31 errors: a column index out of range
        std::vector<int64_t> bad = ci;
        bad[2] = n + 1;
        cudaMemcpy(dci, bad.data(), bad.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
        CHECK(throws<DimensionError>([&] { DeviceCsrOperator b(ctx, drp, dci, 8, dv, m, n, 6); }));
        cudaFree(drp);
        cudaFree(dci);
        cudaFree(dv);
        cudaFree(dn);
    }
    std::printf("cpp api: %s (%d failures)\n", failures ? "FAIL" : "OK", failures);
    return failures ? 1 : 0;
}
