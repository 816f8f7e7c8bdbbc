// ref_binding.cpp -- the maintainer-side bindings of INTEGRATION.md (section 1:
// solve_scheme4_b200 / solve_scheme3_b200, section 5: make_toeplitz_operator_b200),
// compiled against the reference's own headers (/root/reference/proj/include)
// and linked with the unmodified reference library (oracle/_ref) and
// libfractime_b200.so.  TEST INFRASTRUCTURE: tests/integration/build.sh builds
// it into tests/integration/_build/ (git-ignored, travels to the GPU box);
// tests/test_integration.py runs it on the GPU.
//
// Checks (exit code 0 and one "ok ..." line each):
//   1. solve_scheme4_b200(spec, Direct) == reference solve(spec, Direct)  bitwise
//      (schemes.cpp:434-463; u0 = 0 so the RHS is formed identically)
//   2. solve_scheme4_b200(spec, Fast) within 1e-10 of the reference direct solve
//   3. solve_scheme3_b200(spec, Fast / Direct) with u0, phi callbacks, within 1e-10 /
//      1e-14 of the reference direct solve (schemes.cpp:333-352)
//   4. the reference gmres_solve (krylov.cpp:107-223) driven by the GPU
//      LinearOperator make_toeplitz_operator_b200 converges to the same solution as
//      gmres_solve on the reference's own FFT operator (toeplitz.cpp:198-201), and
//      both match lower_toeplitz_forward_solve (toeplitz.cpp:169-186)
//   5. the GPU block operator (ft_block_matvec) equals block_matvec (toeplitz.cpp:145-167)
//   6. errors map to the reference exception classes (validate: invalid_argument)
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "fractime/krylov.hpp"
#include "fractime/schemes.hpp"
#include "fractime/toeplitz.hpp"
#include "fractime/weights.hpp"
#include "fractime_b200.h"

using namespace fractime;

// ---------------- INTEGRATION.md section 1 (as a maintainer would add it) ----------------
namespace {
double forcing_tramp(double x, double t, void* u) {
    return static_cast<const ProblemSpec*>(u)->forcing(x, t);
}
double u0_tramp(double x, void* u) { return static_cast<const ProblemSpec*>(u)->initial_u0(x); }
double phi_tramp(double x, void* u) { return static_cast<const ProblemSpec*>(u)->initial_phi(x); }

void check(int rc) {
    if (rc == FT_OK) return;
    const std::string msg = ft_last_error();
    if (rc == FT_EINVAL) throw std::invalid_argument(msg);
    if (rc == FT_EDOM) throw std::domain_error(msg);
    if (rc == FT_ELENGTH) throw std::length_error(msg);
    throw std::runtime_error(msg);
}

SchemeSolution solve_b200(const ProblemSpec& spec, SolveMethod method, int scheme) {
    ft_problem p{scheme, spec.gamma, spec.time_steps, spec.space_cells, spec.time_length, spec.space_length};
    ft_plan* plan = nullptr;
    check(ft_setup(&p, nullptr, &plan));
    SchemeSolution out;
    out.grid = {spec.scheme, spec.tau(), spec.h(), spec.time_steps, spec.space_cells, {}};
    out.grid.values.resize((spec.space_cells - 1) * spec.time_steps);
    std::vector<double> rhs(out.grid.values.size());
    const int rc = ft_assemble_rhs(plan, forcing_tramp, spec.initial_u0 ? u0_tramp : nullptr,
                                   spec.initial_phi ? phi_tramp : nullptr, const_cast<ProblemSpec*>(&spec),
                                   rhs.data());
    if (rc != FT_OK) {
        ft_destroy(plan);
        check(rc);
    }
    ft_report rep;
    const int rs = method == SolveMethod::Fast ? ft_solve_fast(plan, rhs.data(), out.grid.values.data(), &rep)
                                               : ft_solve_direct(plan, rhs.data(), out.grid.values.data(), &rep);
    ft_destroy(plan);
    check(rs);
    out.report = {rep.method, rep.iterations, rep.residual, rep.seconds};
    return out;
}
}  // namespace

SchemeSolution solve_scheme4_b200(const ProblemSpec& spec, SolveMethod method) {
    return solve_b200(spec, method, FT_SCHEME_DIFFUSION);
}
SchemeSolution solve_scheme3_b200(const ProblemSpec& spec, SolveMethod method) {
    return solve_b200(spec, method, FT_SCHEME_WAVE);
}

// ---------------- INTEGRATION.md section 5 ----------------
LinearOperator make_toeplitz_operator_b200(const ToeplitzOperator& t) {
    auto col = t.first_col(), row = t.first_row();
    return LinearOperator{t.dim(), [col, row](std::span<const double> x) {
                              std::vector<double> y(x.size());
                              check(ft_toeplitz_matvec(col.data(), row.data(), col.size(), 1, x.data(), y.data()));
                              return y;
                          }};
}

// The reference's make_block_operator (toeplitz.cpp:194-197) on the plan's own matrix: the far
// history through the plan's FFT history products (ft_apply), host spans in and out.
LinearOperator make_block_operator_b200(ft_plan* plan, std::size_t dim) {
    return LinearOperator{dim, [plan](std::span<const double> x) {
                              std::vector<double> y(x.size());
                              check(ft_apply(plan, x.data(), y.data()));
                              return y;
                          }};
}

// ---------------- the checks ----------------
static double relerr(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        num = std::fmax(num, std::fabs(a[i] - b[i]));
        den = std::fmax(den, std::fabs(b[i]));
    }
    return num / std::fmax(den, 1e-300);
}

static int failures = 0;
static void expect(bool ok, const std::string& what, double v) {
    std::printf("%s %s %.3e\n", ok ? "ok" : "FAIL", what.c_str(), v);
    if (!ok) ++failures;
}

int main() {
    const double pi = 3.14159265358979323846;
    try {
        // 1-2: Scheme 4, BASELINE config 2 shape at a reduced size (u0 = 0)
        ProblemSpec s4;
        s4.scheme = SchemeId::Diffusion;
        s4.gamma = 0.7;
        s4.time_steps = 256;
        s4.space_cells = 40;
        s4.forcing = [pi](double x, double t) { return std::sin(pi * x) * (1.0 + t * t) + std::cos(3.0 * x) * t; };
        const auto ref4 = solve(s4, SolveMethod::Direct, SolverConfig{});
        const auto dir4 = solve_scheme4_b200(s4, SolveMethod::Direct);
        const auto fast4 = solve_scheme4_b200(s4, SolveMethod::Fast);
        expect(dir4.grid.values == ref4.grid.values, "scheme4 direct bitwise", relerr(dir4.grid.values, ref4.grid.values));
        expect(relerr(fast4.grid.values, ref4.grid.values) <= 1e-10, "scheme4 fast vs reference direct",
               relerr(fast4.grid.values, ref4.grid.values));
        expect(fast4.report.method == "fast" && dir4.report.method == "direct", "report method strings", 0.0);

        // 3: Scheme 3 with u0 and phi callbacks (reference RHS mode)
        ProblemSpec s3;
        s3.scheme = SchemeId::DiffusionWave;
        s3.gamma = 1.5;
        s3.time_steps = 200;
        s3.space_cells = 33;
        s3.forcing = [pi](double x, double t) { return std::sin(pi * x) * t * t + std::cos(pi * x); };
        s3.initial_u0 = [pi](double x) { return std::sin(pi * x); };
        s3.initial_phi = [pi](double x) { return 0.5 * std::sin(pi * x); };
        const auto ref3 = solve(s3, SolveMethod::Direct, SolverConfig{});
        const auto fast3 = solve_scheme3_b200(s3, SolveMethod::Fast);
        const auto dir3 = solve_scheme3_b200(s3, SolveMethod::Direct);
        expect(relerr(fast3.grid.values, ref3.grid.values) <= 1e-10, "scheme3 fast vs reference direct",
               relerr(fast3.grid.values, ref3.grid.values));
        expect(relerr(dir3.grid.values, ref3.grid.values) <= 1e-14, "scheme3 direct vs reference direct",
               relerr(dir3.grid.values, ref3.grid.values));

        // 4: reference GMRES on the GPU operator (BASELINE config 1 column, N = 512)
        const size_t n = 512;
        const double g = 0.5, tau = 1.0 / 4096.0;
        const auto gw = g_weights(g, n);
        const double mu = std::pow(tau, -g) / std::tgamma(2.0 - g);
        std::vector<double> col(n);
        col[0] = 1.0 + mu * gw.values[0];
        for (size_t j = 1; j < n; ++j) col[j] = mu * (gw.values[j] - gw.values[j - 1]);
        const auto T = ToeplitzOperator::lower_triangular(col);
        std::vector<double> b(n);
        for (size_t i = 0; i < n; ++i) b[i] = 1.0 + std::sin(0.01 * (double)i);
        SolverConfig cfg;
        cfg.tol = 1e-12;
        cfg.restart = 40;
        const auto gpu_op = make_toeplitz_operator_b200(T);
        const auto ref_op = make_toeplitz_operator(embed_circulant(T));
        const auto rg = gmres_solve(gpu_op, b, cfg);
        const auto rr = gmres_solve(ref_op, b, cfg);
        const auto xs = lower_toeplitz_forward_solve(T, b);
        expect(rg.converged, "gmres on the GPU operator converged (matvecs)", (double)rg.iterations);
        expect(relerr(rg.solution, xs) <= 1e-10, "gmres(GPU op) vs forward solve", relerr(rg.solution, xs));
        expect(relerr(rg.solution, rr.solution) <= 1e-10, "gmres(GPU op) vs gmres(reference op)",
               relerr(rg.solution, rr.solution));
        const std::vector<double> ya = gpu_op.apply(b), yb = ref_op.apply(b);
        expect(relerr(ya, yb) <= 1e-13, "toeplitz apply GPU vs reference FFT", relerr(ya, yb));

        // 5: block operator
        BlockTridiagonalToeplitzOperator bop(7, T, -3.5);
        std::vector<double> xb(7 * n);
        for (size_t i = 0; i < xb.size(); ++i) xb[i] = std::cos(0.003 * (double)i);
        const auto yr = block_matvec(bop, xb);
        std::vector<double> yg(xb.size());
        check(ft_block_matvec(col.data(), T.first_row().data(), n, 7, -3.5, xb.data(), yg.data()));
        expect(relerr(yg, yr) <= 1e-13, "block matvec GPU vs reference", relerr(yg, yr));

        // 7: the reference's own Scheme 4 fast path (schemes.cpp:464-474: assemble_scheme4 +
        //    make_block_operator + gmres_solve) with the block operator replaced by the plan's
        //    GPU operator: same Krylov solver, same right-hand side, same answer
        {
            ProblemSpec s7 = s4;
            s7.time_steps = 96;     // three leaves: n = 64 and n = 128 products + in-leaf lags
            s7.space_cells = 13;
            const auto system = assemble_scheme4(s7);
            ft_problem p7{FT_SCHEME_DIFFUSION, s7.gamma, s7.time_steps, s7.space_cells, s7.time_length, s7.space_length};
            ft_plan* plan7 = nullptr;
            check(ft_setup(&p7, nullptr, &plan7));
            const auto gpu_block = make_block_operator_b200(plan7, system.rhs.size());
            const auto ref_block = make_block_operator(system.op);
            std::vector<double> xp(system.rhs.size());
            for (size_t i = 0; i < xp.size(); ++i) xp[i] = std::sin(0.37 * (double)i) + 0.01 * (double)(i % 7);
            const auto ag = gpu_block.apply(xp), ar = ref_block.apply(xp);
            expect(relerr(ag, ar) <= 1e-12, "block operator: ft_apply vs reference block_matvec", relerr(ag, ar));
            SolverConfig c7;
            c7.tol = 1e-11;
            c7.restart = 60;
            c7.max_iter = 20000;
            const auto g7 = gmres_solve(gpu_block, system.rhs, c7);
            const auto d7 = solve(s7, SolveMethod::Direct, SolverConfig{});
            expect(g7.converged, "reference gmres on the plan's GPU block operator converged (matvecs)",
                   (double)g7.iterations);
            expect(relerr(g7.solution, d7.grid.values) <= 1e-8, "gmres(GPU block op) vs reference direct",
                   relerr(g7.solution, d7.grid.values));
            ft_destroy(plan7);
        }

        // 6: error mapping (validate: gamma out of range -> invalid_argument)
        bool threw = false;
        try {
            ProblemSpec bad = s4;
            bad.gamma = 1.2;
            (void)solve_scheme4_b200(bad, SolveMethod::Fast);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        expect(threw, "invalid gamma -> std::invalid_argument", 0.0);
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    return failures ? 1 : 0;
}
