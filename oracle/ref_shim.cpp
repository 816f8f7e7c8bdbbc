// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference library (TEST
// INFRASTRUCTURE ONLY).  oracle/build_ref.sh compiles this file together with
// /root/reference/proj/src/*.cpp (read in place, never copied) into
// oracle/_ref/libfractime_ref.so.  Tests and bench.py's reference arm call the
// reference's own public API through it:
//   fractime::solve(spec, method, cfg)            schemes.hpp:109 / schemes.cpp:481-489
//   fractime::lower_toeplitz_forward_solve        toeplitz.hpp:102 / toeplitz.cpp:169-186
//   fractime::gmres_solve + make_toeplitz_operator krylov.cpp:107-223, toeplitz.cpp:204
//   fractime::g_weights / m_weights / power_step   weights.cpp:8-40
//   fractime::assemble_scheme2_reordered / assemble_scheme3_reordered / assemble_scheme4
//                                                  schemes.cpp:149-167, :272-288, :381-410
// Forcing / initial-data callbacks look values up in caller-supplied grids so
// the reference and the GPU path see bit-identical inputs.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "fractime/schemes.hpp"
#include "fractime/toeplitz.hpp"
#include "fractime/weights.hpp"

using namespace fractime;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}

struct Grids {
    const double* F;
    const double* u0;
    const double* phi;
    std::size_t N;
    std::size_t cells;
    double h, tau, tshift, xshift;
};

std::size_t node_of(const Grids& g, double x) {
    long i = std::lround(x / g.h - g.xshift);
    if (i < 1) i = 1;
    if (i > (long)g.cells - 1) i = (long)g.cells - 1;
    return (std::size_t)i;
}
std::size_t step_of(const Grids& g, double t) {
    long n = std::lround(t / g.tau - g.tshift);
    if (n < 1) n = 1;
    if (n > (long)g.N) n = (long)g.N;
    return (std::size_t)n;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

double ref_power_step(uint64_t k, double p) { return power_step(k, p); }

// kind 0 = G (0<gamma<1), 1 = M (1<gamma<2).  Returns -1 with the reference's
// exception message on domain errors.
int ref_weights(int kind, double gamma, uint64_t count, double* out) {
    try {
        auto w = kind == 0 ? g_weights(gamma, count) : m_weights(gamma, count);
        std::memcpy(out, w.values.data(), sizeof(double) * count);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// scheme: 1 = Hyperbolic (Scheme 2), 2 = DiffusionWave (Scheme 3), 3 = Diffusion (Scheme 4)
// method: 2 = Direct, 3 = Fast.  F: node-major forcing grid at the scheme's
// evaluation points (S4: (i h, n tau); S3: (i h, (n-1/2) tau); S2: ((i-1/2) h, n tau)).
// u0: interior nodes x_1..x_{cells-1}, except Scheme 2: x_0..x_{cells-1}.
int ref_solve(int scheme, int method, double gamma, uint64_t time_steps, uint64_t space_cells,
              double time_length, double space_length, const double* F, const double* u0,
              const double* phi, double tol, uint64_t restart, uint64_t max_iter, double* U,
              uint64_t* iterations, double* seconds) {
    try {
        ProblemSpec spec;
        spec.scheme = scheme == 1 ? SchemeId::Hyperbolic : scheme == 2 ? SchemeId::DiffusionWave : SchemeId::Diffusion;
        spec.gamma = gamma;
        spec.time_steps = time_steps;
        spec.space_cells = space_cells;
        spec.time_length = time_length;
        spec.space_length = space_length;
        auto g = std::make_shared<Grids>(Grids{F, u0, phi, time_steps, space_cells, spec.h(),
                                               spec.tau(), scheme == 2 ? -0.5 : 0.0, scheme == 1 ? -0.5 : 0.0});
        spec.forcing = [g](double x, double t) {
            return g->F[(node_of(*g, x) - 1) * g->N + (step_of(*g, t) - 1)];
        };
        if (u0 && scheme == 1) {
            spec.initial_u0 = [g](double x) {
                long i = std::lround(x / g->h);
                if (i < 0) i = 0;
                if (i > (long)g->cells - 1) i = (long)g->cells - 1;
                return g->u0[i];
            };
        } else if (u0) {
            spec.initial_u0 = [g](double x) { return g->u0[node_of(*g, x) - 1]; };
        }
        if (phi) spec.initial_phi = [g](double x) { return g->phi[node_of(*g, x) - 1]; };
        SolverConfig cfg;
        if (tol > 0) cfg.tol = tol;
        if (restart > 0) cfg.restart = restart;
        if (max_iter > 0) cfg.max_iter = max_iter;
        auto sol = solve(spec, method == 2 ? SolveMethod::Direct : SolveMethod::Fast, cfg);
        std::memcpy(U, sol.grid.values.data(), sizeof(double) * sol.grid.values.size());
        if (iterations) *iterations = sol.report.iterations;
        if (seconds) *seconds = sol.report.seconds;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Config 1 (one-sided fractional ODE) through the reference's Toeplitz API
// (SURVEY.md 3.4): column from g_weights + SchemeConstants, then either the
// O(n^2) forward substitution (direct) or GMRES on the FFT circulant matvec.
int ref_ode_column(double gamma, uint64_t N, double time_length, double* col) {
    try {
        ProblemSpec spec;
        spec.scheme = SchemeId::Ode2Sided;
        spec.gamma = gamma;
        spec.time_steps = N;
        spec.time_length = time_length;
        const auto k = SchemeConstants::for_spec(spec);
        const auto g = g_weights(gamma, N);
        col[0] = 1.0 + k.mu * g.values[0];
        for (std::size_t j = 1; j < N; ++j) col[j] = k.mu * (g.values[j] - g.values[j - 1]);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Scheme setup through the reference's own assembly (schemes.cpp:149-167, :272-288,
// :381-410): the Toeplitz first column (Scheme 2: A~ and B~) and, for Scheme 4,
// the assembled right-hand side from grid callbacks (rhs may be null).
int ref_setup(int scheme, double gamma, uint64_t time_steps, uint64_t space_cells, double time_length,
              double space_length, const double* F, const double* u0, double* col, double* col2, double* off,
              double* rhs) {
    try {
        ProblemSpec spec;
        spec.scheme = scheme == 1 ? SchemeId::Hyperbolic : scheme == 2 ? SchemeId::DiffusionWave : SchemeId::Diffusion;
        spec.gamma = gamma;
        spec.time_steps = time_steps;
        spec.space_cells = space_cells;
        spec.time_length = time_length;
        spec.space_length = space_length;
        auto g = std::make_shared<Grids>(Grids{F, u0, nullptr, time_steps, space_cells, spec.h(), spec.tau(),
                                               0.0, 0.0});
        spec.forcing = [g](double x, double t) {
            return g->F ? g->F[(node_of(*g, x) - 1) * g->N + (step_of(*g, t) - 1)] : 0.0;
        };
        if (u0) spec.initial_u0 = [g](double x) { return g->u0[node_of(*g, x) - 1]; };
        const std::size_t N = time_steps;
        if (scheme == 1) {
            auto r = assemble_scheme2_reordered(spec);
            std::memcpy(col, r.a_tilde.first_col().data(), sizeof(double) * N);
            if (col2) std::memcpy(col2, r.b_tilde.first_col().data(), sizeof(double) * N);
        } else if (scheme == 2) {
            auto t = assemble_scheme3_reordered(spec);
            std::memcpy(col, t.first_col().data(), sizeof(double) * N);
        } else {
            auto sys = assemble_scheme4(spec);
            std::memcpy(col, sys.op.diag_block().first_col().data(), sizeof(double) * N);
            if (off) *off = sys.op.off_block_scale();
            if (rhs) std::memcpy(rhs, sys.rhs.data(), sizeof(double) * sys.rhs.size());
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_forward_solve(const double* col, const double* b, uint64_t n, double* x) {
    try {
        auto t = ToeplitzOperator::lower_triangular(std::vector<double>(col, col + n));
        auto y = lower_toeplitz_forward_solve(t, std::span<const double>(b, n));
        std::memcpy(x, y.data(), sizeof(double) * n);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// embed_circulant + toeplitz_matvec (toeplitz.cpp:84-115): the reference's FFT path
int ref_toeplitz_matvec(const double* col, const double* row, uint64_t n, const double* x, double* y) {
    try {
        auto t = ToeplitzOperator::general(std::vector<double>(col, col + n), std::vector<double>(row, row + n));
        auto v = toeplitz_matvec(embed_circulant(t), std::span<const double>(x, n));
        std::memcpy(y, v.data(), sizeof(double) * n);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// BlockTridiagonalToeplitzOperator + block_matvec (toeplitz.cpp:117-167)
int ref_block_matvec(const double* col, const double* row, uint64_t n, uint64_t m, double beta, const double* x,
                     double* y) {
    try {
        auto t = ToeplitzOperator::general(std::vector<double>(col, col + n), std::vector<double>(row, row + n));
        BlockTridiagonalToeplitzOperator op(m, t, beta);
        auto v = block_matvec(op, std::span<const double>(x, n * m));
        std::memcpy(y, v.data(), sizeof(double) * n * m);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_toeplitz_gmres(const double* col, const double* b, uint64_t n, double tol,
                       uint64_t restart, double* x, uint64_t* iterations) {
    try {
        auto t = ToeplitzOperator::lower_triangular(std::vector<double>(col, col + n));
        auto op = make_toeplitz_operator(embed_circulant(t));
        SolverConfig cfg;
        cfg.tol = tol;
        if (restart > 0) cfg.restart = restart;
        auto res = gmres_solve(op, std::span<const double>(b, n), cfg);
        std::memcpy(x, res.solution.data(), sizeof(double) * n);
        if (iterations) *iterations = res.iterations;
        return res.converged ? 0 : 1;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
