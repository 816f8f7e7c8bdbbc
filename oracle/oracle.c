/*
 * oracle.c -- CPU restatement of the reference (`fractime`, arXiv 1710.11593)
 * direct solvers for the L1-Caputo block lower-triangular Toeplitz systems.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_1710_11593_b200/)
 * links, loads or calls this file.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, as the checker.
 *
 * Pinning: every double-precision routine here follows the reference's
 * expression order exactly (compiled with -O2 -ffp-contract=off, same glibc
 * libm), so it reproduces the reference bit-for-bit.  tests/test_oracle.py
 * checks this against the unmodified reference built by oracle/build_ref.sh
 * (oracle/_ref/) and against the reference's own known-answer tests
 * (tests/golden/).  The long-double routines are a higher-precision
 * restatement of the same recurrences (used where the reference's own fp64
 * rounding is the limiting factor).
 *
 * Layout convention (reference schemes.hpp:209-223): node-major,
 *   values[(i-1)*N + (n-1)] = U_i^n,  i = 1..cells-1,  n = 1..N.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ---- weights: reference proj/src/weights.cpp:8-16, :28-40 ---------------- */

double or_power_step(uint64_t k, double p) {
    if (k == 0) return 1.0;
    const double kd = (double)k;
    if (k > 1000000) return pow(kd, p) * expm1(p * log1p(1.0 / kd));
    return pow(kd + 1.0, p) - pow(kd, p);
}

void or_weights(double p, uint64_t count, double* out) {
    for (uint64_t k = 0; k < count; ++k) out[k] = or_power_step(k, p);
}

/* ---- constants: reference proj/src/schemes.cpp:44-56 ---------------------- */
/* scheme ids follow or_scheme in oracle.h */
void or_constants(int scheme, double gamma, double tau, double* mu, double* c) {
    const double g = gamma;
    *mu = pow(tau, -g) / tgamma(2.0 - g);
    switch (scheme) {
        case OR_ODE: *c = *mu; break;
        case OR_HYPER: *c = pow(tau, -g) / (2.0 * tgamma(2.0 - g)); break;
        case OR_WAVE: *c = pow(tau, -g) / tgamma(3.0 - g); break;
        case OR_DIFFUSION: *c = pow(tau, -g) / tgamma(2.0 - g); break;
        default: *c = *mu;
    }
}

/* ---- Toeplitz first columns ---------------------------------------------- */

/* Scheme 4: reference schemes.cpp:393-396. */
void or_col_s4(double gamma, uint64_t N, double h, double tau, double* col) {
    double mu, c;
    or_constants(OR_DIFFUSION, gamma, tau, &mu, &c);
    double* g = (double*)malloc(sizeof(double) * N);
    or_weights(1.0 - gamma, N, g);
    col[0] = 2.0 / (h * h) + c * g[0];
    for (uint64_t j = 1; j < N; ++j) col[j] = c * (g[j] - g[j - 1]);
    free(g);
}

/* Scheme 2 (reordered, per node): reference assemble_scheme2_reordered,
 * schemes.cpp:160-165.  a = A~ first column, b = B~ first column. */
void or_col_s2(double gamma, uint64_t N, double h, double tau, double* a, double* b) {
    double mu, c;
    or_constants(OR_HYPER, gamma, tau, &mu, &c);
    double* g = (double*)malloc(sizeof(double) * N);
    or_weights(1.0 - gamma, N, g);
    a[0] = 1.0 / h + c * g[0];
    if (b) b[0] = 1.0 / h - c * g[0];
    for (uint64_t j = 1; j < N; ++j) {
        a[j] = c * (g[j] - g[j - 1]);
        if (b) b[j] = c * (g[j - 1] - g[j]);
    }
    free(g);
}

/* Scheme 3 (reordered, per node): reference schemes.cpp:277-287. */
void or_col_s3(double gamma, uint64_t N, double h, double tau, double* col) {
    double mu, c;
    or_constants(OR_WAVE, gamma, tau, &mu, &c);
    double* m = (double*)malloc(sizeof(double) * (N + 1));
    or_weights(2.0 - gamma, N + 1, m);
    col[0] = 1.0 / h + c * m[0];
    if (N > 1) col[1] = c * (m[1] - 2.0 * m[0]);
    for (uint64_t j = 2; j < N; ++j) col[j] = c * (m[j - 2] - 2.0 * m[j - 1] + m[j]);
    free(m);
}

/* One-sided fractional ODE D^g u + u = f (BASELINE config 1): the Scheme-4
 * column pattern (schemes.cpp:393-396) with the spatial 2/h^2 replaced by the
 * reaction coefficient 1: col0 = 1 + mu*G0, colj = mu(Gj-Gj-1). */
void or_col_ode(double gamma, uint64_t N, double tau, double* col) {
    double mu, c;
    or_constants(OR_ODE, gamma, tau, &mu, &c);
    double* g = (double*)malloc(sizeof(double) * N);
    or_weights(1.0 - gamma, N, g);
    col[0] = 1.0 + mu * g[0];
    for (uint64_t j = 1; j < N; ++j) col[j] = mu * (g[j] - g[j - 1]);
    free(g);
}

/* ---- right-hand sides ---------------------------------------------------- */

/* Scheme 4: reference schemes.cpp:401-408, R = f(x_i, n tau) + c G_{n-1} u0(x_i).
 * F is the node-major forcing grid f(x_i, t_n). */
void or_rhs_s4(double gamma, uint64_t cells, uint64_t N, double tau, const double* F,
               const double* u0, double* R) {
    double mu, c;
    or_constants(OR_DIFFUSION, gamma, tau, &mu, &c);
    double* g = (double*)malloc(sizeof(double) * N);
    or_weights(1.0 - gamma, N, g);
    for (uint64_t i = 0; i + 1 < cells; ++i) {
        const double u = u0 ? u0[i] : 0.0;
        for (uint64_t n = 0; n < N; ++n) R[i * N + n] = F[i * N + n] + c * g[n] * u;
    }
    free(g);
}

/* Scheme 3: reference Scheme3Rhs schemes.cpp:300-306.  F holds f(x_i,(n-1/2)tau).
 * mode 0 reproduces the reference (no u0 term at n = 1, schemes.cpp:304);
 * mode 1 ("corrected-n1") adds the  +c*M_0*u0  term at n = 1 that the L1
 * derivation gives and the reference omits (probe P2). */
void or_rhs_s3(double gamma, uint64_t cells, uint64_t N, double tau, const double* F,
               const double* u0, const double* phi, int mode, double* R) {
    double mu, c;
    or_constants(OR_WAVE, gamma, tau, &mu, &c);
    double* m = (double*)malloc(sizeof(double) * (N + 1));
    or_weights(2.0 - gamma, N + 1, m);
    for (uint64_t i = 0; i + 1 < cells; ++i) {
        const double u = u0 ? u0[i] : 0.0, p = phi ? phi[i] : 0.0;
        for (uint64_t n = 1; n <= N; ++n) {
            double value = F[i * N + (n - 1)] + c * tau * m[n - 1] * p;
            if (n >= 2) value -= c * (m[n - 2] - m[n - 1]) * u;
            else if (mode == 1) value += c * m[0] * u;
            R[i * N + (n - 1)] = value;
        }
    }
    free(m);
}

/* Scheme 2: reference Scheme2Rhs schemes.cpp:183-187,
 * R = f(x_{i-1/2}, n tau) + c g_{n-1} (u0(x_i) + u0(x_{i-1})).  F holds the
 * forcing at ((i - 1/2) h, n tau); u0 holds u0 at x_0 .. x_{cells-1} (cells
 * values, the left boundary included). */
void or_rhs_s2(double gamma, uint64_t cells, uint64_t N, double tau, const double* F,
               const double* u0, double* R) {
    double mu, c;
    or_constants(OR_HYPER, gamma, tau, &mu, &c);
    double* g = (double*)malloc(sizeof(double) * N);
    or_weights(1.0 - gamma, N, g);
    for (uint64_t i = 1; i < cells; ++i) {
        const double us = u0 ? (u0[i] + u0[i - 1]) : 0.0;
        for (uint64_t n = 1; n <= N; ++n)
            R[(i - 1) * N + (n - 1)] = F[(i - 1) * N + (n - 1)] + c * g[n - 1] * us;
    }
    free(g);
}

/* ODE: R_n = f(n tau) + mu G_{n-1} u0 (the Scheme-4 RHS pattern, schemes.cpp:407). */
void or_rhs_ode(double gamma, uint64_t N, double tau, const double* F, double u0, double* R) {
    double mu, c;
    or_constants(OR_ODE, gamma, tau, &mu, &c);
    double* g = (double*)malloc(sizeof(double) * N);
    or_weights(1.0 - gamma, N, g);
    for (uint64_t n = 0; n < N; ++n) R[n] = F[n] + mu * g[n] * u0;
    free(g);
}

/* ---- direct solvers (fp64, reference summation order) -------------------- */

/* Reference toeplitz.cpp:169-186 (lower_toeplitz_forward_solve). Returns -1 on
 * a zero diagonal (the reference throws std::runtime_error). */
int or_forward_solve(const double* col, const double* b, uint64_t n, double* x) {
    if (col[0] == 0.0) return -1;
    for (uint64_t i = 0; i < n; ++i) {
        double acc = b[i];
        for (uint64_t j = 0; j < i; ++j) acc -= col[i - j] * x[j];
        x[i] = acc / col[0];
    }
    return 0;
}

/* Reference ToeplitzOperator::entry + DenseMatrix::multiply (toeplitz.hpp:44-46,
 * toeplitz.cpp:14-23): y = dense(T) x, acc over j ascending.  This is the
 * reference's own oracle for toeplitz_matvec (toeplitz.hpp:11-12). */
void or_toeplitz_matvec(const double* col, const double* row, uint64_t n, const double* x, double* y) {
    for (uint64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (uint64_t j = 0; j < n; ++j) acc += (j >= i ? row[j - i] : col[i - j]) * x[j];
        y[i] = acc;
    }
}

/* Reference block_matvec (toeplitz.cpp:150-167) with the dense diagonal product:
 * y_b = T x_b, then += beta x_{b-1}, then += beta x_{b+1}. */
void or_block_matvec(const double* col, const double* row, uint64_t n, uint64_t m, double beta, const double* x,
                     double* y) {
    for (uint64_t b = 0; b < m; ++b) {
        or_toeplitz_matvec(col, row, n, x + b * n, y + b * n);
        if (b > 0)
            for (uint64_t k = 0; k < n; ++k) y[b * n + k] += beta * x[(b - 1) * n + k];
        if (b + 1 < m)
            for (uint64_t k = 0; k < n; ++k) y[b * n + k] += beta * x[(b + 1) * n + k];
    }
}

/* Reference solve_scheme4 Direct, schemes.cpp:434-463.  F: f(x_i, n tau). */
void or_direct_s4(double gamma, uint64_t cells, uint64_t N, double h, double tau,
                  const double* F, const double* u0, double* U) {
    double mu, c;
    or_constants(OR_DIFFUSION, gamma, tau, &mu, &c);
    double* g = (double*)malloc(sizeof(double) * N);
    or_weights(1.0 - gamma, N, g);
    const uint64_t dim = cells - 1;
    const double diag = 2.0 / (h * h) + c * g[0];
    const double off = -1.0 / (h * h);
    double* cprime = (double*)malloc(sizeof(double) * dim);
    double* rhs = (double*)malloc(sizeof(double) * dim);
    memset(U, 0, sizeof(double) * dim * N);
    for (uint64_t n = 1; n <= N; ++n) {
        for (uint64_t i = 1; i < cells; ++i) {
            double hist = 0.0;
            for (uint64_t k = 1; k < n; ++k)
                hist += (g[n - k - 1] - g[n - k]) * U[(i - 1) * N + (k - 1)];
            const double u = u0 ? u0[i - 1] : 0.0;
            rhs[i - 1] = F[(i - 1) * N + (n - 1)] + c * hist + c * g[n - 1] * u;
        }
        double denom = diag;
        cprime[0] = off / denom;
        rhs[0] /= denom;
        for (uint64_t i = 1; i < dim; ++i) {
            denom = diag - off * cprime[i - 1];
            cprime[i] = off / denom;
            rhs[i] = (rhs[i] - off * rhs[i - 1]) / denom;
        }
        for (uint64_t i = dim - 1; i-- > 0;) rhs[i] -= cprime[i] * rhs[i + 1];
        for (uint64_t i = 1; i < cells; ++i) U[(i - 1) * N + (n - 1)] = rhs[i - 1];
    }
    free(g);
    free(cprime);
    free(rhs);
}

/* Reference solve_scheme3 Direct, schemes.cpp:333-352 (with Scheme3Rhs
 * :300-306; rhs_mode as in or_rhs_s3).  F: f(x_i, (n-1/2) tau). */
void or_direct_s3(double gamma, uint64_t cells, uint64_t N, double h, double tau,
                  const double* F, const double* u0, const double* phi, int rhs_mode,
                  double* U) {
    double mu, c;
    or_constants(OR_WAVE, gamma, tau, &mu, &c);
    double* m = (double*)malloc(sizeof(double) * (N + 1));
    or_weights(2.0 - gamma, N + 1, m);
    double* R = (double*)malloc(sizeof(double) * (cells - 1) * N);
    or_rhs_s3(gamma, cells, N, tau, F, u0, phi, rhs_mode, R);
    double* history = (double*)malloc(sizeof(double) * (cells - 1));
    memset(U, 0, sizeof(double) * (cells - 1) * N);
    for (uint64_t n = 1; n <= N; ++n) {
        for (uint64_t i = 0; i + 1 < cells; ++i) history[i] = 0.0;
        if (n >= 2) {
            const double w1 = c * (m[1] - 2.0 * m[0]);
            for (uint64_t i = 1; i < cells; ++i) history[i - 1] += w1 * U[(i - 1) * N + (n - 2)];
            for (uint64_t k = 1; k + 1 < n; ++k) {
                const uint64_t j = n - k;
                const double w = c * (m[j - 2] - 2.0 * m[j - 1] + m[j]);
                for (uint64_t i = 1; i < cells; ++i)
                    history[i - 1] += w * U[(i - 1) * N + (k - 1)];
            }
        }
        double u_left = 0.0;
        for (uint64_t i = 1; i < cells; ++i) {
            const double value =
                (R[(i - 1) * N + (n - 1)] - history[i - 1] + u_left / h) / (c * m[0] + 1.0 / h);
            U[(i - 1) * N + (n - 1)] = value;
            u_left = value;
        }
    }
    free(m);
    free(R);
    free(history);
}

/* Reference solve_scheme2 Direct, schemes.cpp:210-232 (with Scheme2Rhs
 * :183-187; u0 as in or_rhs_s2).  F: f((i - 1/2) h, n tau). */
void or_direct_s2(double gamma, uint64_t cells, uint64_t N, double h, double tau,
                  const double* F, const double* u0, double* U) {
    double mu, c;
    or_constants(OR_HYPER, gamma, tau, &mu, &c);
    double* g = (double*)malloc(sizeof(double) * N);
    or_weights(1.0 - gamma, N, g);
    double* R = (double*)malloc(sizeof(double) * (cells - 1) * N);
    or_rhs_s2(gamma, cells, N, tau, F, u0, R);
    double* history = (double*)malloc(sizeof(double) * (cells - 1));
    memset(U, 0, sizeof(double) * (cells - 1) * N);
    for (uint64_t n = 1; n <= N; ++n) {
        for (uint64_t i = 0; i + 1 < cells; ++i) history[i] = 0.0;
        for (uint64_t k = 1; k < n; ++k) {
            const double w = c * (g[n - k - 1] - g[n - k]);
            for (uint64_t i = 1; i < cells; ++i) history[i - 1] += w * U[(i - 1) * N + (k - 1)];
        }
        double u_left = 0.0, hist_left = 0.0;
        for (uint64_t i = 1; i < cells; ++i) {
            const double value = (R[(i - 1) * N + (n - 1)] + history[i - 1] + hist_left -
                                  (c * g[0] - 1.0 / h) * u_left) /
                                 (c * g[0] + 1.0 / h);
            U[(i - 1) * N + (n - 1)] = value;
            u_left = value;
            hist_left = history[i - 1];
        }
    }
    free(g);
    free(R);
    free(history);
}

/* ---- long-double restatements (same recurrences, 64-bit mantissa) -------- */

/* Generic: node-coupled BLTT time march in long double for a given fp64
 * column col[0..N) and RHS R (node-major), spatial operator
 *   kind 0: diagonal     col0 * x = r                      (ODE, cells-1 == 1)
 *   kind 1: tridiagonal  col0 x_i + off (x_{i-1}+x_{i+1})   (Scheme 4)
 *   kind 2: upwind       col0 x_i + off x_{i-1}             (Scheme 3, off=-1/h)
 *   kind 3: Scheme 2     col0 x_i + off x_{i-1}, off = -B~_0, history on x_i + x_{i-1}
 *                        (B~_j = -A~_j for j >= 1, schemes.cpp:162-165)
 * The history is summed in long double over all previous steps.  This is the
 * "exact" reference used for the corrected-mode Scheme 3 and to show the
 * reference's own fp64 rounding. */
void or_march_ld(int kind, uint64_t nodes, uint64_t N, const double* col, double off,
                 const double* R, double* U) {
    long double* X = (long double*)malloc(sizeof(long double) * nodes * N);
    long double* r = (long double*)malloc(sizeof(long double) * nodes);
    long double* cp = (long double*)malloc(sizeof(long double) * nodes);
    const long double d = col[0], o = off;
    for (uint64_t n = 0; n < N; ++n) {
        for (uint64_t i = 0; i < nodes; ++i) {
            long double acc = R[i * N + n];
            for (uint64_t k = 0; k < n; ++k)
                acc -= (long double)col[n - k] * (X[i * N + k] + (kind == 3 && i > 0 ? X[(i - 1) * N + k] : 0.0L));
            r[i] = acc;
        }
        if (kind == 0) {
            for (uint64_t i = 0; i < nodes; ++i) r[i] /= d;
        } else if (kind == 1) {
            long double den = d;
            cp[0] = o / den;
            r[0] /= den;
            for (uint64_t i = 1; i < nodes; ++i) {
                den = d - o * cp[i - 1];
                cp[i] = o / den;
                r[i] = (r[i] - o * r[i - 1]) / den;
            }
            for (uint64_t i = nodes - 1; i-- > 0;) r[i] -= cp[i] * r[i + 1];
        } else {
            long double left = 0.0L;
            for (uint64_t i = 0; i < nodes; ++i) {
                r[i] = (r[i] - o * left) / d;
                left = r[i];
            }
        }
        for (uint64_t i = 0; i < nodes; ++i) X[i * N + n] = r[i];
    }
    for (uint64_t i = 0; i < nodes * N; ++i) U[i] = (double)X[i];
    free(X);
    free(r);
    free(cp);
}

/* ---- seeded synthetic inputs (fixed generator) -------------- */

uint64_t or_splitmix64(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
double or_uniform(uint64_t* state) {
    return ((double)(or_splitmix64(state) >> 11) + 0.5) * 0x1.0p-53;
}
double or_normal(uint64_t* state) {
    const double u1 = or_uniform(state), u2 = or_uniform(state);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* Separable forcing grid  F[i][n] = sum_j a_j trig_j(k_j pi x_i) * t_n^{p_j}
 * (trig 0 = sin, 1 = cos, 2 = 1, 3 = x(1-x), 4 = 1-2x) with x_i = i*h (i = 1..cells-1) and
 * t_n = (n + t_shift) * tau, n = 1..N  -- the reference's evaluation points
 * (schemes.cpp:403-407 diffusion; :301-302 wave with t_shift = -1/2; Scheme 2
 * :184-186 with x_shift = -1/2, x = (i - 1/2) h). */
void or_forcing_modes(uint64_t cells, uint64_t N, double h, double tau, double x_shift, double t_shift,
                      int nmodes, const double* a, const double* k, const double* p,
                      const int* trig, double* F) {
    const double pi = 3.14159265358979323846;
    for (uint64_t i = 1; i < cells; ++i) {
        const double x = ((double)i + x_shift) * h;
        for (uint64_t n = 1; n <= N; ++n) {
            const double t = ((double)n + t_shift) * tau;
            double v = 0.0;
            for (int j = 0; j < nmodes; ++j) {
                const double sp = trig[j] == 0   ? sin(k[j] * pi * x)
                                  : trig[j] == 1 ? cos(k[j] * pi * x)
                                  : trig[j] == 3 ? x * (1.0 - x)
                                  : trig[j] == 4 ? (1.0 - 2.0 * x)
                                                 : 1.0;
                v += a[j] * sp * pow(t, p[j]);
            }
            F[(i - 1) * N + (n - 1)] = v;
        }
    }
}

/* u0 / phi samples amp * sin(pi x_i), i = 1..cells-1 */
void or_sine_grid(uint64_t cells, double h, double amp, double* out) {
    for (uint64_t i = 1; i < cells; ++i) out[i - 1] = amp * sin(3.14159265358979323846 * ((double)i * h));
}
