/* oracle.h -- CPU restatement of the reference direct path (TEST INFRASTRUCTURE
 * ONLY; see oracle.c header).  Scheme ids are oracle-local. */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_ODE = 0, OR_HYPER = 1, OR_WAVE = 2, OR_DIFFUSION = 3 };

double or_power_step(uint64_t k, double p);
void or_weights(double p, uint64_t count, double* out);
void or_constants(int scheme, double gamma, double tau, double* mu, double* c);
void or_col_s4(double gamma, uint64_t N, double h, double tau, double* col);
void or_col_s2(double gamma, uint64_t N, double h, double tau, double* a, double* b);
void or_rhs_s2(double gamma, uint64_t cells, uint64_t N, double tau, const double* F,
               const double* u0, double* R);
void or_direct_s2(double gamma, uint64_t cells, uint64_t N, double h, double tau,
                  const double* F, const double* u0, double* U);
void or_col_s3(double gamma, uint64_t N, double h, double tau, double* col);
void or_col_ode(double gamma, uint64_t N, double tau, double* col);
void or_rhs_s4(double gamma, uint64_t cells, uint64_t N, double tau, const double* F,
               const double* u0, double* R);
void or_rhs_s3(double gamma, uint64_t cells, uint64_t N, double tau, const double* F,
               const double* u0, const double* phi, int mode, double* R);
void or_rhs_ode(double gamma, uint64_t N, double tau, const double* F, double u0, double* R);
int or_forward_solve(const double* col, const double* b, uint64_t n, double* x);
void or_toeplitz_matvec(const double* col, const double* row, uint64_t n, const double* x, double* y);
void or_block_matvec(const double* col, const double* row, uint64_t n, uint64_t m, double beta, const double* x,
                     double* y);
void or_direct_s4(double gamma, uint64_t cells, uint64_t N, double h, double tau,
                  const double* F, const double* u0, double* U);
void or_direct_s3(double gamma, uint64_t cells, uint64_t N, double h, double tau,
                  const double* F, const double* u0, const double* phi, int rhs_mode, double* U);
void or_march_ld(int kind, uint64_t nodes, uint64_t N, const double* col, double off,
                 const double* R, double* U);
uint64_t or_splitmix64(uint64_t* state);
double or_uniform(uint64_t* state);
double or_normal(uint64_t* state);
void or_forcing_modes(uint64_t cells, uint64_t N, double h, double tau, double x_shift, double t_shift,
                      int nmodes, const double* a, const double* k, const double* p,
                      const int* trig, double* F);
void or_sine_grid(uint64_t cells, double h, double amp, double* out);

#ifdef __cplusplus
}
#endif
