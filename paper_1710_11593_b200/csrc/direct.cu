// direct.cu -- the "direct" entry point on the GPU: time marching in the
// reference's summation order (compiled with --fmad=false so every product
// and sum rounds exactly as the reference's x86-64 build does), plus device
// generation of separable right-hand sides.
//
//   Scheme 4 direct : src/schemes.cpp:434-463  (history :447-449, Thomas :453-461)
//   Scheme 3 direct : src/schemes.cpp:333-352  (history :336-343, upwind march :345-351)
//   Scheme 2 direct : src/schemes.cpp:210-232  (history :212-218, upwind march :219-228)
//   ODE direct      : src/toeplitz.cpp:169-186 (lower_toeplitz_forward_solve)
//   RHS             : src/schemes.cpp:401-408 (Scheme 4), :300-306 (Scheme3Rhs)
#include "internal.cuh"

namespace ftb {

// One CTA per problem; the step loop runs inside the kernel.
__global__ void __launch_bounds__(1024) direct_kernel(DirectArgs a) {
    const int pb = blockIdx.x;
    const uint64_t N = a.N;
    const int nodes = a.nodes;
    double* X = a.X + (uint64_t)pb * nodes * N;
    const double* w = a.w + (uint64_t)pb * N;
    double* rhs = a.scratch + (uint64_t)pb * nodes;
    const ProblemConst pc = a.pc[pb];
    for (uint64_t n = 0; n < N; ++n) {
        for (int i = threadIdx.x; i < nodes; i += blockDim.x) {
            const double* xi = X + (uint64_t)i * N;
            if (a.kind == SK_TRIDIAG) {
                // hist = sum_{k=1}^{n-1} (g[n-k-1] - g[n-k]) U(i,k)  (1-based n, k)
                double hist = 0.0;
                for (uint64_t k = 0; k < n; ++k) hist += w[n - k] * xi[k];
                rhs[i] = xi[n] + pc.c * hist;
            } else if (a.kind == SK_UPWIND && a.stencil) {
                // Scheme 2 (schemes.cpp:212-218): history += w * U(i,k), w = c (g[j-1] - g[j])
                double hist = 0.0;
                for (uint64_t k = 0; k < n; ++k) hist += w[n - k] * xi[k];
                rhs[i] = xi[n] + hist;
                a.scratch2[(uint64_t)pb * nodes + i] = hist;
            } else if (a.kind == SK_UPWIND) {
                double hist = 0.0;
                if (n >= 1) {
                    hist += w[1] * xi[n - 1];
                    for (uint64_t k = 0; k + 1 < n; ++k) hist += w[n - k] * xi[k];
                }
                rhs[i] = xi[n] - hist;
            } else {
                double acc = xi[n];
                for (uint64_t k = 0; k < n; ++k) acc -= w[n - k] * xi[k];
                rhs[i] = acc;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const double* cp = a.cprime + (uint64_t)pb * nodes;
            const double* dn = a.den + (uint64_t)pb * nodes;
            if (a.kind == SK_TRIDIAG) {
                const double off = -pc.off;
                rhs[0] /= dn[0];
                for (int i = 1; i < nodes; ++i) rhs[i] = (rhs[i] - off * rhs[i - 1]) / dn[i];
                for (int i = nodes - 1; i-- > 0;) rhs[i] -= cp[i] * rhs[i + 1];
            } else if (a.kind == SK_UPWIND && a.stencil) {
                // schemes.cpp:219-228: (rhs + hist_i + hist_left - (c g0 - 1/h) u_left) / (c g0 + 1/h);
                // pc.off = 1/h - c g0, so  - (c g0 - 1/h) u_left == + off u_left exactly
                const double* hs = a.scratch2 + (uint64_t)pb * nodes;
                double u_left = 0.0, hist_left = 0.0;
                for (int i = 0; i < nodes; ++i) {
                    const double value = (rhs[i] + hist_left + pc.off * u_left) / pc.d;
                    hist_left = hs[i];
                    rhs[i] = value;
                    u_left = value;
                }
            } else if (a.kind == SK_UPWIND) {
                double u_left = 0.0;
                for (int i = 0; i < nodes; ++i) {
                    const double value = (rhs[i] + u_left / pc.h) / pc.d;
                    rhs[i] = value;
                    u_left = value;
                }
            } else {
                for (int i = 0; i < nodes; ++i) rhs[i] = rhs[i] / pc.d;
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nodes; i += blockDim.x) X[(uint64_t)i * N + n] = rhs[i];
        __syncthreads();
    }
}

cudaError_t launch_direct(const DirectArgs& a, int B, cudaStream_t st) {
    int threads = a.nodes < 1024 ? ((a.nodes + 31) / 32) * 32 : 1024;
    direct_kernel<<<B, threads, 0, st>>>(a);
    return cudaGetLastError();
}

// ---- device RHS generation (separable forcing) -------------------------------
__global__ void rhs_modes_kernel(RhsModesArgs a) {
    const uint64_t total = (uint64_t)a.B * a.nodes * a.N;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t n0 = idx % a.N;
        const uint64_t row = idx / a.N;
        const int pb = (int)(row / a.nodes);
        const int i = a.node_begin + (int)(row % a.nodes) + 1;
        const double x = a.scheme == 0 ? 0.0 : a.scheme == 1 ? ((double)i - 0.5) * a.h : (double)i * a.h;
        const double n = (double)(n0 + 1);
        const double t = a.scheme == 2 ? (n - 0.5) * a.tau : n * a.tau;
        double f = 0.0;
        for (int j = 0; j < a.nmodes; ++j) {
            const int tg = a.trig[j];
            const double sp = tg == 0   ? sin(a.k[j] * 3.14159265358979323846 * x)
                              : tg == 1 ? cos(a.k[j] * 3.14159265358979323846 * x)
                              : tg == 3 ? x * (1.0 - x)
                              : tg == 4 ? (1.0 - 2.0 * x)
                                        : 1.0;
            f += a.a[pb * a.nmodes + j] * sp * pow(t, a.p[pb * a.nmodes + j]);
        }
        const double* wv = a.wts + (uint64_t)pb * (a.N + 1);
        const double c = a.cvals[pb];
        const double u0 = a.u0amp ? a.u0amp[pb] * (a.scheme == 0 ? 1.0 : sin(3.14159265358979323846 * x)) : 0.0;
        double v;
        if (a.scheme == 1) {  // Scheme2Rhs: c g_(n-1) (u0(x_i) + u0(x_(i-1)))
            const double amp = a.u0amp ? a.u0amp[pb] : 0.0;
            const double us = amp * sin(3.14159265358979323846 * ((double)i * a.h)) +
                              amp * sin(3.14159265358979323846 * ((double)(i - 1) * a.h));
            v = f + c * wv[n0] * us;
        } else if (a.scheme == 2) {
            const double phi = a.phiamp ? a.phiamp[pb] * sin(3.14159265358979323846 * x) : 0.0;
            v = f + c * a.tau * wv[n0] * phi;
            if (n0 >= 1) v -= c * (wv[n0 - 1] - wv[n0]) * u0;
            else if (a.rhs_mode == 1) v += c * wv[0] * u0;
        } else {
            v = f + c * wv[n0] * u0;
        }
        a.R[idx] = v;
    }
}

// Separable factors of the same right-hand side for the fused path
// (ft_solve_fast_modes): R[row][n] = sum_j A[row][j] T[b][n][j], with the terms
// in rhs_modes_kernel's order (modes, then phi (wave), then u0) and the same
// rounded products, so the leaf's sum reproduces rhs_modes_kernel's value.
int gen_terms(const RhsModesArgs& a) {
    return a.nmodes + (a.scheme == 2 && a.phiamp ? 1 : 0) + (a.u0amp ? 1 : 0);
}

__global__ void gen_tables_kernel(RhsModesArgs a, double* A, double* T, int J) {
    const double pi = 3.14159265358979323846;
    const uint64_t rows = (uint64_t)a.B * a.nodes;
    const uint64_t nA = rows, nT = (uint64_t)a.B * a.N;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < nA + nT;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        if (idx < nA) {  // node factors
            const uint64_t row = idx;
            const int pb = (int)(row / a.nodes);
            const int i = a.node_begin + (int)(row % a.nodes) + 1;
            const double x = a.scheme == 0 ? 0.0 : a.scheme == 1 ? ((double)i - 0.5) * a.h : (double)i * a.h;
            double* Ar = A + row * J;
            int j = 0;
            for (; j < a.nmodes; ++j) {
                const int tg = a.trig[j];
                const double sp = tg == 0   ? sin(a.k[j] * pi * x)
                                  : tg == 1 ? cos(a.k[j] * pi * x)
                                  : tg == 3 ? x * (1.0 - x)
                                  : tg == 4 ? (1.0 - 2.0 * x)
                                            : 1.0;
                Ar[j] = a.a[pb * a.nmodes + j] * sp;
            }
            const double xi = a.scheme == 0 ? 0.0 : (double)i * a.h;
            if (a.scheme == 2 && a.phiamp) Ar[j++] = a.phiamp[pb] * sin(pi * xi);
            if (a.u0amp) {
                if (a.scheme == 1)
                    Ar[j++] = a.u0amp[pb] * sin(pi * ((double)i * a.h)) + a.u0amp[pb] * sin(pi * ((double)(i - 1) * a.h));
                else
                    Ar[j++] = a.u0amp[pb] * (a.scheme == 0 ? 1.0 : sin(pi * xi));
            }
        } else {  // step factors
            const uint64_t e = idx - nA;
            const int pb = (int)(e / a.N);
            const uint64_t n0 = e % a.N;
            const double n = (double)(n0 + 1);
            const double t = a.scheme == 2 ? (n - 0.5) * a.tau : n * a.tau;
            const double* wv = a.wts + (uint64_t)pb * (a.N + 1);
            const double c = a.cvals[pb];
            double* Tr = T + e * J;
            int j = 0;
            for (; j < a.nmodes; ++j) Tr[j] = pow(t, a.p[pb * a.nmodes + j]);
            if (a.scheme == 2) {
                if (a.phiamp) Tr[j++] = c * a.tau * wv[n0];
                if (a.u0amp)  // v -= c (M_(n-2) - M_(n-1)) u0 for n >= 2; corrected mode adds c M_0 u0 at n = 1
                    Tr[j++] = n0 >= 1 ? -(c * (wv[n0 - 1] - wv[n0])) : (a.rhs_mode == 1 ? c * wv[0] : 0.0);
            } else if (a.u0amp) {
                Tr[j++] = c * wv[n0];
            }
        }
    }
}

cudaError_t launch_gen_tables(const RhsModesArgs& a, double* A, double* T, cudaStream_t st) {
    gen_tables_kernel<<<148 * 4, 256, 0, st>>>(a, A, T, gen_terms(a));
    return cudaGetLastError();
}

cudaError_t launch_rhs_modes(const RhsModesArgs& a, cudaStream_t st) {
    rhs_modes_kernel<<<148 * 8, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace ftb

namespace ftb {

// ---- whole fast solve of single-node (ODE) problems: one CTA per problem ----
// u[n] = (r[n] - sum_{j<n} col[n-j] u[j]) / col[0]  (the reference's one-sided ODE
// march, fractional_ode.cpp via SURVEY 8a; same equations as the D&C leaf with
// nodes = 1).  Such a problem is one time row: the D&C's ~2N/32 launches are pure
// latency, so the CTA keeps the solved prefix of u in shared memory and walks
// 32-step blocks: while warp 0 solves block b (its 32 dependent steps by
// shuffles), 12 warps form block b+1's history sum_{j<t0} col[t0+32+k-j] u[j]
// over the steps solved before block b (register-blocked Toeplitz products).
#ifndef FT_ODE_NOHIST
#define FT_ODE_NOHIST 0  // timing probes only (wrong results)
#endif
#ifndef FT_ODE_NOSEQ
#define FT_ODE_NOSEQ 0
#endif
#ifndef FT_ODE_DIV
#define FT_ODE_DIV 0
#endif
constexpr int kOdeSets = 3;                       // history warp sets (4 warps each: 8 outputs per warp)
constexpr int kOdeThreads = 32 * (1 + 4 * kOdeSets);
#ifndef FT_ODE_CHAINS
#define FT_ODE_CHAINS 8
#endif
constexpr int kOdeChains = FT_ODE_CHAINS;  // independent partial sums per lane (loads in flight)

template <bool SC>  // SC: the column is staged in shared memory too (16 N bytes fit)
__global__ void __launch_bounds__(kOdeThreads, 1) ode_whole_kernel(double* X, const double* R, const double* col,
                                                                   const ProblemConst* pcs, uint64_t N) {
    extern __shared__ __align__(16) double s_u[];  // [N] solved steps, then (SC) [N] column
    double* s_col = s_u + N;
    __shared__ double s_hp[2][kOdeSets][32];       // next block's history, per warp set (double-buffered)
    __shared__ double s_c[64];                     // col[0..64)
    const int pb = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const double* c = col + (uint64_t)pb * N;
    const double* r = R + (uint64_t)pb * N;
    double* x = X + (uint64_t)pb * N;
    const double d = pcs[pb].d, dinv = 1.0 / d;
    (void)d;
    (void)dinv;
    if (tid < 64) s_c[tid] = (uint64_t)tid < N ? c[tid] : 0.0;
    double rnext = lane < N ? r[lane] : 0.0;  // (warp 0: block 0's R)
    for (int i = tid; i < kOdeSets * 32; i += blockDim.x) (&s_hp[0][0][0])[i] = 0.0;
    if (SC)
        for (uint64_t i = tid; i < N; i += blockDim.x) s_col[i] = __ldg(c + i);
    auto colv = [&](uint64_t i) { return SC ? s_col[i] : __ldg(c + i); };
    __syncthreads();
    const uint64_t nb = (N + 31) / 32;
    for (uint64_t b = 0; b < nb; ++b) {
        const uint64_t t0 = b * 32;
        const int len = (int)(N - t0 < 32 ? N - t0 : 32);
        const int cur = (int)(b & 1);
        if (w == 0) {
            // block b: its history over steps < t0 - 32 is in s_hp[cur]; add the previous
            // block's 32 steps (u just solved) here, then the 32 dependent steps
            const double rcur = rnext;
            if (t0 + 32 + lane < N) rnext = r[t0 + 32 + lane];  // next block's R: in flight during this one
            double hk = 0.0;
#pragma unroll
            for (int q = 0; q < kOdeSets; ++q) hk += s_hp[cur][q][lane];
            double rk = lane < len ? rcur - hk : 0.0;
            if (b > 0 && lane < len) {
                const uint64_t p0 = t0 - 32;
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[j & 3] = fma(s_c[32 + lane - j], s_u[p0 + j], acc[j & 3]);
                rk -= (acc[0] + acc[1]) + (acc[2] + acc[3]);
            }
            double ux = 0.0;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                if (i >= len || FT_ODE_NOSEQ) break;
#if FT_ODE_DIV
                const double xi = __shfl_sync(0xffffffffu, rk, i) / d;
#else
                const double xi = __shfl_sync(0xffffffffu, rk, i) * dinv;  // (a division is ~10x the latency)
#endif
                if (lane == i) ux = xi;
                if (lane > i) rk = fma(-s_c[lane - i], xi, rk);
            }
            if (lane < len) {
                s_u[t0 + lane] = ux;
                x[t0 + lane] = ux;
            }
        } else if (b + 1 < nb && !FT_ODE_NOHIST) {
            // next block's history over steps < t0 (all solved before this block):
            // warp (set, g) covers outputs k in [8g, 8g+8); each lane a slice of the
            // j range, with a sliding column window (8 FMA per 2 loads), then a
            // reduction over the warp's slices; warp 0 adds the kOdeSets partials
            const int hw = w - 1, g = hw & 3, set = hw >> 2;
            const int sl = set * 32 + lane;
            constexpr int NS = kOdeSets * 32;
            const uint64_t per = ((t0 + NS - 1) / NS) | 1;  // odd slice stride: spread over the banks
            const uint64_t j0 = min(t0, (uint64_t)sl * per), j1 = min(t0, j0 + per);
            const uint64_t kb = t0 + 32 + 8 * g;  // column index of output 8g at step j is kb - j
            double acc[8], cw[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                acc[i] = 0.0;
                cw[i] = (j0 < j1 && kb + i - j0 < N) ? colv(kb + i - j0) : 0.0;
            }
            for (uint64_t j = j0; j < j1; ++j) {
                const double uj = s_u[j];
                const uint64_t nx = kb - j - 1;  // next step's window entry 0 (>= 32)
                const double cn = nx < N ? colv(nx) : 0.0;
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] = fma(cw[i], uj, acc[i]);
#pragma unroll
                for (int i = 7; i > 0; --i) cw[i] = cw[i - 1];
                cw[0] = cn;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
            double v = acc[0];
#pragma unroll
            for (int i = 1; i < 8; ++i) v = lane == i ? acc[i] : v;
            if (lane < 8) s_hp[cur ^ 1][set][8 * g + lane] = v;
        }
        __syncthreads();
    }
}

constexpr uint64_t kOdeSmem = 200 * 1024;
bool ode_whole_ok(uint64_t N) { return N >= 1 && N * sizeof(double) <= kOdeSmem; }

cudaError_t launch_ode_whole(double* X, const double* R, const double* col, const ProblemConst* pc, uint64_t N,
                             int B, cudaStream_t st) {
    const bool sc = 2 * N * sizeof(double) <= kOdeSmem;
    const size_t smem = (sc ? 2 : 1) * N * sizeof(double);
    static bool set = false;
    if (!set) {
        cudaError_t e = cudaFuncSetAttribute(ode_whole_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOdeSmem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ode_whole_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOdeSmem);
        if (e != cudaSuccess) return e;
        set = true;
    }
    if (sc)
        ode_whole_kernel<true><<<B, kOdeThreads, smem, st>>>(X, R, col, pc, N);
    else
        ode_whole_kernel<false><<<B, kOdeThreads, smem, st>>>(X, R, col, pc, N);
    return cudaGetLastError();
}

}  // namespace ftb
