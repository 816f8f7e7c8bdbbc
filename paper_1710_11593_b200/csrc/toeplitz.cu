// toeplitz.cu -- the reference's structured-operator API on the GPU:
//   toeplitz_matvec (src/toeplitz.cpp:98-115, with embed_circulant :84-96) and
//   block_matvec    (src/toeplitz.cpp:150-167)
// as batched direct products.  The reference applies an n x n Toeplitz matrix
// through a length-L >= 2n FFT circulant embedding (rounding ~ eps ||T|| ||x||);
// on B200 the direct product is cheap (n^2 FMA per vector, ~1 ms at n = 65536)
// and exact up to fp64 summation, so it needs no spectra and no setup.
//
//   y[b][i] = sum_j t(i - j) x[b][j]   (+ beta (x[b-1][i] + x[b+1][i]) in block mode)
//   t(d) = first_col[d] (d > 0), first_row[-d] (d <= 0)
//
// One CTA computes 1024 consecutive outputs of one vector (4 per thread); the
// inputs stream through SMEM in chunks of 256 together with the 1279-entry
// diagonal window those outputs need.
#include <algorithm>

#include "internal.cuh"

namespace ftb {

constexpr int kTmThreads = 256;
constexpr int kTmOut = 4 * kTmThreads;   // outputs per CTA
constexpr int kTmChunk = 256;            // inputs per SMEM chunk

__global__ void __launch_bounds__(kTmThreads) toeplitz_matvec_kernel(const double* __restrict__ col,
                                                                     const double* __restrict__ row, uint64_t n,
                                                                     const double* __restrict__ x, double* __restrict__ y,
                                                                     double beta, int block_mode, uint64_t vectors) {
    __shared__ double s_x[kTmChunk];
    __shared__ double s_t[kTmOut + kTmChunk];  // t(d) for d in [I0 - J0 - (kTmChunk-1), I0 - J0 + kTmOut - 1]
    const uint64_t I0 = (uint64_t)blockIdx.x * kTmOut;
    const int tid = threadIdx.x;
    for (uint64_t b = blockIdx.y; b < vectors; b += gridDim.y) {
    const double* xb = x + b * n;
    const int r0 = 4 * tid;  // this thread's outputs I0 + r0 + r, r < 4
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint64_t J0 = 0; J0 < n; J0 += kTmChunk) {
        __syncthreads();
        {
            const uint64_t j = J0 + tid;
            s_x[tid] = j < n ? xb[j] : 0.0;
        }
        // window: s_t[w] = t(dlo + w), dlo = I0 - J0 - (kTmChunk - 1)
        const int64_t dlo = (int64_t)I0 - (int64_t)J0 - (kTmChunk - 1);
        for (int w = tid; w < kTmOut + kTmChunk; w += kTmThreads) {
            const int64_t d = dlo + w;
            double v = 0.0;
            if (d > 0 && (uint64_t)d < n) v = col[d];
            else if (d <= 0 && (uint64_t)(-d) < n) v = row[-d];
            s_t[w] = v;
        }
        __syncthreads();
        // d(i, j) = I0 + r0 + r - J0 - jj  ->  window index r0 + r - jj + (kTmChunk - 1)
#pragma unroll 4
        for (int jj = 0; jj < kTmChunk; ++jj) {
            const double xv = s_x[jj];
            const int w = r0 - jj + (kTmChunk - 1);
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[r] = fma(s_t[w + r], xv, acc[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint64_t i = I0 + r0 + r;
        if (i >= n) continue;
        double v = acc[r];
        if (block_mode) {  // block_matvec (toeplitz.cpp:158-165): left neighbour, then right
            if (b > 0) v += beta * x[(b - 1) * n + i];
            if (b + 1 < vectors) v += beta * x[(b + 1) * n + i];
        }
        y[b * n + i] = v;
    }
    }
}

cudaError_t launch_toeplitz_matvec(const double* col, const double* row, uint64_t n, const double* x, double* y,
                                   double beta, int block_mode, uint64_t vectors, cudaStream_t st) {
    const dim3 grid((unsigned)((n + kTmOut - 1) / kTmOut), (unsigned)(vectors < 65535 ? vectors : 65535));
    toeplitz_matvec_kernel<<<grid, kTmThreads, 0, st>>>(col, row, n, x, y, beta, block_mode, vectors);
    return cudaGetLastError();
}

// ---- the plan's own block system matrix applied through its history products (ft_apply) ----
// After the far history (every D&C product of the schedule, run with the source x and the
// target y = -sum) this kernel adds what the products do not cover: the in-leaf lags
// (t - j < L inside the leaf that holds step t, including the diagonal) and the spatial
// stencil of the step operator,
//   TRIDIAG: d x_i - b (x_(i-1) + x_(i+1)) = (d - 2b) x_i - b ((x_(i-1) - x_i) + (x_(i+1) - x_i))
//   UPWIND : d x_i - s x_(i-1)            = (d - s) x_i - s (x_(i-1) - x_i)
// in the difference form: d - 2b (d - s) is an exact fp64 subtraction (Sterbenz) and the
// neighbour differences carry the rounding error of b |x_(i+1) - x_i| instead of b |x_i|,
// which keeps the residual of a smooth solution meaningful on kappa ~ 1e8 operators.
// One thread per (row, step); a warp reads 32 consecutive steps of a row.
template <int L>
__global__ void __launch_bounds__(256) apply_near_kernel(const double* __restrict__ x, double* __restrict__ y,
                                                         uint64_t N, int nodes, uint64_t rows,
                                                         const ProblemConst* __restrict__ pc,
                                                         const double* __restrict__ col, int kind) {
    __shared__ double s_x[8][L];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t tiles_t = (N + L - 1) / L;
    for (uint64_t tile = (uint64_t)blockIdx.x * 8 + w; tile < rows * tiles_t; tile += (uint64_t)gridDim.x * 8) {
        const uint64_t r = tile / tiles_t, t0 = (tile - r * tiles_t) * L;
        const uint64_t t = t0 + lane;
        const int pb = (int)(r / nodes), i = (int)(r - (uint64_t)pb * nodes);
        const bool ok = t < N;
        const double xv = ok ? x[r * N + t] : 0.0;
        __syncwarp();
        s_x[w][lane] = xv;
        __syncwarp();
        const double* c = col + (uint64_t)pb * N;
        double acc = 0.0;  // lags 1 .. lane inside the leaf, oldest first
        for (int j = 0; j < lane; ++j) acc = fma(c[lane - j], s_x[w][j], acc);
        const ProblemConst k = pc[pb];
        double sp;
        if (kind == SK_TRIDIAG) {
            const double xl = (ok && i > 0) ? x[(r - 1) * N + t] : 0.0;
            const double xr = (ok && i + 1 < nodes) ? x[(r + 1) * N + t] : 0.0;
            sp = fma(k.d - 2.0 * k.off, xv, -k.off * ((xl - xv) + (xr - xv)));
        } else if (kind == SK_UPWIND) {
            const double xl = (ok && i > 0) ? x[(r - 1) * N + t] : 0.0;
            sp = fma(k.d - k.off, xv, -k.off * (xl - xv));
        } else {
            sp = k.d * xv;
        }
        if (ok) y[r * N + t] = (acc - y[r * N + t]) + sp;
    }
}

cudaError_t launch_apply_near(const double* x, double* y, uint64_t N, int nodes, uint64_t rows,
                              const ProblemConst* pc, const double* col, int kind, int L, cudaStream_t st) {
    if (L != 32) return cudaErrorInvalidValue;
    const uint64_t tiles = rows * ((N + 31) / 32);
    const unsigned grid = (unsigned)std::min<uint64_t>((tiles + 7) / 8, 148ull * 64);
    apply_near_kernel<32><<<grid, 256, 0, st>>>(x, y, N, nodes, rows, pc, col, kind);
    return cudaGetLastError();
}

// max |y - r| and max |r| over n values (ft_residual): out[0], out[1] as ordered uint64 bit patterns
__global__ void __launch_bounds__(256) resid_max_kernel(const double* __restrict__ y, const double* __restrict__ r,
                                                        uint64_t n, unsigned long long* out) {
    double d = 0.0, m = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double rv = r[i];
        const double dv = fabs(y[i] - rv);
        d = dv > d || dv != dv ? dv : d;  // a NaN sticks
        m = fmax(m, fabs(rv));
    }
    for (int o = 16; o; o >>= 1) {
        const double d2 = __shfl_xor_sync(0xffffffffu, d, o);
        d = (d2 > d || d2 != d2) ? d2 : d;
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    if ((threadIdx.x & 31) == 0) {
        // non-negative doubles order like their bit patterns; NaN (all exponent bits) sorts above inf
        atomicMax(&out[0], (unsigned long long)__double_as_longlong(d));
        atomicMax(&out[1], (unsigned long long)__double_as_longlong(m));
    }
}

cudaError_t launch_resid_max(const double* y, const double* r, uint64_t n, unsigned long long* out, cudaStream_t st) {
    resid_max_kernel<<<148 * 8, 256, 0, st>>>(y, r, n, out);
    return cudaGetLastError();
}

}  // namespace ftb
