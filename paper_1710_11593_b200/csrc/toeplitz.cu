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

}  // namespace ftb
