// fft.cuh -- batched fp64 complex FFT in shared memory (in-place radix-16/8/4/2
// passes, data staged through registers).  Forward = decimation in frequency
// (natural order in, digit-reversed order out); inverse = decimation in time
// (digit-reversed in, natural out).  Convolutions multiply spectra pointwise
// in the digit-reversed domain, so no reordering pass exists anywhere.  The
// kernel spectra are produced by the same forward routine, so their order
// matches by construction.
//
// Replaces the reference's radix-2 bit-reversal FFT (src/fft.cpp:50-79) as the
// arithmetic of the history product; see DESIGN.md for the pass plan.
#pragma once
#include "internal.cuh"

namespace ftb {

// Shared-memory index padding: one pad slot per 16 complex values keeps the
// radix-16 column reads of the last pass conflict-free.
__device__ __forceinline__ int sphys(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int spad_len(int n) { return n + (n >> 4) + 1; }

// cos(2*pi*k/16), k = 0..15 (compile-time k after unrolling)
__device__ __forceinline__ double c16(int k) {
    switch (k & 15) {
        case 0: return 1.0;
        case 1: case 15: return 0.92387953251128675613;
        case 2: case 14: return 0.70710678118654752440;
        case 3: case 13: return 0.38268343236508977173;
        case 4: case 12: return 0.0;
        case 5: case 11: return -0.38268343236508977173;
        case 6: case 10: return -0.70710678118654752440;
        case 7: case 9: return -0.92387953251128675613;
        default: return -1.0;
    }
}

// multiply by w_S^i = exp(-+2 pi i * i / S) for S | 16 (compile-time i, S)
template <int S, bool INV>
__device__ __forceinline__ cplx twc(cplx v, int i) {
    const int k = i * (16 / S);  // angle 2 pi k / 16, k in [0, 8)
    if (k == 0) return v;
    if (k == 4) return INV ? cplx{-v.y, v.x} : cplx{v.y, -v.x};
    const double c = c16(k);
    const double s = c16((k + 12) & 15);  // sin(2 pi k/16) = cos(2 pi (k-4)/16)
    // forward: (x + iy)(c - is);  inverse: (x + iy)(c + is)
    if (INV) return {fma(v.x, c, -v.y * s), fma(v.y, c, v.x * s)};
    return {fma(v.x, c, v.y * s), fma(v.y, c, -v.x * s)};
}

template <int R>
__device__ __forceinline__ constexpr int bitrev(int q) {
    int r = 0;
    for (int b = 1; b < R; b <<= 1) {
        r = (r << 1) | (q & 1);
        q >>= 1;
    }
    return r;
}

// In-register R-point DFT, natural order in and out.
template <int R, bool INV>
__device__ __forceinline__ void dft_reg(cplx (&v)[R]) {
#pragma unroll
    for (int s = R / 2; s >= 1; s >>= 1) {
#pragma unroll
        for (int b = 0; b < R; b += 2 * s) {
#pragma unroll
            for (int i = 0; i < s; ++i) {
                const cplx a = v[b + i], c = v[b + i + s];
                v[b + i] = cadd(a, c);
                const cplx d = csub(a, c);
                if (s == 1) v[b + i + s] = d;
                else if (s == 2) v[b + i + s] = twc<4, INV>(d, i);
                else if (s == 4) v[b + i + s] = twc<8, INV>(d, i);
                else v[b + i + s] = twc<16, INV>(d, i);
            }
        }
    }
    cplx t[R];
#pragma unroll
    for (int q = 0; q < R; ++q) t[q] = v[bitrev<R>(q)];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = t[q];
}

// Twiddles w_S^(j q), q = 1..R-1, from the multi-resolution table
// tw[S' + k] = exp(-2 pi i k / S') (every power-of-two S'): four coalesced loads
// (w_S^j, w_{S/2}^j = w_S^2j, w_{S/4}^j, w_{S/8}^j) and at most 11 products.
template <int R>
__device__ __forceinline__ void pass_twiddles(cplx (&w)[R], const cplx* __restrict__ tw, int S, int j) {
    w[0] = {1.0, 0.0};
#ifdef FT_TW_DIRECT
    // direct lookups w_S^{qj} = tw[S + qj] (qj < S): no product chain, exact table values
#pragma unroll
    for (int q = 1; q < R; ++q) w[q] = ldgc(&tw[S + q * j]);
#else
    if (R >= 2) w[1] = ldgc(&tw[S + j]);
    if (R >= 4) {
        w[2] = ldgc(&tw[(S >> 1) + j]);
        w[3] = cmul(w[1], w[2]);
    }
    if (R >= 8) {
        w[4] = ldgc(&tw[(S >> 2) + j]);
#pragma unroll
        for (int q = 5; q < 8; ++q) w[q] = cmul(w[4], w[q - 4]);
    }
    if (R >= 16) {
        w[8] = ldgc(&tw[(S >> 3) + j]);
#pragma unroll
        for (int q = 9; q < 16; ++q) w[q] = cmul(w[8], w[q - 8]);
    }
#endif
}

// R-point forward DFT (natural order in/out) of R/2 data points followed by R/2
// zeros: the first radix-2 stage degenerates to v[i+R/2] = v[i] w_R^i.
template <int R>
__device__ __forceinline__ void dft_reg_halfzero(cplx (&v)[R]) {
#pragma unroll
    for (int i = 0; i < R / 2; ++i) {
        if (R == 16) v[i + 8] = twc<16, false>(v[i], i);
        else if (R == 8) v[i + 4] = twc<8, false>(v[i], i);
        else if (R == 4) v[i + 2] = twc<4, false>(v[i], i);
        else v[i + 1] = v[i];
    }
#pragma unroll
    for (int s = R / 4; s >= 1; s >>= 1) {
#pragma unroll
        for (int b = 0; b < R; b += 2 * s) {
#pragma unroll
            for (int i = 0; i < s; ++i) {
                const cplx a = v[b + i], c = v[b + i + s];
                v[b + i] = cadd(a, c);
                const cplx d = csub(a, c);
                if (s == 1) v[b + i + s] = d;
                else if (s == 2) v[b + i + s] = twc<4, false>(d, i);
                else if (s == 4) v[b + i + s] = twc<8, false>(d, i);
                else v[b + i + s] = twc<16, false>(d, i);
            }
        }
    }
    cplx t[R];
#pragma unroll
    for (int q = 0; q < R; ++q) t[q] = v[bitrev<R>(q)];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = t[q];
}

// One in-place DIF pass over all sequences of `total` points, group size S.
template <int R>
__device__ __forceinline__ void fwd_pass(cplx* buf, int total, int S, const cplx* __restrict__ tw,
                                         int logT, int logS) {
    constexpr int LR = R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1;
    const int logQ = logS - LR;
    const int Q = 1 << logQ;
    const int tasks = total >> LR;
    for (int t = threadIdx.x; t < tasks; t += blockDim.x) {
        const int j = t & (Q - 1);
        const int base = ((t >> logQ) << logS) + j;
        cplx v[R];
#pragma unroll
        for (int p = 0; p < R; ++p) v[p] = buf[sphys(base + p * Q)];
        dft_reg<R, false>(v);
        if (Q > 1) {
            cplx w[R];
            pass_twiddles<R>(w, tw, S, j);
#pragma unroll
            for (int q = 1; q < R; ++q) v[q] = cmul(v[q], w[q]);
        }
#pragma unroll
        for (int q = 0; q < R; ++q) buf[sphys(base + q * Q)] = v[q];
    }
}

template <int R>
__device__ __forceinline__ void inv_pass(cplx* buf, int total, int S, const cplx* __restrict__ tw,
                                         int logT, int logS) {
    constexpr int LR = R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1;
    const int logQ = logS - LR;
    const int Q = 1 << logQ;
    const int tasks = total >> LR;
    for (int t = threadIdx.x; t < tasks; t += blockDim.x) {
        const int j = t & (Q - 1);
        const int base = ((t >> logQ) << logS) + j;
        cplx v[R];
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = buf[sphys(base + q * Q)];
        if (Q > 1) {
            cplx w[R];
            pass_twiddles<R>(w, tw, S, j);
#pragma unroll
            for (int q = 1; q < R; ++q) v[q] = cmulc(v[q], w[q]);
        }
        dft_reg<R, true>(v);
#pragma unroll
        for (int p = 0; p < R; ++p) buf[sphys(base + p * Q)] = v[p];
    }
}

// radix of the first (largest-S) pass for an m-point transform; the rest are 16
__device__ __forceinline__ int first_radix(int logm) {
    const int r = logm & 3;
    return r == 0 ? 16 : (1 << r);
}

// Forward transform of G sequences of m = 2^logm points (total = G*m) in buf.
// Caller synchronises before (data written) and after (data read).
__device__ __forceinline__ void fft_forward(cplx* buf, int total, int logm, const cplx* tw,
                                            int logT) {
    int logS = logm;
    bool first = true;
    while (logS > 0) {
        const int R = first ? first_radix(logm) : 16;
        const int S = 1 << logS;
        switch (R) {
            case 16: fwd_pass<16>(buf, total, S, tw, logT, logS); break;
            case 8: fwd_pass<8>(buf, total, S, tw, logT, logS); break;
            case 4: fwd_pass<4>(buf, total, S, tw, logT, logS); break;
            default: fwd_pass<2>(buf, total, S, tw, logT, logS); break;
        }
        __syncthreads();
        logS -= (R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1);
        first = false;
    }
}

__device__ __forceinline__ void fft_inverse(cplx* buf, int total, int logm, const cplx* tw,
                                            int logT) {
    // passes in reverse order: group sizes 16, 256, ... then the first-radix pass at S = m
    const int r0 = first_radix(logm);
    const int l0 = r0 == 16 ? 4 : r0 == 8 ? 3 : r0 == 4 ? 2 : 1;
    int logS = (logm - l0) == 0 ? logm : 4;
    while (true) {
        const bool last = (logS == logm);
        const int R = last ? r0 : 16;
        const int S = 1 << logS;
        switch (R) {
            case 16: inv_pass<16>(buf, total, S, tw, logT, logS); break;
            case 8: inv_pass<8>(buf, total, S, tw, logT, logS); break;
            case 4: inv_pass<4>(buf, total, S, tw, logT, logS); break;
            default: inv_pass<2>(buf, total, S, tw, logT, logS); break;
        }
        __syncthreads();
        if (last) break;
        logS = (logS + 4 <= logm - l0) ? logS + 4 : logm;
    }
}

// ---- compile-time specialised transforms (the history-product hot path) ----
// With the pass geometry known at compile time every shared-memory access of a
// butterfly is base + immediate offset, and twiddle indices are base + j.
__host__ __device__ constexpr int lg2c(int r) { return r == 16 ? 4 : r == 8 ? 3 : r == 4 ? 2 : 1; }
__host__ __device__ constexpr int first_radix_c(int logm) { return (logm & 3) == 0 ? 16 : (1 << (logm & 3)); }

template <int R, int LOGS, bool INV>
__device__ __forceinline__ void pass_c(cplx* buf, int total, const cplx* __restrict__ tw) {
    constexpr int LR = lg2c(R);
    constexpr int LOGQ = LOGS - LR;
    constexpr int Q = 1 << LOGQ;
    constexpr int S = 1 << LOGS;
    const int tasks = total >> LR;
    for (int t = threadIdx.x; t < tasks; t += blockDim.x) {
        const int j = t & (Q - 1);
        const int base = ((t >> LOGQ) << LOGS) + j;
        // physical index of base + p*Q: for Q >= 16 the padding term is linear in p
        const int pb = sphys(base);
        cplx v[R];
#pragma unroll
        for (int p = 0; p < R; ++p) {
            // phys(base + pQ) - phys(base) = pQ + (pQ >> 4) for every power-of-two Q
            // (base % 16 < Q when Q < 16; pQ % 16 == 0 when Q >= 16)
            const int off = p * Q + ((p * Q) >> 4);
            v[p] = buf[pb + off];
        }
        if (!INV) {
            dft_reg<R, false>(v);
            if (Q > 1) {
                cplx w[R];
                pass_twiddles<R>(w, tw, S, j);
#pragma unroll
                for (int q = 1; q < R; ++q) v[q] = cmul(v[q], w[q]);
            }
        } else {
            if (Q > 1) {
                cplx w[R];
                pass_twiddles<R>(w, tw, S, j);
#pragma unroll
                for (int q = 1; q < R; ++q) v[q] = cmulc(v[q], w[q]);
            }
            dft_reg<R, true>(v);
        }
#pragma unroll
        for (int p = 0; p < R; ++p) {
            const int off = p * Q + ((p * Q) >> 4);
            buf[pb + off] = v[p];
        }
    }
}

template <int LOGM, int LOGS, bool FIRST>
__device__ __forceinline__ void fwd_passes_c(cplx* buf, int total, const cplx* tw) {
    constexpr int R = FIRST ? first_radix_c(LOGM) : 16;
    pass_c<R, LOGS, false>(buf, total, tw);
    __syncthreads();
    if constexpr (LOGS - lg2c(R) > 0) fwd_passes_c<LOGM, LOGS - lg2c(R), false>(buf, total, tw);
}

// inverse: same passes in reverse order (smallest group first)
template <int LOGM, int LOGS, bool FIRST>
__device__ __forceinline__ void inv_passes_c(cplx* buf, int total, const cplx* tw) {
    constexpr int R = FIRST ? first_radix_c(LOGM) : 16;
    if constexpr (LOGS - lg2c(R) > 0) inv_passes_c<LOGM, LOGS - lg2c(R), false>(buf, total, tw);
    pass_c<R, LOGS, true>(buf, total, tw);
    __syncthreads();
}

template <int LOGM>
__device__ __forceinline__ void fft_forward_c(cplx* buf, int total, const cplx* tw) {
    fwd_passes_c<LOGM, LOGM, true>(buf, total, tw);
}
template <int LOGM>
__device__ __forceinline__ void fft_inverse_c(cplx* buf, int total, const cplx* tw) {
    inv_passes_c<LOGM, LOGM, true>(buf, total, tw);
}

}  // namespace ftb
