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
#include <algorithm>

#include "internal.cuh"

namespace ftb {

// One CTA per problem; the step loop runs inside the kernel.
// The sequential spatial solve of step n for problem pb by one warp.  The chain
// runs redundantly on every lane in the reference's order (same operations,
// same rounding); each block of 32 nodes' operands is loaded coalesced one block
// ahead and broadcast by shuffles, so the chain waits only on its own latency.
__device__ __forceinline__ void dm_sweep(const DirectArgs& a, int pb, uint64_t n, int lane) {
    const int nodes = a.nodes;
    const uint64_t N = a.N;
    double* rhs = a.scratch + (uint64_t)pb * nodes;
    double* X = a.X + (uint64_t)pb * nodes * N;
    const ProblemConst pc = a.pc[pb];
    auto ld = [&](const double* p, int i) { return i < nodes ? __ldcg(p + i) : 0.0; };
    if (a.kind == SK_DIAG) {
        for (int i = lane; i < nodes; i += 32) X[(uint64_t)i * N + n] = __ldcg(rhs + i) / pc.d;
        return;
    }
    if (a.kind == SK_TRIDIAG) {
        const double* cp = a.cprime + (uint64_t)pb * nodes;
        const double* dn = a.den + (uint64_t)pb * nodes;
        const double off = -pc.off;
        double prev = 0.0;
        double r_cur = ld(rhs, lane), d_cur = ld(dn, lane);
        for (int i0 = 0; i0 < nodes; i0 += 32) {  // forward: rhs[i] = (rhs[i] - off rhs[i-1]) / den[i]
            const double r_nx = ld(rhs, i0 + 32 + lane), d_nx = ld(dn, i0 + 32 + lane);
            double mine = 0.0;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const double v = __shfl_sync(0xffffffffu, r_cur, k), d = __shfl_sync(0xffffffffu, d_cur, k);
                if (i0 + k < nodes) {
                    prev = i0 + k == 0 ? v / d : (v - off * prev) / d;
                    if (lane == k) mine = prev;
                }
            }
            if (i0 + lane < nodes) rhs[i0 + lane] = mine;
            r_cur = r_nx;
            d_cur = d_nx;
        }
        __syncwarp();
        // backward: rhs[i] -= cprime[i] rhs[i+1], i = nodes-2 .. 0 (rhs[nodes-1] is final)
        double next = prev;
        if (lane == 0) X[(uint64_t)(nodes - 1) * N + n] = next;
        const int top = nodes - 1;  // blocks of 32 below node top, descending
        auto ldb = [&](const double* p, int i) { return i >= 0 ? __ldcg(p + i) : 0.0; };
        double rb = ldb(rhs, top - 1 - lane), cb = ldb(cp, top - 1 - lane);
        for (int i0 = top - 1; i0 >= 0; i0 -= 32) {  // nodes i0, i0-1, ..., i0-31
            const double rn = ldb(rhs, i0 - 32 - lane), cn = ldb(cp, i0 - 32 - lane);
            double mine = 0.0;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const double v = __shfl_sync(0xffffffffu, rb, k), c = __shfl_sync(0xffffffffu, cb, k);
                if (i0 - k >= 0) {
                    next = v - c * next;
                    if (lane == k) mine = next;
                }
            }
            if (i0 - lane >= 0) X[(uint64_t)(i0 - lane) * N + n] = mine;
            rb = rn;
            cb = cn;
        }
        return;
    }
    // upwind marches (Scheme 3; Scheme 2 with the stencil history)
    const double* hs = a.scratch2 + (uint64_t)pb * nodes;
    double u_left = 0.0, hist_left = 0.0;
    double r_cur = ld(rhs, lane), h_cur = a.stencil ? ld(hs, lane) : 0.0;
    for (int i0 = 0; i0 < nodes; i0 += 32) {
        const double r_nx = ld(rhs, i0 + 32 + lane), h_nx = a.stencil ? ld(hs, i0 + 32 + lane) : 0.0;
        double mine = 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const double v = __shfl_sync(0xffffffffu, r_cur, k), hk = __shfl_sync(0xffffffffu, h_cur, k);
            if (i0 + k < nodes) {
                double value;
                if (a.stencil) {  // schemes.cpp:219-228 (pc.off = 1/h - c g0)
                    value = (v + hist_left + pc.off * u_left) / pc.d;
                    hist_left = hk;
                } else {          // schemes.cpp:345-351
                    value = (v + u_left / pc.h) / pc.d;
                }
                u_left = value;
                if (lane == k) mine = value;
            }
        }
        if (i0 + lane < nodes) X[(uint64_t)(i0 + lane) * N + n] = mine;
        r_cur = r_nx;
        h_cur = h_nx;
    }
}

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

// ---- multi-CTA reference-order march (the on-device oracle at scale) ----------
// Same arithmetic, same summation order as direct_kernel (bitwise equal), but the
// per-node history sums run on every SM: each CTA owns groups of 32 rows (one
// summing thread per row), the other warps stage the rows' solved prefixes
// X[row][k0, k0 + kDmChunk) through double-buffered shared memory with coalesced
// L2 loads (ld.global.cg: X is rewritten during the kernel, L1 could be stale).
// The sequential spatial sweep (Thomas / upwind / divide, schemes.cpp:453-461,
// :345-351) runs on extra warps of CTA 0 (dm_sweep, one warp per problem).  Steps are ordered by two monotonic
// global counters: `hist` (CTAs that published step n's right-hand sides) and
// `solved` (steps whose U the sweep has written).  For sums whose last term is
// U(n-1) (every kind but the wave scheme, which adds w[1] U(n-1) first) the CTAs
// form step n's partial sum over k < n-1 while the sweep is still solving step
// n-1, then add the last term: the same order, so still bitwise.
constexpr int kDmLoadWarps = 15;
constexpr int kDmThreads = 32 * (1 + kDmLoadWarps);  // history warps (+ kDmSweepWarps sweep warps, CTA 0 only)
constexpr int kDmSweepWarps = 4;                     // concurrent per-problem spatial sweeps (batched plans)
constexpr int kDmChunk = 256;                        // time steps per staged tile (64 KB in flight per CTA)
constexpr int kDmPitch = kDmChunk + 1;               // odd pitch: conflict-free column reads
constexpr int kDmMaxGroups = 64;                     // row groups of 32 per CTA

__device__ __forceinline__ unsigned dm_ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void dm_st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void dm_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * (1 + kDmLoadWarps)) : "memory"); }

__global__ void __launch_bounds__(kDmThreads + 32 * kDmSweepWarps) direct_multi_kernel(DirectArgs a, unsigned* ctr, int rows,
                                                                       int groups) {
    extern __shared__ double dm_smem[];  // [2][32][kDmPitch] staged tiles, [kDmMaxGroups][32] partials, [2][kDmChunk] weights
    double* part = dm_smem + 2 * 32 * kDmPitch;
    unsigned* hist_cnt = ctr;
    unsigned* solved = ctr + 1;
    const uint64_t N = a.N;
    const int nodes = a.nodes;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool pipelined = !(a.kind == SK_UPWIND && !a.stencil);
    if (warp > kDmLoadWarps) {  // ---- the sequential spatial sweeps (CTA 0; one warp per problem) ----
        if (blockIdx.x != 0) return;
        const int B = rows / nodes;
        const int sw = warp - 1 - kDmLoadWarps;
        for (uint64_t n = 0; n < N; ++n) {
            if (sw == 0 && lane == 0)
                while (dm_ld_acquire(hist_cnt) < (unsigned)(n + 1) * gridDim.x) __nanosleep(32);
            asm volatile("bar.sync 2, %0;" ::"n"(32 * kDmSweepWarps) : "memory");
            __threadfence();
            for (int pb = sw; pb < B; pb += kDmSweepWarps)
                dm_sweep(a, pb, n, lane);
            __threadfence();
            asm volatile("bar.sync 2, %0;" ::"n"(32 * kDmSweepWarps) : "memory");
            if (sw == 0 && lane == 0) dm_st_release(solved, (unsigned)(n + 1));
        }
        return;
    }
    // ---- history CTAs: groups g = blockIdx.x + j gridDim.x of 32 rows of one problem ----
    const int gpp = (nodes + 31) / 32;  // row groups per problem
    const int my_groups = groups > (int)blockIdx.x ? (groups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    double* wbuf = part + kDmMaxGroups * 32;  // [2][kDmChunk] weights w[n - k] of the staged chunk
    auto group_row = [&](int j, int r, int& pb) {  // global row of lane r of the CTA's j-th group (-1: none)
        const int g = (int)blockIdx.x + j * (int)gridDim.x;
        pb = g / gpp;
        const int i = (g % gpp) * 32 + r;
        return i < nodes ? pb * nodes + i : -1;
    };
    auto wait_solved = [&](unsigned target) {
        if (tid == 0)
            while (dm_ld_acquire(solved) < target) __nanosleep(64);
        dm_bar();
    };
    for (uint64_t n = 0; n < N; ++n) {
        // terms of the pre-sum: k in [0, kp); pipelined kinds leave k = n-1 for later
        const uint64_t kp = n >= 1 ? n - 1 : 0;
        wait_solved(pipelined ? (unsigned)kp : (unsigned)n);
        const int nch = (int)((kp + kDmChunk - 1) / kDmChunk);
        const int items = my_groups * nch;
        // item it = (group j, chunk c); loaders fill buf[it & 1] one item ahead of the summers
        auto load_item = [&](int it) {
            const int j = it / nch, c = it % nch;
            const uint64_t k0 = (uint64_t)c * kDmChunk;
            const int len = (int)(kp - k0 < (uint64_t)kDmChunk ? kp - k0 : (uint64_t)kDmChunk);
            double* buf = dm_smem + (it & 1) * 32 * kDmPitch;
            int pb = 0;
            for (int e = tid - 32; e < 32 * kDmChunk; e += 32 * kDmLoadWarps) {
                const int r = e / kDmChunk, q = e % kDmChunk;
                const int row = group_row(j, r, pb);
                if (row >= 0 && q < len) buf[r * kDmPitch + q] = __ldcg(a.X + (uint64_t)row * N + k0 + q);
            }
            group_row(j, 0, pb);
            const double* w = a.w + (uint64_t)pb * N;
            for (int q = tid - 32; q < len; q += 32 * kDmLoadWarps) wbuf[(it & 1) * kDmChunk + q] = __ldg(w + (n - k0 - q));
        };
        double acc = 0.0;  // summer lane's running sum (current group)
        if (warp >= 1 && items > 0) load_item(0);
        dm_bar();
        for (int it = 0; it < items; ++it) {
            if (warp >= 1) {
                if (it + 1 < items) load_item(it + 1);
            } else {
                const int j = it / nch, c = it % nch;
                int pb = 0;
                const int row = group_row(j, lane, pb);
                const uint64_t k0 = (uint64_t)c * kDmChunk;
                const int len = (int)(kp - k0 < (uint64_t)kDmChunk ? kp - k0 : (uint64_t)kDmChunk);
                const double* buf = dm_smem + (it & 1) * 32 * kDmPitch + lane * kDmPitch;
                const double* wv = wbuf + (it & 1) * kDmChunk;  // wv[q] = w[n - k0 - q]
                if (c == 0) acc = 0.0;
                if (row >= 0) {
                    const double* w = a.w + (uint64_t)pb * N;
                    if (a.kind == SK_DIAG && c == 0) acc = __ldcg(a.X + (uint64_t)row * N + n);
                    if (a.kind == SK_UPWIND && !a.stencil && c == 0) acc += w[1] * __ldcg(a.X + (uint64_t)row * N + n - 1);
                    // one dependent add per term in the reference's order; the smem operands of the
                    // next terms are independent and issued ahead (unrolled)
                    int q = 0;
                    if (a.kind == SK_DIAG) {
                        for (; q + 8 <= len; q += 8) {
#pragma unroll
                            for (int u = 0; u < 8; ++u) acc -= wv[q + u] * buf[q + u];
                        }
                        for (; q < len; ++q) acc -= wv[q] * buf[q];
                    } else {
                        for (; q + 8 <= len; q += 8) {
#pragma unroll
                            for (int u = 0; u < 8; ++u) acc += wv[q + u] * buf[q + u];
                        }
                        for (; q < len; ++q) acc += wv[q] * buf[q];
                    }
                }
                if (c == nch - 1) part[j * 32 + lane] = acc;
            }
            dm_bar();
        }
        // finish step n: (pipelined) the last term k = n-1 once the sweep has solved it
        if (pipelined) wait_solved((unsigned)n);
        if (warp == 0) {
            for (int j = 0; j < my_groups; ++j) {
                int pb = 0;
                const int row = group_row(j, lane, pb);
                if (row < 0) continue;
                const int i = row - pb * nodes;
                const double* xi = a.X + (uint64_t)row * N;
                const double* w = a.w + (uint64_t)pb * N;
                const ProblemConst& pc = a.pc[pb];
                double s = nch > 0 ? part[j * 32 + lane] : 0.0;
                double r;
                if (a.kind == SK_DIAG) {
                    if (nch == 0) s = __ldcg(xi + n);
                    if (n >= 1) s -= w[1] * __ldcg(xi + n - 1);
                    r = s;
                } else if (a.kind == SK_UPWIND && !a.stencil) {
                    if (nch == 0 && n >= 1) s += w[1] * __ldcg(xi + n - 1);
                    r = __ldcg(xi + n) - s;
                } else {
                    if (n >= 1) s += w[1] * __ldcg(xi + n - 1);
                    if (a.kind == SK_TRIDIAG) {
                        r = __ldcg(xi + n) + pc.c * s;
                    } else {  // Scheme 2 stencil
                        r = __ldcg(xi + n) + s;
                        a.scratch2[(uint64_t)pb * nodes + i] = s;
                    }
                }
                a.scratch[row] = r;
            }
        }
        dm_bar();
        if (tid == 0) {
            __threadfence();
            atomicAdd(hist_cnt, 1u);
        }
    }
}

size_t direct_multi_smem() { return sizeof(double) * (2 * 32 * kDmPitch + kDmMaxGroups * 32 + 2 * kDmChunk); }

cudaError_t launch_direct(const DirectArgs& a, int B, cudaStream_t st) {
    const int rows = B * a.nodes;
    static const bool single = getenv("FT_DIRECT_SINGLE") != nullptr;  // A/B: the one-CTA-per-problem march
    if (single || a.ctr == nullptr) {
        int threads = a.nodes < 1024 ? ((a.nodes + 31) / 32) * 32 : 1024;
        direct_kernel<<<B, threads, 0, st>>>(a);
        return cudaGetLastError();
    }
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = direct_multi_smem();
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(direct_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, direct_multi_kernel, kDmThreads + 32 * kDmSweepWarps, smem);
    if (e != cudaSuccess) return e;
    const int groups = B * ((a.nodes + 31) / 32);  // groups never straddle problems (one weight row each)
    int ctas = std::min(groups, sms * std::max(occ, 1));
    ctas = std::max(ctas, (groups + kDmMaxGroups - 1) / kDmMaxGroups);
    if (ctas > sms * occ) return cudaErrorInvalidConfiguration;  // more rows than the partial buffers hold
    e = cudaMemsetAsync(a.ctr, 0, 2 * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    DirectArgs aa = a;
    unsigned* ctr = a.ctr;
    int r = rows, g = groups;
    void* args[] = {&aa, &ctr, &r, &g};
    return cudaLaunchCooperativeKernel((const void*)direct_multi_kernel, dim3(ctas), dim3(kDmThreads + 32 * kDmSweepWarps), args,
                                       smem, st);
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
    static DeviceOnce set;
    if (set.first()) {
        cudaError_t e = cudaFuncSetAttribute(ode_whole_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOdeSmem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ode_whole_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOdeSmem);
        if (e != cudaSuccess) return e;
        set.done();
    }
    if (sc)
        ode_whole_kernel<true><<<B, kOdeThreads, smem, st>>>(X, R, col, pc, N);
    else
        ode_whole_kernel<false><<<B, kOdeThreads, smem, st>>>(X, R, col, pc, N);
    return cudaGetLastError();
}

}  // namespace ftb
