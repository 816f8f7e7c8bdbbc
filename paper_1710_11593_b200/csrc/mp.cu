// mp.cu -- the history product ("middle product") of the time-axis
// divide-and-conquer, as a batched fp64 FFT convolution, plus the per-level
// kernel spectra it multiplies by.
//
// For a D&C block [lo, hi) of n = 2h steps with midpoint mid = lo + h:
//     R[row][t] -= sum_{lo <= j < mid} col[t - j] * U[row][j],   t in [mid, hi)
// The length-n cyclic convolution of the zero-padded source block with the
// column is exact for these outputs.  It is split by the CRT
//     x^n - 1 = prod_b (x^m - zeta_b),   zeta_b = exp(2 pi i b / K),  m = n / K
// into K independent twisted length-m cyclic convolutions ("branches"), one
// per CTA of a K-CTA thread-block cluster; the inverse K-point DFT across
// branches is done through distributed shared memory.  Two real rows are
// packed into one complex sequence.  Lags < J (the near field) are removed
// from the spectra and summed exactly (SURVEY.md 0.6 / probe P7).
//
// Replaces: reference toeplitz_matvec (src/toeplitz.cpp:98-115) +
// embed_circulant (:84-96) + fft::transform (src/fft.cpp:50-79) as used by
// the GMRES fast paths (src/schemes.cpp:464-474, :353-369).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "fft.cuh"
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace ftb {

__device__ __forceinline__ cplx conjc(cplx a) { return {a.x, -a.y}; }

struct PairInfo {
    uint64_t row1;  // first row of the packed pair
    int pb;         // problem index
    int has2;       // second row exists
};

template <int LOGN>
struct Plan1 {
    static constexpr int n = 1 << LOGN;
    static constexpr int h = n / 2;
    static constexpr int RL = (LOGN & 3) == 0 ? 16 : (1 << (LOGN & 3));  // last (fused) radix
    static constexpr int Q0 = n / 16;                                     // first pass stride
};

template <int LOGS, int LOGN>
__device__ __forceinline__ void mid_fwd(cplx* buf, int total, const cplx* tw) {
    // forward passes with S from LOGS down to (but excluding) the fused last one
    if constexpr (LOGS > lg2c(Plan1<LOGN>::RL)) {
        pass_c<16, LOGS, false>(buf, total, tw);
        __syncthreads();
        mid_fwd<LOGS - 4, LOGN>(buf, total, tw);
    }
}
template <int LOGS, int LOGN>
__device__ __forceinline__ void mid_inv(cplx* buf, int total, const cplx* tw) {
    if constexpr (LOGS > lg2c(Plan1<LOGN>::RL)) {
        mid_inv<LOGS - 4, LOGN>(buf, total, tw);
        pass_c<16, LOGS, true>(buf, total, tw);
        __syncthreads();
    }
}

// SPLIT = true: no cluster; CTA (b, pair) writes its branch result to
// a.scratch and mpB_kernel performs the cross-branch combine (K >= 4 levels:
// 16-CTA clusters packed badly -- 14 active clusters -- and stalled on
// cluster barriers, ncu).
template <int K, int LOGM, bool SPLIT, bool FOLDED = false>
__global__ void __launch_bounds__(kMpThreads, 2) mp_kernel(MpArgs a) {
    pdl_launch_dependents(a.pdl_trigger);
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* buf = reinterpret_cast<cplx*>(smem_raw);
    __shared__ PairInfo s_pair[kMpTile / 32];
    const int b = SPLIT ? (int)blockIdx.x : (int)cg::this_cluster().block_rank();
    constexpr int m = 1 << LOGM, logm = LOGM;
    const int G = a.G, n = a.n;
    const int total = G * m;
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    const int pair0 = (SPLIT ? a.pair_begin : 0) + blockIdx.y * G;
    const uint64_t N = a.N;

    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        const int rp = min(pair0 + g, npairs - 1);
        const int pb = rp / a.pairs_per_problem, lp = rp - pb * a.pairs_per_problem;
        const int i1 = 2 * lp;
        s_pair[g] = {(uint64_t)(pb * a.nodes + i1), pb, (pair0 + g < npairs && i1 + 1 < a.nodes) ? 1 : 0};
    }
    // branch twist factors zeta_b^q = exp(2 pi i b q / K)
    cplx zeta[K / 2];
#pragma unroll
    for (int q = 0; q < K / 2; ++q) zeta[q] = conjc(ldgc(&a.tw[K + ((b * q) & (K - 1))]));
    __syncthreads();

    // 1+2a. fold the (zero-padded) source block into branch b, twist, and run the
    //    first forward pass (S = m, radix 16) straight from HBM: task (g, j) owns
    //    the branch points r = j + p m/16, p < 16, i.e. K/2 chunk loads per point.
    static_assert(LOGM >= 8, "cluster branches are at least 256 points");
    constexpr int Q0 = m / 16;
    // theta_b^(p Q0) = exp(2 pi i b p / (16 K)) for the 16 rows of a task
    __shared__ cplx s_tq[16];
    if (threadIdx.x < 16) s_tq[threadIdx.x] = conjc(ldgc(&a.tw[n + ((b * (int)threadIdx.x * Q0) & (n - 1))]));
    __syncthreads();
    for (int t = threadIdx.x; t < total / 16; t += blockDim.x) {
        const int g = t / Q0, j = t - g * Q0;
        const PairInfo pi = s_pair[g];
        const double* x1 = a.U + pi.row1 * N + a.lo + j;
        const bool live = pair0 + g < npairs;
        cplx v[16];
        if constexpr (FOLDED) {
            // branch input already folded + twisted by mp_fold_kernel (in place in scratch)
            const cplx* in = a.scratch + ((uint64_t)(pair0 + g - a.pair_begin) * K + b) * m + j;
#pragma unroll
            for (int p = 0; p < 16; ++p) v[p] = ldgc(&in[(uint64_t)p * Q0]);
        } else {
#pragma unroll
        for (int p = 0; p < 16; ++p) v[p] = {0.0, 0.0};
#pragma unroll
        for (int q = 0; q < K / 2; ++q) {
            double u1[16], u2[16];
#pragma unroll
            for (int p = 0; p < 16; ++p) {
                const uint64_t o = (uint64_t)q * m + (uint64_t)p * Q0;
                u1[p] = live ? x1[o] : 0.0;
                u2[p] = (live && pi.has2) ? x1[N + o] : 0.0;
            }
#pragma unroll
            for (int p = 0; p < 16; ++p) v[p] = q == 0 ? cplx{u1[p], u2[p]} : cadd(v[p], cmul(cplx{u1[p], u2[p]}, zeta[q]));
        }
        if (b) {
            const cplx tj = conjc(ldgc(&a.tw[n + b * j]));  // theta_b^j
#pragma unroll
            for (int p = 0; p < 16; ++p) v[p] = cmul(v[p], cmul(tj, s_tq[p]));
        }
        }
        dft_reg<16, false>(v);
        cplx w[16];
        pass_twiddles<16>(w, a.tw, m, j);
#pragma unroll
        for (int q = 1; q < 16; ++q) v[q] = cmul(v[q], w[q]);
        const int pbx = sphys(g * m + j);
#pragma unroll
        for (int q = 0; q < 16; ++q) buf[pbx + q * (Q0 + (Q0 >> 4))] = v[q];
    }
    __syncthreads();
    mid_fwd<LOGM - 4, LOGM>(buf, total, a.tw);

    // 2b. fused: last forward pass (twiddle-free), branch spectrum, first inverse pass
    {
        constexpr int RL = Plan1<LOGM>::RL;
        for (int t = threadIdx.x; t < total / RL; t += blockDim.x) {
            const int base = t * RL;
            const int g = base >> LOGM;
            const int pbx = sphys(base);
            cplx v[RL];
#pragma unroll
            for (int p = 0; p < RL; ++p) v[p] = buf[pbx + p];
            dft_reg<RL, false>(v);
            const cplx* sp = a.spec + ((uint64_t)s_pair[g].pb * K + b) * m + (base & (m - 1));
#pragma unroll
            for (int p = 0; p < RL; ++p) v[p] = cmul(v[p], ldgc(&sp[p]));
            dft_reg<RL, true>(v);
#pragma unroll
            for (int p = 0; p < RL; ++p) buf[pbx + p] = v[p];
        }
    }
    __syncthreads();
    mid_inv<LOGM - 4, LOGM>(buf, total, a.tw);
    pass_c<16, LOGM, true>(buf, total, a.tw);  // last inverse pass (S = m) -> SMEM for the combine
    if constexpr (SPLIT) {
        cplx* out = a.scratch + ((uint64_t)(pair0 - a.pair_begin) * K + b) * m;
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) out[idx] = buf[sphys(idx)];
        return;
    } else {
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();

    // 3. inverse K-point DFT across the cluster's branches (DSMEM), near field, store.
    //    Item (g, r): read the K branch values once, untwist by w_n^(bb r), then a
    //    K-point DFT gives every output q in [K/2, K) of this r.
    constexpr int logK = K == 2 ? 1 : K == 4 ? 2 : K == 8 ? 3 : 4;
    const int logslice = logm - logK;
    const uint64_t tend = a.hi < N ? a.hi : N;
    const int work = total >> logK;  // G * slice
    const cplx* rb[K];
#pragma unroll
    for (int bb = 0; bb < K; ++bb) rb[bb] = cluster.map_shared_rank(buf, bb);
    constexpr int CH2 = K >= 8 ? 1 : 8 / K;
    for (int base = threadIdx.x; base < work; base += CH2 * kMpThreads) {
        // prefetch the targets' current right-hand sides for every output of the chunk
        double r1[CH2][K / 2], r2[CH2][K / 2];
#pragma unroll
        for (int c = 0; c < CH2; ++c) {
            const int idx = base + c * kMpThreads;
            const int rr = idx & ((1 << logslice) - 1);
            const int g = min(idx, work - 1) >> logslice;
            const int r = (b << logslice) + rr;
            const PairInfo pi = s_pair[g];
            const bool ok = idx < work && pair0 + g < npairs;
#pragma unroll
            for (int q = 0; q < K / 2; ++q) {
                const uint64_t t = a.mid + (uint64_t)q * m + r;
                const bool okt = ok && t < tend;
                r1[c][q] = (okt && a.rsrc) ? a.rsrc[pi.row1 * N + t] : 0.0;
                r2[c][q] = (okt && pi.has2 && a.rsrc) ? a.rsrc[(pi.row1 + 1) * N + t] : 0.0;
            }
        }
#pragma unroll
        for (int c = 0; c < CH2; ++c) {
            const int idx = base + c * kMpThreads;
            if (idx >= work) break;
            const int rr = idx & ((1 << logslice) - 1);
            const int g = idx >> logslice;
            const int r = (b << logslice) + rr;
            if (pair0 + g >= npairs) continue;
            cplx wv[K];
#pragma unroll
            for (int bb = 0; bb < K; ++bb) wv[bb] = rb[bb][sphys((g << logm) + r)];
            if (K > 2) {
                const cplx w1 = ldgc(&a.tw[n + r]);  // w_n^r
                cplx wp = w1;
#pragma unroll
                for (int bb = 1; bb < K; ++bb) {
                    wv[bb] = cmul(wv[bb], wp);
                    if (bb + 1 < K) wp = cmul(wp, w1);
                }
                dft_reg<K, false>(wv);  // wv[q] = sum_bb w_bb w_n^(bb r) w_K^(bb q)
            } else {
                const cplx t = cmul(wv[1], ldgc(&a.tw[n + r]));
                wv[1] = csub(wv[0], t);  // q = 1: w_2^1 = -1
            }
            const PairInfo pi = s_pair[g];
            const uint64_t row1 = pi.row1;
#pragma unroll
            for (int q = K / 2; q < K; ++q) {
                const uint64_t t = a.mid + (uint64_t)(q - K / 2) * m + r;
                if (t >= tend) continue;
                cplx y = wv[q];
                const int tp = (int)(t - a.mid);
                if (tp < a.J - 1) {  // exact near field: lags t - j < J
                    const double* cp = a.col + (uint64_t)pi.pb * N;
                    const double* x1 = a.U + row1 * N;
                    const uint64_t jlo = (t >= a.lo + (uint64_t)(a.J - 1)) ? t - (uint64_t)(a.J - 1) : a.lo;
                    double s1 = 0.0, s2 = 0.0;
                    for (uint64_t j = a.mid; j-- > jlo;) {
                        const double cv = cp[t - j];
                        s1 = fma(cv, x1[j], s1);
                        if (pi.has2) s2 = fma(cv, x1[N + j], s2);
                    }
                    y.x += s1;
                    y.y += s2;
                }
                a.X[row1 * N + t] = r1[c][q - K / 2] - y.x;
                if (pi.has2) a.X[(row1 + 1) * N + t] = r2[c][q - K / 2] - y.y;
            }
        }
    }
    cluster.sync();
    }
}

// Pre-fold of the split K-branch levels (four-step first pass): thread <->
// (pair, r), r < m.  Reads the K/2 source chunks x_q = U[lo + q m + r] of the
// packed row pair once, forms every branch's input
//     f_b(r) = theta_b^r sum_q x_q zeta_b^q,  zeta_b = e^(2 pi i b / K),  theta_b = e^(2 pi i b / n)
// with one K-point DFT (upper half of the inputs is the zero padding), and
// writes f_b to scratch[pair][b][r]; mp_kernel<.., FOLDED> then reads its
// branch straight from there instead of re-reading and folding the whole
// source block in every branch CTA (K-fold L2 traffic and K/2 complex MACs
// per point, ncu).
template <int K, int LOGM>
__global__ void __launch_bounds__(kMpThreads) mp_fold_kernel(MpArgs a) {
    pdl_launch_dependents(a.pdl_trigger);
    pdl_wait();
    constexpr int m = 1 << LOGM;
    const int n = a.n;
    const int pl = blockIdx.y;
    const int rp = a.pair_begin + pl;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    if (rp >= npairs || r >= m) return;
    const uint64_t N = a.N;
    const int pb = rp / a.pairs_per_problem, lp = rp - pb * a.pairs_per_problem;
    const int i1 = 2 * lp;
    const bool has2 = i1 + 1 < a.nodes;
    const uint64_t row1 = (uint64_t)(pb * a.nodes + i1);
    const double* x1 = a.U + row1 * N + a.lo + r;
    cplx v[K];
#pragma unroll
    for (int q = 0; q < K / 2; ++q) {
        v[q].x = x1[(uint64_t)q * m];
        v[q].y = has2 ? x1[N + (uint64_t)q * m] : 0.0;
    }
#pragma unroll
    for (int q = K / 2; q < K; ++q) v[q] = {0.0, 0.0};
    dft_reg<K, true>(v);  // v[b] = sum_q x_q e^(+2 pi i b q / K)
    cplx* out = a.scratch + (uint64_t)pl * K * m + r;
    out[0] = v[0];
#pragma unroll
    for (int bb = 1; bb < K; ++bb) out[(uint64_t)bb * m] = cmulc(v[bb], ldgc(&a.tw[n + bb * r]));
    // (the persistent split kernel forms these twists from 4 coalesced loads, pass_twiddles)
}

// Cross-branch combine of the split K-branch levels: thread <-> (pair, r):
// read the K branch values, untwist by w_n^(b r), K-point DFT, store the K/2
// target outputs t = mid + (q - K/2) m + r (plus the exact near field).
template <int K, int LOGM>
__global__ void __launch_bounds__(kMpThreads) mpB_kernel(MpArgs a) {
    pdl_launch_dependents(a.pdl_trigger);
    pdl_wait();
    constexpr int m = 1 << LOGM;
    const int n = a.n;
    const int pl = blockIdx.y;  // pair within the batch
    const int rp = a.pair_begin + pl;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    if (rp >= npairs || r >= m) return;
    const uint64_t N = a.N;
    const int pb = rp / a.pairs_per_problem, lp = rp - pb * a.pairs_per_problem;
    const int i1 = 2 * lp;
    const bool has2 = i1 + 1 < a.nodes;
    const uint64_t row1 = (uint64_t)(pb * a.nodes + i1);
    const uint64_t tend = a.hi < N ? a.hi : N;
    double r1[K / 2], r2[K / 2];
#pragma unroll
    for (int q = 0; q < K / 2; ++q) {
        const uint64_t t = a.mid + (uint64_t)q * m + r;
        r1[q] = (t < tend && a.rsrc) ? a.rsrc[row1 * N + t] : 0.0;
        r2[q] = (t < tend && has2 && a.rsrc) ? a.rsrc[(row1 + 1) * N + t] : 0.0;
    }
    const cplx* in = a.scratch + (uint64_t)pl * K * m + r;
    cplx wv[K];
#pragma unroll
    for (int bb = 0; bb < K; ++bb) wv[bb] = in[(uint64_t)bb * m];
    const cplx w1 = ldgc(&a.tw[n + r]);  // w_n^r
    cplx wp = w1;
#pragma unroll
    for (int bb = 1; bb < K; ++bb) {
        wv[bb] = cmul(wv[bb], wp);
        if (bb + 1 < K) wp = cmul(wp, w1);
    }
    dft_reg<K, false>(wv);
#pragma unroll
    for (int q = K / 2; q < K; ++q) {
        const uint64_t t = a.mid + (uint64_t)(q - K / 2) * m + r;
        if (t >= tend) continue;
        cplx y = wv[q];
        const int tp = (int)(t - a.mid);
        if (tp < a.J - 1) {
            const double* cp = a.col + (uint64_t)pb * N;
            const double* x1 = a.U + row1 * N;
            const uint64_t jlo = (t >= a.lo + (uint64_t)(a.J - 1)) ? t - (uint64_t)(a.J - 1) : a.lo;
            double s1 = 0.0, s2 = 0.0;
            for (uint64_t j = a.mid; j-- > jlo;) {
                const double cv = cp[t - j];
                s1 = fma(cv, x1[j], s1);
                if (has2) s2 = fma(cv, x1[N + j], s2);
            }
            y.x += s1;
            y.y += s2;
        }
        a.X[row1 * N + t] = r1[q - K / 2] - y.x;
        if (has2) a.X[(row1 + 1) * N + t] = r2[q - K / 2] - y.y;
    }
}

// ---- persistent split K-branch levels (n = 32768, 65536) ----------------------
// The three passes of a split level (fold, K branch transforms, combine) as ONE
// persistent kernel fed by a task queue, per row pair instead of per batch: task
// group g = { fold(g), branch(g - D, 0..K-1), combine(g - 2D) }.  A pair's folded
// branch inputs / branch results live in ring slot p % RS of the scratch (RS >=
// 2D + 1 pairs, ~50 MB: L2-resident, so the round trip no longer goes to HBM),
// and every task waits (one thread, acquire loads) only for the tasks it reads:
// branch(p, .) for fold(p); combine(p) for all K branches; fold(p) for the
// combine that last used its slot.  Memory-bound folds / combines and the
// FP64-bound branch FFTs of different pairs run side by side on every SM
// instead of as separate full-GPU launches.  Scratch reads use ld.global.cg
// (slots are rewritten during the kernel); the source and target streams are
// marked evict-first (ld/st.global.cs) so they do not push the ring out of L2.
struct SplitQ {
    unsigned* ctr;  // [0] task counter; [1, 1+RS) folds done, [1+RS, 1+2RS) branches done,
                    // [1+2RS, 1+3RS) combines done -- per slot, cumulative over the slot's uses
    int RS, D, npairs, ntasks;
    int probe;  // timing probes (wrong results): bit 0 skips branch work, bit 1 fold / combine work;
                // bit 2 (A/B, results unchanged) keeps the ring lines instead of discarding them
};

__device__ __forceinline__ void spq_wait(const unsigned* c, unsigned target) {
    if (threadIdx.x == 0) {
        unsigned v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
            if (v >= target) break;
            __nanosleep(64);
        }
    }
    __syncthreads();
}
__device__ __forceinline__ void spq_signal_add(unsigned* c) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(c, 1u);
    }
}
__device__ __forceinline__ cplx ldcgc(const cplx* p) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    return {v.x, v.y};
}

#ifndef FT_SPLIT_PARTS
#define FT_SPLIT_PARTS 4
#endif
constexpr int kSplitParts = FT_SPLIT_PARTS;  // fold / combine tasks per pair (m / 4 points each; 2 and 8 measured
                                // the same or slower, as were smem-staged cp.async variants)  // fold / combine tasks per pair (m / 4 points each: shorter tasks)

template <int K, int LOGM>
__global__ void __launch_bounds__(kMpThreads, 2) mp_split_kernel(MpArgs a, SplitQ q) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* buf = reinterpret_cast<cplx*>(smem_raw);
    __shared__ int s_task;
    constexpr int m = 1 << LOGM;
    constexpr int Q0 = m / 16;
    const int n = a.n;
    const uint64_t N = a.N;
    const int RS = q.RS;
    unsigned* fold_done = q.ctr + 1;
    unsigned* br_done = q.ctr + 1 + RS;
    unsigned* comb_done = q.ctr + 1 + 2 * RS;
    const uint64_t tend = a.hi < N ? a.hi : N;
    for (;;) {
        __syncthreads();  // previous task's shared state is dead
        if (threadIdx.x == 0) s_task = (int)atomicAdd(q.ctr, 1u);
        __syncthreads();
        const int task = s_task;
        if (task >= q.ntasks) return;
        constexpr int NS = kSplitParts, GT = NS + K + NS;  // tasks per group
        const int g = task / GT, r = task - g * GT;
        const int p = r < NS ? g : r < NS + K ? g - q.D : g - 2 * q.D;
        if (p < 0 || p >= q.npairs) continue;
        const int slot = p % RS;
        const unsigned use = (unsigned)(p / RS);
        cplx* sc = a.scratch + (uint64_t)slot * K * m;
        const int pb = p / a.pairs_per_problem, lp = p - pb * a.pairs_per_problem;
        const int i1 = 2 * lp;
        const bool has2 = i1 + 1 < a.nodes;
        const uint64_t row1 = (uint64_t)(pb * a.nodes + i1);
        if (r < NS) {
            // ---- fold(p, part): f_b(rr) = theta_b^rr sum_q x_q(rr) zeta_b^q (mp_fold_kernel) ----
            spq_wait(comb_done + slot, use * NS);  // the slot's previous pair is fully combined
            const double* x1 = a.U + row1 * N + a.lo;
#pragma unroll 1
            for (int rr = r * (m / NS) + threadIdx.x; rr < (r + 1) * (m / NS) && !(q.probe & 2); rr += blockDim.x) {
                cplx v[K];
#pragma unroll
                for (int qq = 0; qq < K / 2; ++qq) {
                    v[qq].x = __ldcs(x1 + (uint64_t)qq * m + rr);
                    v[qq].y = has2 ? __ldcs(x1 + N + (uint64_t)qq * m + rr) : 0.0;
                }
#pragma unroll
                for (int qq = K / 2; qq < K; ++qq) v[qq] = {0.0, 0.0};
                dft_reg<K, true>(v);
                // twists theta_b^rr = w_n^(b rr), b < K: 4 coalesced table loads + products
                // (pass_twiddles) instead of K-1 loads at stride b rr (uncoalesced, ncu)
                cplx tw[K];
                pass_twiddles<K>(tw, a.tw, n, rr);
                cplx* out = sc + rr;
                out[0] = v[0];
#pragma unroll
                for (int bb = 1; bb < K; ++bb) out[(uint64_t)bb * m] = cmulc(v[bb], tw[bb]);
            }
            spq_signal_add(fold_done + slot);
        } else if (r < NS + K) {
            // ---- branch(p, b): m-point transform, branch spectrum, inverse (mp_kernel<.., FOLDED>) ----
            const int b = r - NS;
            spq_wait(fold_done + slot, (use + 1u) * NS);
            const cplx* in = sc + (uint64_t)b * m;  // folded and twisted by fold(p)
            if (q.probe & 1) {  // timing probe: no branch work
                spq_signal_add(br_done + slot);
                continue;
            }
            for (int t = threadIdx.x; t < m / 16; t += blockDim.x) {
                const int j = t;
                cplx v[16];
#pragma unroll
                for (int pp = 0; pp < 16; ++pp) v[pp] = ldcgc(&in[j + pp * Q0]);
                dft_reg<16, false>(v);
                cplx w[16];
                pass_twiddles<16>(w, a.tw, m, j);
#pragma unroll
                for (int qq = 1; qq < 16; ++qq) v[qq] = cmul(v[qq], w[qq]);
                const int pbx = sphys(j);
#pragma unroll
                for (int qq = 0; qq < 16; ++qq) buf[pbx + qq * (Q0 + (Q0 >> 4))] = v[qq];
            }
            __syncthreads();
            mid_fwd<LOGM - 4, LOGM>(buf, m, a.tw);
            {
                constexpr int RL = Plan1<LOGM>::RL;
                for (int t = threadIdx.x; t < m / RL; t += blockDim.x) {
                    const int base = t * RL;
                    const int pbx = sphys(base);
                    cplx v[RL];
#pragma unroll
                    for (int pp = 0; pp < RL; ++pp) v[pp] = buf[pbx + pp];
                    dft_reg<RL, false>(v);
                    const cplx* sp = a.spec + ((uint64_t)pb * K + b) * m + base;
#pragma unroll
                    for (int pp = 0; pp < RL; ++pp) v[pp] = cmul(v[pp], ldgc(&sp[pp]));
                    dft_reg<RL, true>(v);
#pragma unroll
                    for (int pp = 0; pp < RL; ++pp) buf[pbx + pp] = v[pp];
                }
            }
            __syncthreads();
            mid_inv<LOGM - 4, LOGM>(buf, m, a.tw);
            pass_c<16, LOGM, true>(buf, m, a.tw);
            __syncthreads();
            cplx* out = sc + (uint64_t)b * m;
            for (int idx = threadIdx.x; idx < m; idx += blockDim.x) out[idx] = buf[sphys(idx)];
            spq_signal_add(br_done + slot);
        } else {
            // ---- combine(p, part): untwist, K-point DFT, the K/2 target outputs (mpB_kernel) ----
            const int part = r - NS - K;
            spq_wait(br_done + slot, (use + 1u) * K);
#pragma unroll 1
            for (int rr = part * (m / NS) + threadIdx.x; rr < (part + 1) * (m / NS) && !(q.probe & 2); rr += blockDim.x) {
                double r1[K / 2], r2[K / 2];
#pragma unroll
                for (int qq = 0; qq < K / 2; ++qq) {
                    const uint64_t t = a.mid + (uint64_t)qq * m + rr;
                    r1[qq] = (t < tend && a.rsrc) ? __ldcs(a.rsrc + row1 * N + t) : 0.0;
                    r2[qq] = (t < tend && has2 && a.rsrc) ? __ldcs(a.rsrc + (row1 + 1) * N + t) : 0.0;
                }
                cplx wv[K];
#pragma unroll
                for (int bb = 0; bb < K; ++bb) wv[bb] = ldcgc(&sc[(uint64_t)bb * m + rr]);
                cplx tw[K];  // untwists w_n^(b rr): 4 coalesced loads + products, shallow dependency chain
                pass_twiddles<K>(tw, a.tw, n, rr);
#pragma unroll
                for (int bb = 1; bb < K; ++bb) wv[bb] = cmul(wv[bb], tw[bb]);
                dft_reg<K, false>(wv);
                // the slot's branch results are dead once read: drop their L2 lines without the
                // write-back (otherwise every ring write eventually costs a DRAM write, ncu)
                __syncwarp();
                if ((rr & 7) == 0 && !(q.probe & 4)) {
#pragma unroll
                    for (int bb = 0; bb < K; ++bb)
                        asm volatile("discard.global.L2 [%0], 128;" ::"l"(&sc[(uint64_t)bb * m + rr]) : "memory");
                }
#pragma unroll
                for (int qq = K / 2; qq < K; ++qq) {
                    const uint64_t t = a.mid + (uint64_t)(qq - K / 2) * m + rr;
                    if (t >= tend) continue;
                    cplx y = wv[qq];
                    const int tp = (int)(t - a.mid);
                    if (tp < a.J - 1) {
                        const double* cp = a.col + (uint64_t)pb * N;
                        const double* x1 = a.U + row1 * N;
                        const uint64_t jlo = (t >= a.lo + (uint64_t)(a.J - 1)) ? t - (uint64_t)(a.J - 1) : a.lo;
                        double s1 = 0.0, s2 = 0.0;
                        for (uint64_t j = a.mid; j-- > jlo;) {
                            const double cv = cp[t - j];
                            s1 = fma(cv, x1[j], s1);
                            if (has2) s2 = fma(cv, x1[N + j], s2);
                        }
                        y.x += s1;
                        y.y += s2;
                    }
                    __stcs(a.X + row1 * N + t, r1[qq - K / 2] - y.x);
                    if (has2) __stcs(a.X + (row1 + 1) * N + t, r2[qq - K / 2] - y.y);
                }
            }
            spq_signal_add(comb_done + slot);
        }
    }
}

// ---- single-CTA n-point FFT history product (512 <= n <= 8192) -------------
// One CTA transforms G row pairs of n = 2^LOGN points (the zero-padded source
// block).  Passes (radix 16 from S = n down, remainder radix last):
//   * first forward pass reads U straight from HBM (the upper half is zero and
//     pruned), writes SMEM;
//   * last forward pass + spectrum multiply + first inverse pass are fused in
//     registers (one SMEM round trip instead of three);
//   * last inverse pass computes only the needed half (t in [mid, hi)) and
//     writes R := R - y straight to HBM.
// The spectrum (spec1_kernel) uses the same pass plan, so digit-reversed
// orders agree.
// Mid passes, each preceded by its barrier, so callers can issue the next
// phase's global loads (spectrum, twiddles, targets) before the final barrier.
template <int LOGS, int LOGN>
__device__ __forceinline__ void mid_fwd_s(cplx* buf, int total, const cplx* tw) {
    if constexpr (LOGS > lg2c(Plan1<LOGN>::RL)) {
        __syncthreads();
        pass_c<16, LOGS, false>(buf, total, tw);
        mid_fwd_s<LOGS - 4, LOGN>(buf, total, tw);
    }
}
template <int LOGS, int LOGN>
__device__ __forceinline__ void mid_inv_s(cplx* buf, int total, const cplx* tw) {
    if constexpr (LOGS > lg2c(Plan1<LOGN>::RL)) {
        mid_inv_s<LOGS - 4, LOGN>(buf, total, tw);
        __syncthreads();
        pass_c<16, LOGS, true>(buf, total, tw);
    }
}

// Last inverse pass (S = n, radix 16) inputs of task t: twiddles and the
// targets' right-hand sides (outputs p >= 8 are the targets [mid, mid + h)).
template <int Q0>
__device__ __forceinline__ void mp1_last_prefetch(const MpArgs& a, const PairInfo* s_pair, int pair0, int npairs,
                                                  int t, cplx (&w)[16], double (&r1)[8], double (&r2)[8]) {
    const int g = t / Q0, j = t - g * Q0;
    const PairInfo pi = s_pair[g];
    const bool live = pair0 + g < npairs;
    const uint64_t tend = a.hi < a.N ? a.hi : a.N;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        const uint64_t tt = a.mid + j + (uint64_t)p * Q0;
        const bool ok = live && tt < tend;
        r1[p] = (ok && a.rsrc) ? a.rsrc[pi.row1 * a.N + tt] : 0.0;
        r2[p] = (ok && pi.has2 && a.rsrc) ? a.rsrc[(pi.row1 + 1) * a.N + tt] : 0.0;
    }
    pass_twiddles<16>(w, a.tw, Q0 * 16, j);
}

template <int Q0>
__device__ __forceinline__ void mp1_last_task(const MpArgs& a, cplx* buf, const PairInfo* s_pair, int pair0,
                                              int npairs, int t, const cplx (&w)[16], const double (&r1)[8],
                                              const double (&r2)[8]) {
    constexpr int n = Q0 * 16;
    const int g = t / Q0, j = t - g * Q0;
    const PairInfo pi = s_pair[g];
    const uint64_t N = a.N;
    const uint64_t tend = a.hi < N ? a.hi : N;
    const int pbx = sphys(g * n + j);
    cplx v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = buf[pbx + q * (Q0 + (Q0 >> 4))];
#pragma unroll
    for (int q = 1; q < 16; ++q) v[q] = cmulc(v[q], w[q]);
    dft_reg<16, true>(v);
    if (pair0 + g >= npairs) return;
#pragma unroll
    for (int p = 8; p < 16; ++p) {
        const uint64_t tt = a.mid + j + (uint64_t)(p - 8) * Q0;
        if (tt >= tend) continue;
        cplx y = v[p];
        const int tp = (int)(tt - a.mid);
        if (tp < a.J - 1) {  // exact near field: lags t - j < J
            const double* cp = a.col + (uint64_t)pi.pb * N;
            const double* xr = a.U + pi.row1 * N;
            const uint64_t jlo = (tt >= a.lo + (uint64_t)(a.J - 1)) ? tt - (uint64_t)(a.J - 1) : a.lo;
            double s1 = 0.0, s2 = 0.0;
            for (uint64_t jj = a.mid; jj-- > jlo;) {
                const double cv = cp[tt - jj];
                s1 = fma(cv, xr[jj], s1);
                if (pi.has2) s2 = fma(cv, xr[N + jj], s2);
            }
            y.x += s1;
            y.y += s2;
        }
        a.X[pi.row1 * N + tt] = r1[p - 8] - y.x;
        if (pi.has2) a.X[(pi.row1 + 1) * N + tt] = r2[p - 8] - y.y;
    }
}

// G = kMpTile / n row pairs per CTA (compile time; pairs past the end are
// dead).  When a CTA holds exactly 16 points per thread (n <= kMpTile), each
// phase's global loads -- spectrum for the fused pass, twiddles and targets for
// the last pass -- are issued before the barrier that precedes the phase
// (ncu: these L1/L2 round trips were the top long-scoreboard stalls).
template <int LOGN>
#ifndef FT_MP1G_MINB
#define FT_MP1G_MINB 2
#endif
#ifndef FT_MP1_MINB
#define FT_MP1_MINB 2
#endif
__global__ void __launch_bounds__(kMpThreads, FT_MP1_MINB) mp1_kernel(MpArgs a) {
    pdl_launch_dependents(a.pdl_trigger);
    pdl_wait();
    using PL = Plan1<LOGN>;
    constexpr int n = PL::n, Q0 = PL::Q0, RL = PL::RL;
    constexpr int G = n >= kMpTile ? 1 : kMpTile / n;
    constexpr int total = G * n;
#ifdef FT_MP1_NOPRE
    constexpr bool PRE = false;
#else
    constexpr bool PRE = total == kMpThreads * 16;
#endif
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* buf = reinterpret_cast<cplx*>(smem_raw);
    __shared__ PairInfo s_pair[G];
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    const int pair0 = blockIdx.x * G;
    const uint64_t N = a.N;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        const int rp = min(pair0 + g, npairs - 1);
        const int pb = rp / a.pairs_per_problem, lp = rp - pb * a.pairs_per_problem;
        const int i1 = 2 * lp;
        s_pair[g] = {(uint64_t)(pb * a.nodes + i1), pb, (pair0 + g < npairs && i1 + 1 < a.nodes) ? 1 : 0};
    }
    __syncthreads();

    // pass 0 (S = n, radix 16) from HBM; inputs p >= 8 are the zero padding
#pragma unroll 1
    for (int t = threadIdx.x; t < total / 16; t += kMpThreads) {
        const int g = t / Q0, j = t - g * Q0;
        const PairInfo pi = s_pair[g];
        const double* x1 = a.U + pi.row1 * N + a.lo + j;
        const bool live = pair0 + g < npairs;
        cplx v[16];
#pragma unroll
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            v[p].x = live ? x1[(uint64_t)p * Q0] : 0.0;
            v[p].y = (live && pi.has2) ? x1[N + (uint64_t)p * Q0] : 0.0;
        }
        dft_reg_halfzero<16>(v);  // inputs 8..15 are the zero padding
        cplx w[16];
        pass_twiddles<16>(w, a.tw, n, j);
#pragma unroll
        for (int q = 1; q < 16; ++q) v[q] = cmul(v[q], w[q]);
        const int pb = sphys(g * n + j);
#pragma unroll
        for (int q = 0; q < 16; ++q) buf[pb + q * (Q0 + (Q0 >> 4))] = v[q];
    }
    mid_fwd_s<LOGN - 4, LOGN>(buf, total, a.tw);

    // fused: last forward pass (S = RL, twiddle-free), spectrum, first inverse pass
    constexpr int FT = total / RL / kMpThreads;  // fused tasks per thread (PRE)
    cplx spv[PRE ? 16 : 1];
    if constexpr (PRE) {
#pragma unroll
        for (int k = 0; k < FT; ++k) {
            const int base = (threadIdx.x + k * kMpThreads) * RL;
            const cplx* sp = a.spec + (uint64_t)s_pair[base >> LOGN].pb * n + (base & (n - 1));
#pragma unroll
            for (int p = 0; p < RL; ++p) spv[k * RL + p] = ldgc(&sp[p]);
        }
    }
    __syncthreads();
    if constexpr (PRE) {
#pragma unroll
        for (int k = 0; k < FT; ++k) {
            const int pbx = sphys((threadIdx.x + k * kMpThreads) * RL);
            cplx v[RL];
#pragma unroll
            for (int p = 0; p < RL; ++p) v[p] = buf[pbx + p];
            dft_reg<RL, false>(v);
#pragma unroll
            for (int p = 0; p < RL; ++p) v[p] = cmul(v[p], spv[k * RL + p]);
            dft_reg<RL, true>(v);
#pragma unroll
            for (int p = 0; p < RL; ++p) buf[pbx + p] = v[p];
        }
    } else {
        for (int t = threadIdx.x; t < total / RL; t += kMpThreads) {
            const int base = t * RL;
            const int pbx = sphys(base);
            cplx v[RL];
#pragma unroll
            for (int p = 0; p < RL; ++p) v[p] = buf[pbx + p];
            dft_reg<RL, false>(v);
            const cplx* sp = a.spec + (uint64_t)s_pair[base >> LOGN].pb * n + (base & (n - 1));
#pragma unroll
            for (int p = 0; p < RL; ++p) v[p] = cmul(v[p], ldgc(&sp[p]));
            dft_reg<RL, true>(v);
#pragma unroll
            for (int p = 0; p < RL; ++p) buf[pbx + p] = v[p];
        }
    }
    mid_inv_s<LOGN - 4, LOGN>(buf, total, a.tw);

    // last inverse pass (S = n, radix 16): outputs p >= 8 are the targets [mid, mid + h)
    if constexpr (PRE) {
        cplx w[16];
        double r1[8], r2[8];
        mp1_last_prefetch<Q0>(a, s_pair, pair0, npairs, threadIdx.x, w, r1, r2);
        __syncthreads();
        mp1_last_task<Q0>(a, buf, s_pair, pair0, npairs, threadIdx.x, w, r1, r2);
    } else {
        __syncthreads();
#pragma unroll 1
        for (int t = threadIdx.x; t < total / 16; t += kMpThreads) {
            cplx w[16];
            double r1[8], r2[8];
            mp1_last_prefetch<Q0>(a, s_pair, pair0, npairs, t, w, r1, r2);
            mp1_last_task<Q0>(a, buf, s_pair, pair0, npairs, t, w, r1, r2);
        }
    }
}

// ---- group-private variant (n <= kMpTile): no CTA-wide barriers -------------
// Every pass of the n-point transform of pair g touches only that pair's SMEM
// region, and with the task numbering below the n/16 threads that own it form a
// contiguous group (half a warp for n = 256, a warp for 512, 2/4 warps for
// 1024/2048).  Groups synchronise privately (__syncwarp or a named barrier per
// group), so they drift out of phase: one group's HBM loads overlap another's
// FFT work instead of the whole CTA waiting at each barrier.
template <int LOGN>
struct GroupSync {
    static constexpr int GT = (1 << LOGN) / 16;  // threads per pair
    __device__ static __forceinline__ void sync(int g) {
        if constexpr (GT <= 32) {
            __syncwarp();
        } else if constexpr (GT < kMpThreads) {
            asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(GT) : "memory");
        } else {
            __syncthreads();
        }
    }
};

template <int LOGS, int LOGN>
__device__ __forceinline__ void mid_fwd_g(cplx* buf, int total, const cplx* tw, int g) {
    if constexpr (LOGS > lg2c(Plan1<LOGN>::RL)) {
        GroupSync<LOGN>::sync(g);
        pass_c<16, LOGS, false>(buf, total, tw);
        mid_fwd_g<LOGS - 4, LOGN>(buf, total, tw, g);
    }
}
template <int LOGS, int LOGN>
__device__ __forceinline__ void mid_inv_g(cplx* buf, int total, const cplx* tw, int g) {
    if constexpr (LOGS > lg2c(Plan1<LOGN>::RL)) {
        mid_inv_g<LOGS - 4, LOGN>(buf, total, tw, g);
        GroupSync<LOGN>::sync(g);
        pass_c<16, LOGS, true>(buf, total, tw);
    }
}

template <int LOGN>
__global__ void __launch_bounds__(kMpThreads, FT_MP1G_MINB) mp1g_kernel(MpArgs a) {
    pdl_launch_dependents(a.pdl_trigger);
    pdl_wait();
    using PL = Plan1<LOGN>;
    constexpr int n = PL::n, Q0 = PL::Q0, RL = PL::RL;
    static_assert(n <= kMpTile, "group-private plan needs n <= kMpTile");
    constexpr int G = kMpTile / n, GT = n / 16;
    constexpr int total = kMpTile;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* buf = reinterpret_cast<cplx*>(smem_raw);
    const int tid = threadIdx.x;
    const int g = tid / GT, j = tid - g * GT;  // pass-0 / last-pass task tid: pair g, column j (GT == Q0)
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    const int pair = blockIdx.x * G + g;
    const bool live = pair < npairs;
    const uint64_t N = a.N;
    PairInfo pi;
    {
        const int rp = min(pair, npairs - 1);
        const int pb = rp / a.pairs_per_problem, lp = rp - pb * a.pairs_per_problem;
        pi = {(uint64_t)(pb * a.nodes + 2 * lp), pb, (live && 2 * lp + 1 < a.nodes) ? 1 : 0};
    }

    // pass 0 (S = n, radix 16) from HBM; inputs p >= 8 are the zero padding
    {
        const double* x1 = a.U + pi.row1 * N + a.lo + j;
        cplx v[16];
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            v[p].x = live ? x1[(uint64_t)p * Q0] : 0.0;
            v[p].y = (live && pi.has2) ? x1[N + (uint64_t)p * Q0] : 0.0;
        }
        dft_reg_halfzero<16>(v);
        cplx w[16];
        pass_twiddles<16>(w, a.tw, n, j);
#pragma unroll
        for (int q = 1; q < 16; ++q) v[q] = cmul(v[q], w[q]);
        const int pb = sphys(g * n + j);
#pragma unroll
        for (int q = 0; q < 16; ++q) buf[pb + q * (Q0 + (Q0 >> 4))] = v[q];
    }
    mid_fwd_g<LOGN - 4, LOGN>(buf, total, a.tw, g);

    // fused pass: this group's tasks t = g*(n/RL) + j + k*GT, k < 16/RL
    constexpr int FT = 16 / RL;
    cplx spv[16];
#pragma unroll
    for (int k = 0; k < FT; ++k) {
        const int base = (g * (n / RL) + j + k * GT) * RL;
        const cplx* sp = a.spec + (uint64_t)pi.pb * n + (base & (n - 1));
#pragma unroll
        for (int p = 0; p < RL; ++p) spv[k * RL + p] = ldgc(&sp[p]);
    }
    GroupSync<LOGN>::sync(g);
#pragma unroll
    for (int k = 0; k < FT; ++k) {
        const int pbx = sphys((g * (n / RL) + j + k * GT) * RL);
        cplx v[RL];
#pragma unroll
        for (int p = 0; p < RL; ++p) v[p] = buf[pbx + p];
        dft_reg<RL, false>(v);
#pragma unroll
        for (int p = 0; p < RL; ++p) v[p] = cmul(v[p], spv[k * RL + p]);
        dft_reg<RL, true>(v);
#pragma unroll
        for (int p = 0; p < RL; ++p) buf[pbx + p] = v[p];
    }
    mid_inv_g<LOGN - 4, LOGN>(buf, total, a.tw, g);

    // last inverse pass (S = n, radix 16): outputs p >= 8 are the targets [mid, mid + h)
    const uint64_t tend = a.hi < N ? a.hi : N;
    double r1[8], r2[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        const uint64_t tt = a.mid + j + (uint64_t)p * Q0;
        const bool ok = live && tt < tend;
        r1[p] = (ok && a.rsrc) ? a.rsrc[pi.row1 * N + tt] : 0.0;
        r2[p] = (ok && pi.has2 && a.rsrc) ? a.rsrc[(pi.row1 + 1) * N + tt] : 0.0;
    }
    cplx w[16];
    pass_twiddles<16>(w, a.tw, n, j);
    GroupSync<LOGN>::sync(g);
    const int pbx = sphys(g * n + j);
    cplx v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = buf[pbx + q * (Q0 + (Q0 >> 4))];
#pragma unroll
    for (int q = 1; q < 16; ++q) v[q] = cmulc(v[q], w[q]);
    dft_reg<16, true>(v);
    if (!live) return;
#pragma unroll
    for (int p = 8; p < 16; ++p) {
        const uint64_t tt = a.mid + j + (uint64_t)(p - 8) * Q0;
        if (tt >= tend) continue;
        cplx y = v[p];
        const int tp = (int)(tt - a.mid);
        if (tp < a.J - 1) {  // exact near field: lags t - j < J
            const double* cp = a.col + (uint64_t)pi.pb * N;
            const double* xr = a.U + pi.row1 * N;
            const uint64_t jlo = (tt >= a.lo + (uint64_t)(a.J - 1)) ? tt - (uint64_t)(a.J - 1) : a.lo;
            double s1 = 0.0, s2 = 0.0;
            for (uint64_t jj = a.mid; jj-- > jlo;) {
                const double cv = cp[tt - jj];
                s1 = fma(cv, xr[jj], s1);
                if (pi.has2) s2 = fma(cv, xr[N + jj], s2);
            }
            y.x += s1;
            y.y += s2;
        }
        a.X[pi.row1 * N + tt] = r1[p - 8] - y.x;
        if (pi.has2) a.X[(pi.row1 + 1) * N + tt] = r2[p - 8] - y.y;
    }
}

// ---- radix-8, high-occupancy variant (256 <= n <= 4096; opt-in, FT_MP8=0x1f00) -----------
// mp1g_kernel holds 16 complex points per thread (128 registers): 16 warps per SM, and ncu
// shows the FP64 pipe ~50 % busy with every warp waiting on fixed-latency, shared-memory and
// global-load dependencies.  This variant tests the occupancy hypothesis: 8 points per thread
// in radix-8 passes at <= 85 registers, 24 warps per SM (3 CTAs of 256 threads and a
// 2048-point tile for n <= 2048; FT_MP8_MINB=4: <= 64 registers with ~400 B of spills, 32
// warps).  Same structure otherwise: pass 0 from HBM with the zero half pruned, group-private
// barriers, last forward pass + spectrum + first inverse pass fused in registers, last
// inverse pass straight to HBM.  Shared-memory padding is one slot per 8 points
// (conflict-free 16-byte accesses for every pass stride and for the 8 contiguous points of
// the fused pass).  The spectrum comes from spec8_kernel (same pass plan, so the
// digit-reversed orders agree).
// Measured on B200 (round 2, cfg4 per level, ms; mp1g / mp8 at 24 warps / mp8 at 32 warps):
//   n = 256: 20.1 / 21.6 / 27.2   512: 18.4 / 22.9 / 28.9   1024: 20.5 / 27.1 / 34.7
//   2048: 24.5 / 28.0 / 36.6      4096: 23.0 / 31.2 / 44.6
// More warps do not help: the level is bound by the shared-memory / L1 data path and the
// FP64 pipe together (each ~50-55 % busy in mp1g), and radix 8 adds shared-memory round
// trips and twiddle loads per point.  Kept as the measured reference point, not the default.
__device__ __forceinline__ int sphys8(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int sphys8_len(int n) { return n + (n >> 3) + 1; }
#ifndef FT_MP8_DEFAULT
#define FT_MP8_DEFAULT 0
#endif

template <int LOGN>
struct Plan8 {
    static constexpr int n = 1 << LOGN;
    static constexpr int NP = (LOGN - 1) / 3;      // radix-8 passes before the fused one
    static constexpr int LOGRL = LOGN - 3 * NP;    // fused radix 2, 4 or 8
    static constexpr int RL = 1 << LOGRL;
    static constexpr int Q0 = n / 8;
    static constexpr int GT = n / 8;               // threads per pair
    static constexpr int TPB = GT < 256 ? 256 : GT;
    static constexpr int TILE = TPB * 8;
    static constexpr int G = TILE / n;
};

template <int GT, int TPB>
__device__ __forceinline__ void group_sync8(int g) {
    if constexpr (GT <= 32) {
        __syncwarp();
    } else if constexpr (GT < TPB) {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(GT) : "memory");
    } else {
        __syncthreads();
    }
}

// one radix-8 pass of group size S = 2^LOGS over this thread's butterfly (tl = thread within the pair)
template <int LOGS, bool INV>
__device__ __forceinline__ void pass8(cplx* gb, int tl, const cplx* __restrict__ tw) {
    constexpr int LOGQ = LOGS - 3, Q = 1 << LOGQ, S = 1 << LOGS;
    const int j = tl & (Q - 1);
    const int base = ((tl >> LOGQ) << LOGS) + j;
    cplx* b = gb + sphys8(base);
    cplx v[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) v[p] = b[p * Q + ((p * Q) >> 3)];
    if (!INV) {
        dft_reg<8, false>(v);
        cplx w[8];
        pass_twiddles<8>(w, tw, S, j);
#pragma unroll
        for (int q = 1; q < 8; ++q) v[q] = cmul(v[q], w[q]);
    } else {
        cplx w[8];
        pass_twiddles<8>(w, tw, S, j);
#pragma unroll
        for (int q = 1; q < 8; ++q) v[q] = cmulc(v[q], w[q]);
        dft_reg<8, true>(v);
    }
#pragma unroll
    for (int p = 0; p < 8; ++p) b[p * Q + ((p * Q) >> 3)] = v[p];
}

template <int LOGS, int LOGN>
__device__ __forceinline__ void mid_fwd8(cplx* gb, int tl, const cplx* tw, int g) {
    using PL = Plan8<LOGN>;
    if constexpr (LOGS > PL::LOGRL) {
        group_sync8<PL::GT, PL::TPB>(g);
        pass8<LOGS, false>(gb, tl, tw);
        mid_fwd8<LOGS - 3, LOGN>(gb, tl, tw, g);
    }
}
template <int LOGS, int LOGN>
__device__ __forceinline__ void mid_inv8(cplx* gb, int tl, const cplx* tw, int g) {
    using PL = Plan8<LOGN>;
    if constexpr (LOGS > PL::LOGRL) {
        mid_inv8<LOGS - 3, LOGN>(gb, tl, tw, g);
        group_sync8<PL::GT, PL::TPB>(g);
        pass8<LOGS, true>(gb, tl, tw);
    }
}

template <int LOGN>
#ifndef FT_MP8_MINB
#define FT_MP8_MINB 3  // CTAs of 256 threads per SM (3: <= 85 registers, no spills; 4: <= 64)
#endif
__global__ void __launch_bounds__(Plan8<LOGN>::TPB, FT_MP8_MINB * 256 / Plan8<LOGN>::TPB) mp8_kernel(MpArgs a) {
    pdl_launch_dependents(a.pdl_trigger);
    pdl_wait();
    using PL = Plan8<LOGN>;
    constexpr int n = PL::n, Q0 = PL::Q0, RL = PL::RL, GT = PL::GT, G = PL::G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* buf = reinterpret_cast<cplx*>(smem_raw);
    const int tid = threadIdx.x;
    const int g = tid / GT, j = tid - g * GT;
    cplx* gb = buf + sphys8(g * n);
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    const int pair = blockIdx.x * G + g;
    const bool live = pair < npairs;
    const uint64_t N = a.N;
    PairInfo pi;
    {
        const int rp = min(pair, npairs - 1);
        const int pb = rp / a.pairs_per_problem, lp = rp - pb * a.pairs_per_problem;
        pi = {(uint64_t)(pb * a.nodes + 2 * lp), pb, (live && 2 * lp + 1 < a.nodes) ? 1 : 0};
    }
    // pass 0 (S = n) from HBM; inputs p >= 4 are the zero padding
    {
        const double* x1 = a.U + pi.row1 * N + a.lo + j;
        cplx v[8];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            v[p].x = live ? x1[(uint64_t)p * Q0] : 0.0;
            v[p].y = (live && pi.has2) ? x1[N + (uint64_t)p * Q0] : 0.0;
        }
        dft_reg_halfzero<8>(v);
        cplx w[8];
        pass_twiddles<8>(w, a.tw, n, j);
#pragma unroll
        for (int q = 1; q < 8; ++q) v[q] = cmul(v[q], w[q]);
        cplx* b = gb + sphys8(j);
#pragma unroll
        for (int q = 0; q < 8; ++q) b[q * (Q0 + (Q0 >> 3))] = v[q];
    }
    mid_fwd8<LOGN - 3, LOGN>(gb, j, a.tw, g);
    // fused: last forward pass (radix RL, twiddle-free), spectrum, first inverse pass, on the
    // 8 contiguous points 8 j .. 8 j + 7 of the pair
    {
        const cplx* sp = a.spec + (uint64_t)pi.pb * n + 8 * j;
        cplx spv[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) spv[p] = ldgc(&sp[p]);
        group_sync8<GT, PL::TPB>(g);
        cplx* b = gb + 9 * j;  // sphys8(8 j)
#pragma unroll
        for (int k = 0; k < 8 / RL; ++k) {
            cplx v[RL];
#pragma unroll
            for (int p = 0; p < RL; ++p) v[p] = b[k * RL + p];
            dft_reg<RL, false>(v);
#pragma unroll
            for (int p = 0; p < RL; ++p) v[p] = cmul(v[p], spv[k * RL + p]);
            dft_reg<RL, true>(v);
#pragma unroll
            for (int p = 0; p < RL; ++p) b[k * RL + p] = v[p];
        }
    }
    mid_inv8<LOGN - 3, LOGN>(gb, j, a.tw, g);
    // last inverse pass (S = n): outputs p >= 4 are the targets [mid, mid + h)
    const uint64_t tend = a.hi < N ? a.hi : N;
    cplx w[8];
    pass_twiddles<8>(w, a.tw, n, j);
    group_sync8<GT, PL::TPB>(g);
    cplx v[8];
    {
        const cplx* b = gb + sphys8(j);
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = b[q * (Q0 + (Q0 >> 3))];
    }
#pragma unroll
    for (int q = 1; q < 8; ++q) v[q] = cmulc(v[q], w[q]);
    double r1[4], r2[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const uint64_t tt = a.mid + j + (uint64_t)p * Q0;
        const bool ok = live && tt < tend;
        r1[p] = (ok && a.rsrc) ? a.rsrc[pi.row1 * N + tt] : 0.0;
        r2[p] = (ok && pi.has2 && a.rsrc) ? a.rsrc[(pi.row1 + 1) * N + tt] : 0.0;
    }
    dft_reg<8, true>(v);
    if (!live) return;
#pragma unroll
    for (int p = 4; p < 8; ++p) {
        const uint64_t tt = a.mid + j + (uint64_t)(p - 4) * Q0;
        if (tt >= tend) continue;
        cplx y = v[p];
        const int tp = (int)(tt - a.mid);
        if (tp < a.J - 1) {  // exact near field: lags t - j < J
            const double* cp = a.col + (uint64_t)pi.pb * N;
            const double* xr = a.U + pi.row1 * N;
            const uint64_t jlo = (tt >= a.lo + (uint64_t)(a.J - 1)) ? tt - (uint64_t)(a.J - 1) : a.lo;
            double s1 = 0.0, s2 = 0.0;
#pragma unroll 1
            for (uint64_t jj = a.mid; jj-- > jlo;) {
                const double cv = cp[tt - jj];
                s1 = fma(cv, xr[jj], s1);
                if (pi.has2) s2 = fma(cv, xr[N + jj], s2);
            }
            y.x += s1;
            y.y += s2;
        }
        a.X[pi.row1 * N + tt] = r1[p - 4] - y.x;
        if (pi.has2) a.X[(pi.row1 + 1) * N + tt] = r2[p - 4] - y.y;
    }
}

// Spectrum of one level in the radix-8 plan order: full n-point column (lags J <= k < min(n, N)),
// scaled 1/n.  One CTA of n / 8 threads per problem.
template <int LOGN>
__global__ void __launch_bounds__(Plan8<LOGN>::GT, 1) spec8_kernel(const double* col, uint64_t N, int J, cplx* spec,
                                                                   const cplx* tw) {
    using PL = Plan8<LOGN>;
    constexpr int n = PL::n, Q0 = PL::Q0, RL = PL::RL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* buf = reinterpret_cast<cplx*>(smem_raw);
    const int pb = blockIdx.x, j = threadIdx.x;
    const double* c = col + (uint64_t)pb * N;
    const uint64_t kend = (uint64_t)n < N ? (uint64_t)n : N;
    {
        cplx v[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            const uint64_t k = (uint64_t)j + (uint64_t)p * Q0;
            v[p] = {(k >= (uint64_t)J && k < kend) ? c[k] : 0.0, 0.0};
        }
        dft_reg<8, false>(v);
        cplx w[8];
        pass_twiddles<8>(w, tw, n, j);
#pragma unroll
        for (int q = 1; q < 8; ++q) v[q] = cmul(v[q], w[q]);
        cplx* b = buf + sphys8(j);
#pragma unroll
        for (int q = 0; q < 8; ++q) b[q * (Q0 + (Q0 >> 3))] = v[q];
    }
    mid_fwd8<LOGN - 3, LOGN>(buf, j, tw, 0);
    __syncthreads();
    const double scale = 1.0 / (double)n;
    cplx* b = buf + 9 * j;
#pragma unroll
    for (int k = 0; k < 8 / RL; ++k) {
        cplx v[RL];
#pragma unroll
        for (int p = 0; p < RL; ++p) v[p] = b[k * RL + p];
        dft_reg<RL, false>(v);
#pragma unroll
        for (int p = 0; p < RL; ++p) spec[(uint64_t)pb * n + 8 * j + k * RL + p] = {v[p].x * scale, v[p].y * scale};
    }
}

// ---- persistent, TMA-staged variant of mp1g_kernel ------------------------------
// One CTA per SM slot loops over tiles of G = kMpTile / n row pairs.  While a tile is being
// transformed, the NEXT tile's source rows (G pairs x 2 rows x h doubles = 32 KB, one
// contiguous segment per row) are copied HBM -> shared memory by the TMA unit
// (cp.async.bulk, completion counted on an mbarrier) and the lines of its targets are
// prefetched into L2; pass 0 then reads its inputs from shared memory.  ncu on mp1g_kernel:
// the first use of the source loads was 10 % of all stall samples (HBM latency exposed once
// per CTA, two CTAs per SM).  Needs 16-byte aligned row segments (even N; lo is a multiple
// of the leaf length).  Measured on B200 (round 2): correct, but slower than mp1g_kernel
// (see launch_mp1), so it is opt-in (FT_MP1P=1) and kept as the TMA reference point.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int LOGN>
__global__ void __launch_bounds__(kMpThreads, 2) mp1p_kernel(MpArgs a, int ntiles) {
    pdl_launch_dependents(a.pdl_trigger);
    pdl_wait();
    using PL = Plan1<LOGN>;
    constexpr int n = PL::n, h = PL::h, Q0 = PL::Q0, RL = PL::RL;
    static_assert(n <= kMpTile, "group-private plan needs n <= kMpTile");
    constexpr int G = kMpTile / n, GT = n / 16;
    constexpr int total = kMpTile;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* buf = reinterpret_cast<cplx*>(smem_raw);
    double* stage = reinterpret_cast<double*>(buf + spad_len(total));  // [G][2][h] source rows of the tile
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(stage + 2 * G * h);
    const int tid = threadIdx.x;
    const int g = tid / GT, j = tid - g * GT;
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    const uint64_t N = a.N;
    const uint64_t tend = a.hi < N ? a.hi : N;

    // issue (tid < 2G): row (tid & 1) of pair tid >> 1 of tile t -> stage; every issuer arrives
    auto issue = [&](int t) {
        if (tid < 2 * G) {
            const int pg = tid >> 1, r = tid & 1;
            const int pair = t * G + pg;
            const int pb = min(pair, npairs - 1) / a.pairs_per_problem;
            const int lp = min(pair, npairs - 1) - pb * a.pairs_per_problem;
            const bool ok = pair < npairs && 2 * lp + r < a.nodes;
            if (ok) {
                mbar_arrive_expect_tx(mbar, h * 8);
                bulk_g2s(stage + (size_t)(2 * pg + r) * h, a.U + ((uint64_t)(pb * a.nodes + 2 * lp + r)) * N + a.lo,
                         h * 8, mbar);
            } else {
                mbar_arrive_expect_tx(mbar, 0);
            }
        }
        // the tile's targets: into L2 while the previous tile is transformed (128-byte lines)
        if (a.rsrc) {
            constexpr int LPR = h * 8 / 128 > 0 ? h * 8 / 128 : 1;  // lines per row
            for (int e = tid; e < 2 * G * LPR; e += kMpThreads) {
                const int rr = e / LPR, ln = e - rr * LPR;
                const int pair = t * G + (rr >> 1);
                const int pb = min(pair, npairs - 1) / a.pairs_per_problem;
                const int lp = min(pair, npairs - 1) - pb * a.pairs_per_problem;
                if (pair < npairs && 2 * lp + (rr & 1) < a.nodes && a.mid + (uint64_t)ln * 16 < tend)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a.rsrc + ((uint64_t)(pb * a.nodes + 2 * lp + (rr & 1))) * N +
                                                                     a.mid + (uint64_t)ln * 16));
            }
        }
    };
    if (tid == 0) {
        mbar_init(mbar, 2 * G);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int tile = blockIdx.x;
    if (tile < ntiles) issue(tile);
    unsigned parity = 0;
    for (; tile < ntiles; tile += gridDim.x) {
        const int pair = tile * G + g;
        const bool live = pair < npairs;
        PairInfo pi;
        {
            const int rp = min(pair, npairs - 1);
            const int pb = rp / a.pairs_per_problem, lp = rp - pb * a.pairs_per_problem;
            pi = {(uint64_t)(pb * a.nodes + 2 * lp), pb, (live && 2 * lp + 1 < a.nodes) ? 1 : 0};
        }
        // pass 0 (S = n, radix 16) from the staged rows; inputs p >= 8 are the zero padding
        {
            cplx w[16];
            pass_twiddles<16>(w, a.tw, n, j);
            mbar_wait(mbar, parity);
            parity ^= 1u;
            const double* s1 = stage + (size_t)(2 * g) * h + j;
            cplx v[16];
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                v[p].x = live ? s1[p * Q0] : 0.0;
                v[p].y = (live && pi.has2) ? s1[h + p * Q0] : 0.0;
            }
            __syncthreads();  // every thread has its inputs (and is done with the previous tile)
            if (tile + (int)gridDim.x < ntiles) issue(tile + gridDim.x);
            dft_reg_halfzero<16>(v);
#pragma unroll
            for (int q = 1; q < 16; ++q) v[q] = cmul(v[q], w[q]);
            const int pb = sphys(g * n + j);
#pragma unroll
            for (int q = 0; q < 16; ++q) buf[pb + q * (Q0 + (Q0 >> 4))] = v[q];
        }
        mid_fwd_g<LOGN - 4, LOGN>(buf, total, a.tw, g);

        // fused pass: this group's tasks t = g*(n/RL) + j + k*GT, k < 16/RL
        constexpr int FT = 16 / RL;
        {
            cplx spv[16];
#pragma unroll
            for (int k = 0; k < FT; ++k) {
                const int base = (g * (n / RL) + j + k * GT) * RL;
                const cplx* sp = a.spec + (uint64_t)pi.pb * n + (base & (n - 1));
#pragma unroll
                for (int p = 0; p < RL; ++p) spv[k * RL + p] = ldgc(&sp[p]);
            }
            GroupSync<LOGN>::sync(g);
#pragma unroll
            for (int k = 0; k < FT; ++k) {
                const int pbx = sphys((g * (n / RL) + j + k * GT) * RL);
                cplx v[RL];
#pragma unroll
                for (int p = 0; p < RL; ++p) v[p] = buf[pbx + p];
                dft_reg<RL, false>(v);
#pragma unroll
                for (int p = 0; p < RL; ++p) v[p] = cmul(v[p], spv[k * RL + p]);
                dft_reg<RL, true>(v);
#pragma unroll
                for (int p = 0; p < RL; ++p) buf[pbx + p] = v[p];
            }
        }
        mid_inv_g<LOGN - 4, LOGN>(buf, total, a.tw, g);

        // last inverse pass (S = n, radix 16): outputs p >= 8 are the targets [mid, mid + h)
        double r1[8], r2[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            const uint64_t tt = a.mid + j + (uint64_t)p * Q0;
            const bool ok = live && tt < tend;
            r1[p] = (ok && a.rsrc) ? a.rsrc[pi.row1 * N + tt] : 0.0;
            r2[p] = (ok && pi.has2 && a.rsrc) ? a.rsrc[(pi.row1 + 1) * N + tt] : 0.0;
        }
        cplx w[16];
        pass_twiddles<16>(w, a.tw, n, j);
        GroupSync<LOGN>::sync(g);
        const int pbx = sphys(g * n + j);
        cplx v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = buf[pbx + q * (Q0 + (Q0 >> 4))];
#pragma unroll
        for (int q = 1; q < 16; ++q) v[q] = cmulc(v[q], w[q]);
        dft_reg<16, true>(v);
        if (live) {
#pragma unroll
            for (int p = 8; p < 16; ++p) {
                const uint64_t tt = a.mid + j + (uint64_t)(p - 8) * Q0;
                if (tt >= tend) continue;
                cplx y = v[p];
                const int tp = (int)(tt - a.mid);
                if (tp < a.J - 1) {  // exact near field: lags t - j < J
                    const double* cp = a.col + (uint64_t)pi.pb * N;
                    const double* xr = a.U + pi.row1 * N;
                    const uint64_t jlo = (tt >= a.lo + (uint64_t)(a.J - 1)) ? tt - (uint64_t)(a.J - 1) : a.lo;
                    double s1 = 0.0, s2 = 0.0;
                    for (uint64_t jj = a.mid; jj-- > jlo;) {
                        const double cv = cp[tt - jj];
                        s1 = fma(cv, xr[jj], s1);
                        if (pi.has2) s2 = fma(cv, xr[N + jj], s2);
                    }
                    y.x += s1;
                    y.y += s2;
                }
                a.X[pi.row1 * N + tt] = r1[p - 8] - y.x;
                if (pi.has2) a.X[(pi.row1 + 1) * N + tt] = r2[p - 8] - y.y;
            }
        }
        // (the next tile's pass 0 writes this group's region of buf only after the CTA barrier
        // that every thread reaches after finishing the reads above)
    }
}

// Spectrum of one level for the single-CTA plan: full n-point column (lags
// J <= k < min(n, N)), same passes, scaled 1/n, stored in plan order.
template <int LOGN>
__global__ void __launch_bounds__(kMpThreads, 1) spec1_kernel(const double* col, uint64_t N, int J, cplx* spec,
                                                         const cplx* tw) {
    using PL = Plan1<LOGN>;
    constexpr int n = PL::n, Q0 = PL::Q0, RL = PL::RL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* buf = reinterpret_cast<cplx*>(smem_raw);
    const int pb = blockIdx.x;
    const double* c = col + (uint64_t)pb * N;
    const uint64_t kend = (uint64_t)n < N ? (uint64_t)n : N;
    for (int t = threadIdx.x; t < n / 16; t += blockDim.x) {
        const int j = t;
        cplx v[16];
#pragma unroll
        for (int p = 0; p < 16; ++p) {
            const uint64_t k = (uint64_t)j + (uint64_t)p * Q0;
            v[p] = {(k >= (uint64_t)J && k < kend) ? c[k] : 0.0, 0.0};
        }
        dft_reg<16, false>(v);
        cplx w[16];
        pass_twiddles<16>(w, tw, n, j);
#pragma unroll
        for (int q = 1; q < 16; ++q) v[q] = cmul(v[q], w[q]);
        const int pbx = sphys(j);
#pragma unroll
        for (int q = 0; q < 16; ++q) buf[pbx + q * (Q0 + (Q0 >> 4))] = v[q];
    }
    __syncthreads();
    mid_fwd<LOGN - 4, LOGN>(buf, n, tw);
    const double scale = 1.0 / (double)n;
    for (int t = threadIdx.x; t < n / RL; t += blockDim.x) {
        const int base = t * RL;
        const int pbx = sphys(base);
        cplx v[RL];
#pragma unroll
        for (int p = 0; p < RL; ++p) v[p] = buf[pbx + p];
        dft_reg<RL, false>(v);
#pragma unroll
        for (int p = 0; p < RL; ++p) spec[(uint64_t)pb * n + base + p] = {v[p].x * scale, v[p].y * scale};
    }
}

// ---- direct history product for small blocks --------------------------------
// For n = 2h <= 256 the product is a small dense Toeplitz matrix applied to
// every row (h/2 FMA per unknown, fewer than the FFT's ~30-60 instructions):
//   R[row][mid + t'] -= sum_{j < h} col[h + t' - j] U[row][lo + j].
// Each thread owns 16 consecutive outputs of one row; a warp spans 32 rows
// with the same outputs so the column window is warp-uniform (SMEM
// broadcast), and the 16x16 block products are fully unrolled on registers.
#ifndef FT_DIR_THREADS
#define FT_DIR_THREADS 128  // 4 CTAs of 4 warps per SM: config 5 92.0 -> 91.5 ms (n = 128 level 6.3 -> 5.8), config 4 neutral; 512 slower
#endif
constexpr int kDirThreads = FT_DIR_THREADS;  // threads per direct-product CTA

template <int H>
__global__ void __launch_bounds__(kDirThreads, 512 / kDirThreads) mp_direct_kernel(MpArgs a) {
    pdl_launch_dependents(a.pdl_trigger);
    pdl_wait();
    constexpr int TT = H < 16 ? H : 16;
    constexpr int TPR = H / TT;                      // threads per row
    constexpr int RPC = kDirThreads / TPR;            // rows per CTA
    constexpr int LD = H + 1;                        // padded row stride (conflict-free)
    __shared__ double s_c[2 * H + TT];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* s_u = reinterpret_cast<double*>(smem_raw);   // [RPC][LD] source U
    double* s_r = s_u + RPC * LD;                        // [RPC][LD] target R -> result
    const int tid = threadIdx.x;
    const uint64_t row0 = (uint64_t)blockIdx.x * RPC;
    const uint64_t N = a.N;
    const uint64_t tend = a.hi < N ? a.hi : N;
    const int nt = (tend - a.mid) < (uint64_t)H ? (int)(tend - a.mid) : H;  // valid targets
    const int pb0 = (int)(row0 / a.nodes);
    const double* colp = a.col + (uint64_t)pb0 * N;
    for (int k = tid; k < 2 * H + TT; k += blockDim.x) s_c[k] = (k >= 1 && k < 2 * H && (uint64_t)k < N) ? colp[k] : 0.0;
    // coalesced staging: a warp reads 32 consecutive time steps of one row; all
    // of a thread's loads are issued before any store (memory-level parallelism)
    constexpr int PER = RPC * H / kDirThreads;  // 16
    double uu[PER], rv[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = tid + i * kDirThreads;
        const int r2 = e / H, j = e - r2 * H;
        const uint64_t row = row0 + r2;
        const bool ok = row < (uint64_t)a.rows;
        uu[i] = ok ? a.U[row * N + a.lo + j] : 0.0;
        rv[i] = (ok && j < nt && a.rsrc) ? a.rsrc[row * N + a.mid + j] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = tid + i * kDirThreads;
        const int r2 = e / H, j = e - r2 * H;
        s_u[r2 * LD + j] = uu[i];
        s_r[r2 * LD + j] = rv[i];
    }
    __syncthreads();
    const int p = tid / RPC;                         // output tile
    const int rr = tid - p * RPC;
    const uint64_t row = row0 + rr;
    const bool in_range = row < (uint64_t)a.rows;  // rows past the end compute on zeros
    const int pb = in_range ? (int)(row / a.nodes) : pb0;
    const bool uniform = (pb == pb0);
    const double* cpx = a.col + (uint64_t)pb * N;
    const double* u = s_u + rr * LD;
    double acc[TT];
#pragma unroll
    for (int t = 0; t < TT; ++t) acc[t] = 0.0;
    const int t1 = p * TT;
    // CTAs spanning two problems (batched plans whose node count is not a
    // multiple of the rows per CTA) take their column from global memory
    const double* cwin = uniform ? s_c : nullptr;
    double* s_cx = s_r + RPC * LD;  // per-thread fallback window (unused when uniform)
    (void)s_cx;
#pragma unroll 1
    for (int jb = 0; jb < H; jb += TT) {
        double wv[2 * TT - 1];
        const int base = H + t1 - jb - (TT - 1);
        if (cwin) {
#pragma unroll
            for (int i = 0; i < 2 * TT - 1; ++i) wv[i] = cwin[base + i];
        } else {
#pragma unroll
            for (int i = 0; i < 2 * TT - 1; ++i) {
                const int k = base + i;
                wv[i] = (k >= 1 && (uint64_t)k < N) ? cpx[k] : 0.0;
            }
        }
        double uv[TT];
#pragma unroll
        for (int i = 0; i < TT; ++i) uv[i] = u[jb + i];
#pragma unroll
        for (int jj = 0; jj < TT; ++jj)
#pragma unroll
            for (int t = 0; t < TT; ++t) acc[t] = fma(wv[t - jj + (TT - 1)], uv[jj], acc[t]);
    }
    double* rres = s_r + rr * LD + t1;
#pragma unroll
    for (int t = 0; t < TT; ++t) rres[t] -= acc[t];
    __syncthreads();
    for (int e = tid; e < RPC * H; e += blockDim.x) {
        const int r2 = e / H, j = e - r2 * H;
        const uint64_t rw = row0 + r2;
        if (rw < (uint64_t)a.rows && j < nt) a.X[rw * N + a.mid + j] = s_r[r2 * LD + j];
    }
}

// Kernel spectra of one D&C level for every problem: branch b of the column
// (lags J <= k < min(n, N)), folded, twisted, forward-transformed, scaled 1/n.
struct SpecArgs {
    const double* col;
    uint64_t N;
    int n, m, K, J;
    cplx* spec;  // [B][K][m]
    const cplx* tw;
    int logT;
};

__global__ void __launch_bounds__(kMpThreads) spectra_kernel(SpecArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* buf = reinterpret_cast<cplx*>(smem_raw);
    const int b = blockIdx.x, pb = blockIdx.y;
    const int K = a.K, m = a.m, n = a.n;
    const int logm = __ffs(m) - 1;
    const double* col = a.col + (uint64_t)pb * a.N;
    const uint64_t kend = (uint64_t)n < a.N ? (uint64_t)n : a.N;
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
        cplx v = {0.0, 0.0};
        for (int q = 0; q < K; ++q) {
            const uint64_t k = (uint64_t)q * m + r;
            const double c = (k >= (uint64_t)a.J && k < kend) ? col[k] : 0.0;
            const cplx zeta = conjc(a.tw[K + ((b * q) & (K - 1))]);
            v = cadd(v, cplx{c * zeta.x, c * zeta.y});
        }
        v = cmulc(v, a.tw[n + b * r]);
        buf[sphys(r)] = v;
    }
    __syncthreads();
    fft_forward(buf, m, logm, a.tw, a.logT);
    const double scale = 1.0 / (double)n;
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
        const cplx v = buf[sphys(r)];
        a.spec[((uint64_t)pb * K + b) * m + r] = {v.x * scale, v.y * scale};
    }
}

// ---- host launchers ---------------------------------------------------------

size_t mp_smem_bytes(int G, int m) { return sizeof(cplx) * (size_t)spad_len(G * m); }

static uint64_t split_batch_bytes() {
    static const uint64_t b = [] {
        const char* e = getenv("FT_MP_BATCH_MB");  // tuning knob (default: the whole scratch)
        const uint64_t v = e ? (uint64_t)atoll(e) << 20 : kMpScratchBytes;
        return std::min<uint64_t>(std::max<uint64_t>(v, 1ull << 20), kMpScratchBytes);
    }();
    return b;
}

// persistent split level (mp_split_kernel): default; FT_SPLIT_BATCHED=1 is the A/B switch back
// to the batched fold / branch / combine launches below
static bool split_persistent() {
    static const bool on = getenv("FT_SPLIT_BATCHED") == nullptr;
    return on;
}
constexpr uint64_t kSplitCtrOffset = kMpScratchBytes - (64u << 10);  // queue counters: last 64 KB of the scratch

template <int K, int LOGM>
static cudaError_t launch_mp_split_persistent(const MpArgs& a, cudaStream_t st) {
    constexpr int m = 1 << LOGM;
    const size_t smem = mp_smem_bytes(1, m);
    static DeviceOnce attr_set;
    static int occ = 0, sms = 0;
    if (attr_set.first()) {
        cudaError_t e = cudaFuncSetAttribute(mp_split_kernel<K, LOGM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mp_split_kernel<K, LOGM>, kMpThreads, smem);
        if (e != cudaSuccess) return e;
        attr_set.done();
    }
    const int ctas = sms * std::max(occ, 1);
    SplitQ q;
    q.npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    // lookahead: about twice the task groups the resident CTAs hold at once
    static const int dknob = getenv("FT_SPLIT_D") ? atoi(getenv("FT_SPLIT_D")) : 0;  // tuning knob
    q.D = dknob > 0 ? dknob : std::max(4, 2 * ctas / (K + 2 * kSplitParts) + 2);
    // ring: pairs p - 2D .. p are live; fold(p) reuses the slot of pair p - RS, whose combine sits
    // RS - 2D groups back -- give it D more groups so folds rarely wait on a running combine
    static const int rknob = getenv("FT_SPLIT_RS") ? atoi(getenv("FT_SPLIT_RS")) : 0;  // tuning knob
    q.RS = rknob > 0 ? rknob : 3 * q.D + 1;
    if ((uint64_t)q.RS * K * m * sizeof(cplx) > kSplitCtrOffset) q.RS = (int)(kSplitCtrOffset / ((uint64_t)K * m * sizeof(cplx)));
    if (q.RS < 2 * q.D + 1) q.D = (q.RS - 1) / 2;
    q.ntasks = (q.npairs + 2 * q.D) * (K + 2 * kSplitParts);
    static const int probe = getenv("FT_SPLIT_PROBE") ? atoi(getenv("FT_SPLIT_PROBE")) : 0;
    q.probe = probe;
    q.ctr = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(a.scratch) + kSplitCtrOffset);
    cudaError_t e = cudaMemsetAsync(q.ctr, 0, sizeof(unsigned) * (1 + 3 * (size_t)q.RS), st);
    if (e != cudaSuccess) return e;
    // co-residency is what makes the dependency waits safe (a waiting CTA only waits on tasks
    // dequeued before its own): never more CTAs than fit at once
    return launch_ex(mp_split_kernel<K, LOGM>, dim3(std::min(ctas, q.ntasks)), dim3(kMpThreads), smem, st, 1, a, q);
}

template <int K, int LOGM>
static cudaError_t launch_mp_split(const MpArgs& a0, cudaStream_t st) {
    if (split_persistent()) return launch_mp_split_persistent<K, LOGM>(a0, st);
    static DeviceOnce attr_set;
    if (attr_set.first()) {
        cudaFuncSetAttribute(mp_kernel<K, LOGM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mp_smem_bytes(1, (1 << LOGM) > kMpTile ? (1 << LOGM) : kMpTile));
        cudaFuncSetAttribute(mp_kernel<K, LOGM, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mp_smem_bytes(1, (1 << LOGM) > kMpTile ? (1 << LOGM) : kMpTile));
        attr_set.done();
    }
    // pre-fold measured faster for K = 16 (n = 65536: 63.5 -> 52.0 ms per level), slower
    // for K = 8 (42.8 -> 46.4 ms: the extra scratch round trip outweighs the K-fold re-reads)
    static const int prefold_min_k = getenv("FT_PREFOLD_MIN_K") ? atoi(getenv("FT_PREFOLD_MIN_K")) : 16;
    const bool prefold = K >= prefold_min_k && getenv("FT_NO_PREFOLD") == nullptr;
    constexpr int m = 1 << LOGM;
    const int npairs = (a0.rows / a0.nodes) * a0.pairs_per_problem;
    const int batch = (int)std::max<uint64_t>(1, split_batch_bytes() / ((uint64_t)K * m * sizeof(cplx)));
    MpArgs a = a0;
    for (int p0 = 0; p0 < npairs; p0 += batch) {
        a.pair_begin = p0;
        a.pair_count = std::min(batch, npairs - p0);
        if (prefold) {
            cudaError_t e = launch_ex(mp_fold_kernel<K, LOGM>, dim3(m / kMpThreads, a.pair_count), dim3(kMpThreads),
                                      0, st, 1, a);
            if (e != cudaSuccess) return e;
            e = launch_ex(mp_kernel<K, LOGM, true, true>, dim3(K, a.pair_count), dim3(kMpThreads),
                          mp_smem_bytes(a.G, m), st, 1, a);
            if (e != cudaSuccess) return e;
        } else {
            cudaError_t e = launch_ex(mp_kernel<K, LOGM, true>, dim3(K, a.pair_count), dim3(kMpThreads),
                                      mp_smem_bytes(a.G, m), st, 1, a);
            if (e != cudaSuccess) return e;
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        e = launch_ex(mpB_kernel<K, LOGM>, dim3(m / kMpThreads, a.pair_count), dim3(kMpThreads), 0, st, 1, a);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <int K, int LOGM>
static cudaError_t launch_mp_k(const MpArgs& a, int groups, cudaStream_t st) {
    if (a.scratch) return launch_mp_split<K, LOGM>(a, st);
    static DeviceOnce attr_set;
    if (attr_set.first()) {
        cudaFuncSetAttribute(mp_kernel<K, LOGM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mp_smem_bytes(1, (1 << LOGM) > kMpTile ? (1 << LOGM) : kMpTile));
        if (K > 8) cudaFuncSetAttribute(mp_kernel<K, LOGM, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr_set.done();
    }
    return launch_ex(mp_kernel<K, LOGM, false>, dim3(K, groups, 1), dim3(kMpThreads), mp_smem_bytes(a.G, a.m), st,
                     (unsigned)K, a);
}

template <int H>
static cudaError_t launch_direct_h(const MpArgs& a, cudaStream_t st) {
    constexpr int RPC = kDirThreads / (H / (H < 16 ? H : 16));
    const size_t smem = sizeof(double) * 2 * RPC * (H + 1);
    static DeviceOnce attr_set;
    if (attr_set.first()) {
        cudaFuncSetAttribute(mp_direct_kernel<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set.done();
    }
    const int ctas = (a.rows + RPC - 1) / RPC;
    return launch_ex(mp_direct_kernel<H>, dim3(ctas), dim3(kDirThreads), smem, st, 1, a);
}

bool mp_is_direct(int n) { return n <= 2 * kMpDirectMaxH; }
bool mp_is_single(int n) {
    static const int single_max = getenv("FT_SINGLE_MAX") ? atoi(getenv("FT_SINGLE_MAX")) : kMpSingleMaxN;
    return !mp_is_direct(n) && n >= 256 && n <= single_max;
}

// Levels that run the radix-8 high-occupancy kernel (mp8_kernel) instead of mp1g_kernel:
// FT_MP8 = bit mask over log2 n (bit 8 = n 256 ... bit 12 = n 4096); read once.
bool mp8_level(int n) {
    static const int mask = getenv("FT_MP8") ? (int)strtol(getenv("FT_MP8"), nullptr, 0) : FT_MP8_DEFAULT;
    const int lg = __builtin_ctz(n);
    return lg >= 8 && lg <= 12 && ((mask >> lg) & 1);
}

template <int LOGN>
static cudaError_t launch_mp8(const MpArgs& a, cudaStream_t st) {
    using PL = Plan8<LOGN>;
    const size_t smem = sizeof(cplx) * (size_t)(sphys8_len(PL::TILE));
    static DeviceOnce attr_set;
    if (attr_set.first()) {
        cudaFuncSetAttribute(mp8_kernel<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set.done();
    }
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    return launch_ex(mp8_kernel<LOGN>, dim3((npairs + PL::G - 1) / PL::G), dim3(PL::TPB), smem, st, 1, a);
}

template <int LOGN>
static cudaError_t launch_mp1(const MpArgs& a, cudaStream_t st) {
    constexpr int n = 1 << LOGN;
    if constexpr (LOGN <= 12) {
        if (mp8_level(n)) return launch_mp8<LOGN>(a, st);
    }
    constexpr int G = n >= kMpTile ? 1 : kMpTile / n;  // as in mp1_kernel
#ifndef FT_MP1_SMEM_PAD
#define FT_MP1_SMEM_PAD 0
#endif
    const size_t smem = mp_smem_bytes(G, n) + FT_MP1_SMEM_PAD;
    static DeviceOnce attr_set;
    if (attr_set.first()) {
        cudaFuncSetAttribute(mp1_kernel<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set.done();
    }
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    const int ctas = (npairs + G - 1) / G;
    if constexpr (n <= kMpTile) {
        static const bool cta_sync = getenv("FT_MP1_CTA") != nullptr;  // A/B switch
        if (!cta_sync) {
            static DeviceOnce gattr;
            if (gattr.first()) {
                cudaFuncSetAttribute(mp1g_kernel<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                gattr.done();
            }
            // persistent TMA-staged variant (opt-in, FT_MP1P=1: measured slower than the plain
            // launch -- cfg4 388 vs 366 ms, n = 4096 level 3.65 vs 2.89 ms per launch: the CTA
            // barrier per tile re-synchronises the groups and the hardware CTA scheduler already
            // overlaps one CTA's loads with the other's transform); 16-byte aligned row segments
            static const bool tma = getenv("FT_MP1P") != nullptr;
            if (tma && (a.N & 1) == 0 && (a.lo & 1) == 0 && a.mid - a.lo == (uint64_t)(n / 2)) {
                static DeviceOnce pattr;
                const size_t psmem = smem + sizeof(double) * 2 * G * (n / 2) + 16;
                static int slots = 0;
                if (pattr.first()) {
                    cudaFuncSetAttribute(mp1p_kernel<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
                    pattr.done();
                }
                if (slots == 0) {
                    int dev = 0, sms = 0, per = 0;
                    cudaGetDevice(&dev);
                    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mp1p_kernel<LOGN>, kMpThreads, psmem);
                    slots = sms * (per > 0 ? per : 1);
                }
                return launch_ex(mp1p_kernel<LOGN>, dim3(std::min(ctas, slots)), dim3(kMpThreads), psmem, st, 1, a, ctas);
            }
            return launch_ex(mp1g_kernel<LOGN>, dim3(ctas), dim3(kMpThreads), smem, st, 1, a);
        }
    }
    return launch_ex(mp1_kernel<LOGN>, dim3(ctas), dim3(kMpThreads), smem, st, 1, a);
}

template <int LOGN>
static cudaError_t launch_spec1(const double* col, uint64_t N, int B, int J, cplx* spec, const cplx* tw,
                                cudaStream_t st) {
    constexpr int n = 1 << LOGN;
    if constexpr (LOGN <= 12) {
        if (mp8_level(n)) {
            using PL = Plan8<LOGN>;
            const size_t smem8 = sizeof(cplx) * (size_t)(sphys8_len(n));
            static DeviceOnce attr8;
            if (attr8.first()) {
                cudaFuncSetAttribute(spec8_kernel<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8);
                attr8.done();
            }
            spec8_kernel<LOGN><<<B, PL::GT, smem8, st>>>(col, N, J, spec, tw);
            return cudaGetLastError();
        }
    }
    static DeviceOnce attr_set;
    if (attr_set.first()) {
        cudaFuncSetAttribute(spec1_kernel<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mp_smem_bytes(1, n));
        attr_set.done();
    }
    spec1_kernel<LOGN><<<B, kMpThreads, mp_smem_bytes(1, n), st>>>(col, N, J, spec, tw);
    return cudaGetLastError();
}

cudaError_t launch_spectra_single(const double* col, uint64_t N, int B, int n, int J, cplx* spec, const cplx* tw,
                                  cudaStream_t st) {
    switch (n) {
        case 256: return launch_spec1<8>(col, N, B, J, spec, tw, st);
        case 512: return launch_spec1<9>(col, N, B, J, spec, tw, st);
        case 1024: return launch_spec1<10>(col, N, B, J, spec, tw, st);
        case 2048: return launch_spec1<11>(col, N, B, J, spec, tw, st);
        case 4096: return launch_spec1<12>(col, N, B, J, spec, tw, st);
        case 8192: return launch_spec1<13>(col, N, B, J, spec, tw, st);
    }
    return cudaErrorInvalidValue;
}

// Kernels launch_mp issues for this product (split levels: 2 or 3 per pair batch).
int mp_kernel_count(const MpArgs& a) {
    if (mp_is_single(a.n) || mp_is_direct(a.n) || !a.scratch || split_persistent()) return 1;
    static const int prefold_min_k = getenv("FT_PREFOLD_MIN_K") ? atoi(getenv("FT_PREFOLD_MIN_K")) : 16;
    const bool prefold = a.K >= prefold_min_k && getenv("FT_NO_PREFOLD") == nullptr;
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    const int batch = (int)std::max<uint64_t>(1, split_batch_bytes() / ((uint64_t)a.K * a.m * sizeof(cplx)));
    return ((npairs + batch - 1) / batch) * (prefold ? 3 : 2);
}

cudaError_t launch_mp(const MpArgs& a, int groups, cudaStream_t st) {
    if (mp_is_single(a.n)) {
        switch (a.n) {
            case 256: return launch_mp1<8>(a, st);
            case 512: return launch_mp1<9>(a, st);
            case 1024: return launch_mp1<10>(a, st);
            case 2048: return launch_mp1<11>(a, st);
            case 4096: return launch_mp1<12>(a, st);
            case 8192: return launch_mp1<13>(a, st);
        }
    }
    if (mp_is_direct(a.n)) {
        switch (a.n / 2) {
            case 8: return launch_direct_h<8>(a, st);
            case 16: return launch_direct_h<16>(a, st);
            case 32: return launch_direct_h<32>(a, st);
            case 64: return launch_direct_h<64>(a, st);
            case 128: return launch_direct_h<128>(a, st);
        }
    }
    const int key = a.K * 100 + (__builtin_ctz(a.m));
    switch (key) {
        case 212: return launch_mp_k<2, 12>(a, groups, st);
        case 412: return launch_mp_k<4, 12>(a, groups, st);
        case 812: return launch_mp_k<8, 12>(a, groups, st);
        case 1612: return launch_mp_k<16, 12>(a, groups, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_spectra(const double* col, uint64_t N, int B, int n, int m, int K, int J,
                           cplx* spec, const cplx* tw, int logT, cudaStream_t st) {
    static DeviceOnce attr_set;
    if (attr_set.first()) {
        cudaFuncSetAttribute(spectra_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mp_smem_bytes(1, kMpBranchMax));
        attr_set.done();
    }
    SpecArgs a{col, N, n, m, K, J, spec, tw, logT};
    spectra_kernel<<<dim3(K, B), kMpThreads, mp_smem_bytes(1, m), st>>>(a);
    return cudaGetLastError();
}

}  // namespace ftb
