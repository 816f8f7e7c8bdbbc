// leaf.cu -- the leaf of the time-axis divide-and-conquer: L consecutive time
// steps, each one a spatial solve of the step operator, with the in-leaf
// history (lags < L) applied exactly in registers.
//
// Step operator solve: instead of the reference's Thomas
// sweep (src/schemes.cpp:453-461), which is sequential over nodes and loses
// ~1e-10 relative on the cfg4 operator, the constant tridiagonal operator
// d I - b (S + S^T) with Dirichlet ends is inverted through its Green's
// function:  x = G0 (F + B - r) + alpha lam^i + gam lam^(n+1-i)  where F and B
// are forward / backward lam-decay scans of r.  Scans are parallel (thread,
// warp shuffle, cross-warp) and accurate to ~1e-13 on cfg4 (probe in DESIGN.md).
// The upwind operator of Scheme 3 (src/schemes.cpp:345-351) is the forward
// scan alone; the ODE is a scalar divide.
//
// Multi-slab mode (problems larger than one CTA): each CTA owns a contiguous
// slab of nodes and publishes two scan carries per step; every CTA combines
// the carries of all slabs of its problem (cooperative launch, per-step flags).
#include "internal.cuh"

namespace ftb {

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int KIND, int NPT, int L, bool MULTI>
__global__ void __launch_bounds__(kLeafThreads, 1) leaf_kernel(LeafArgs a) {
    __shared__ double s_wt[2][32][2];  // per-warp scan totals (double buffered)
    __shared__ double s_own[2][2];     // padded-slab owner values (F at last node, B at first)
    __shared__ double s_ext[2][2];     // multi-slab EL / ER

    const int cta = blockIdx.x;
    const int pb = cta / a.P, s = cta - pb * a.P;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int nw = blockDim.x >> 5;
    const ProblemConst pc = a.pc[pb];
    const int slab0 = s * a.slab;
    const int mreal = min(a.slab, a.nodes - slab0);
    const bool padded = mreal != (int)blockDim.x * NPT;
    const uint64_t N = a.N;
    const double* colp = a.col + (uint64_t)pb * N;
    const double* lp = a.lampow + (uint64_t)pb * a.lp_stride;
    const int len = a.len;

    double cw[L];
#pragma unroll
    for (int j = 0; j < L; ++j) cw[j] = (j > 0 && (uint64_t)j < N) ? colp[j] : 0.0;

    double tile[NPT][L];
#pragma unroll
    for (int v = 0; v < NPT; ++v) {
        const int q = tid * NPT + v;
        const bool valid = q < mreal;
        const double* src = a.src + (uint64_t)(pb * a.nodes + slab0 + q) * N + a.t0;
#pragma unroll
        for (int k = 0; k < L; ++k) tile[v][k] = (valid && k < len) ? src[k] : 0.0;
    }

    // decay powers
    const double lam = pc.lam;
    double lamq[NPT], lamR[NPT], lamv1[NPT], lamNv[NPT];
#pragma unroll
    for (int v = 0; v < NPT; ++v) {
        const int q = tid * NPT + v;
        lamq[v] = lp[min(q, a.lp_stride - 1)];
        lamR[v] = (q < mreal) ? lp[mreal - 1 - q] : 0.0;
        lamv1[v] = lp[v + 1];
        lamNv[v] = lp[NPT - v];
    }
    double pw[5], pwW[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        pw[d] = lp[min(NPT << d, a.lp_stride - 1)];
        pwW[d] = lp[min((32 * NPT) << d, a.lp_stride - 1)];
    }
    const double lamLaneF = lp[min(NPT * lane, a.lp_stride - 1)];
    const double lamLaneB = lp[min(NPT * (31 - lane), a.lp_stride - 1)];

    // owner of the last real node of the slab
    const int own_t = (mreal - 1) / NPT, own_v = (mreal - 1) - own_t * NPT;

    // multi-slab constants
    const double lamA = MULTI ? lp[min(slab0 + 1, a.lp_stride - 1)] : lam;                   // lam^(a_s)
    const double lamB = MULTI ? lp[min(a.nodes - (slab0 + mreal) + 1, a.lp_stride - 1)] : lam;  // lam^(n+1-b_s)

#pragma unroll
    for (int k = 0; k < L; ++k) {
        if (k >= len) break;
        const int par = k & 1;
        double x[NPT];
        if (KIND == SK_DIAG) {
#pragma unroll
            for (int v = 0; v < NPT; ++v) x[v] = tile[v][k] / pc.d;
        } else {
            // ---- forward scan (both kinds) ----
            double in[NPT];
#pragma unroll
            for (int v = 0; v < NPT; ++v) in[v] = (KIND == SK_UPWIND) ? tile[v][k] / pc.d : tile[v][k];
            double f[NPT];
            double acc = 0.0;
#pragma unroll
            for (int v = 0; v < NPT; ++v) {
                acc = fma(lam, acc, in[v]);
                f[v] = acc;
            }
            double SF = acc;
#pragma unroll
            for (int d = 0; d < 5; ++d) {
                const double y = __shfl_up_sync(0xffffffffu, SF, 1 << d);
                if (lane >= (1 << d)) SF = fma(pw[d], y, SF);
            }
            double exF = __shfl_up_sync(0xffffffffu, SF, 1);
            if (lane == 0) exF = 0.0;
            // ---- backward scan (tridiagonal only) ----
            double bl[NPT];
            double SB = 0.0, exB = 0.0;
            if (KIND == SK_TRIDIAG) {
                double accb = 0.0;
#pragma unroll
                for (int v = NPT - 1; v >= 0; --v) {
                    accb = fma(lam, accb, in[v]);
                    bl[v] = accb;
                }
                SB = accb;
#pragma unroll
                for (int d = 0; d < 5; ++d) {
                    const double y = __shfl_down_sync(0xffffffffu, SB, 1 << d);
                    if (lane + (1 << d) < 32) SB = fma(pw[d], y, SB);
                }
                exB = __shfl_down_sync(0xffffffffu, SB, 1);
                if (lane == 31) exB = 0.0;
            }
            if (lane == 31) s_wt[par][w][0] = SF;
            if (lane == 0) s_wt[par][w][1] = SB;
            __syncthreads();
            // ---- cross-warp carries (every warp redundantly) ----
            double tf = lane < nw ? s_wt[par][lane][0] : 0.0;
            double tb = lane < nw ? s_wt[par][lane][1] : 0.0;
#pragma unroll
            for (int d = 0; d < 5; ++d) {
                const double y = __shfl_up_sync(0xffffffffu, tf, 1 << d);
                if (lane >= (1 << d)) tf = fma(pwW[d], y, tf);
                if (KIND == SK_TRIDIAG) {
                    const double z = __shfl_down_sync(0xffffffffu, tb, 1 << d);
                    if (lane + (1 << d) < nw) tb = fma(pwW[d], z, tb);
                }
            }
            const double CF = w > 0 ? __shfl_sync(0xffffffffu, tf, w - 1) : 0.0;  // F at last node of warp w-1
            const double totF = __shfl_sync(0xffffffffu, tf, nw - 1);             // F at padded end
            double CB = 0.0, totB = 0.0;
            if (KIND == SK_TRIDIAG) {
                CB = (w + 1 < nw) ? __shfl_sync(0xffffffffu, tb, w + 1) : 0.0;
                totB = __shfl_sync(0xffffffffu, tb, 0);
            }
            const double Fprev = fma(lamLaneF, CF, exF);
            double Fv[NPT], Bv[NPT];
#pragma unroll
            for (int v = 0; v < NPT; ++v) Fv[v] = fma(lamv1[v], Fprev, f[v]);
            if (KIND == SK_TRIDIAG) {
                const double Bnext = fma(lamLaneB, CB, exB);
#pragma unroll
                for (int v = 0; v < NPT; ++v) Bv[v] = fma(lamNv[v], Bnext, bl[v]);
            }
            // slab totals: F at the last real node, B at the first node
            double cF = totF, cB = totB;
            if (padded) {
                if (tid == own_t) {
#pragma unroll
                    for (int v = 0; v < NPT; ++v)
                        if (v == own_v) s_own[par][0] = Fv[v];
                }
                __syncthreads();
                cF = s_own[par][0];
            }
            double EL = 0.0, ER = 0.0;
            if (!MULTI) {
                if (KIND == SK_TRIDIAG) {
                    const double p0 = pc.G0 * lam * cB, pM1 = pc.G0 * lam * cF;
                    const double alpha = (pc.Lam * pM1 - p0) * pc.inv1mL2;
                    const double gam = (pc.Lam * p0 - pM1) * pc.inv1mL2;
                    EL = alpha * lam;
                    ER = gam * lam;
                }
            } else {
                // publish this slab's carries, gather every slab's
                const unsigned stepno = a.step_base + (unsigned)k + 1u;
                double* xch = a.xch + (uint64_t)par * gridDim.x * 2;
                if (tid == 0) {
                    xch[2 * cta] = cF;
                    xch[2 * cta + 1] = cB;
                    __threadfence();
                    st_release(&a.flags[cta], stepno);
                }
                if (w == 0) {
                    const int base = pb * a.P;
                    double fin = 0.0, bin = 0.0, fM = 0.0, b1 = 0.0;
                    for (int s2 = lane; s2 < a.P; s2 += 32) {
                        while (ld_acquire(&a.flags[base + s2]) < stepno) {
                        }
                        const double f2 = __ldcg(&xch[2 * (base + s2)]);
                        const double b2 = __ldcg(&xch[2 * (base + s2) + 1]);
                        const int s0 = s2 * a.slab;
                        const int last = min(s0 + a.slab, a.nodes) - 1;
                        if (s2 < s) fin = fma(lp[slab0 - 1 - last], f2, fin);
                        if (s2 > s) bin = fma(lp[s0 - (slab0 + mreal)], b2, bin);
                        if (KIND == SK_TRIDIAG) {
                            fM = fma(lp[a.nodes - 1 - last], f2, fM);
                            b1 = fma(lp[s0], b2, b1);
                        }
                    }
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) {
                        fin += __shfl_xor_sync(0xffffffffu, fin, o);
                        bin += __shfl_xor_sync(0xffffffffu, bin, o);
                        fM += __shfl_xor_sync(0xffffffffu, fM, o);
                        b1 += __shfl_xor_sync(0xffffffffu, b1, o);
                    }
                    if (lane == 0) {
                        if (KIND == SK_TRIDIAG) {
                            const double p0 = pc.G0 * lam * b1, pM1 = pc.G0 * lam * fM;
                            const double alpha = (pc.Lam * pM1 - p0) * pc.inv1mL2;
                            const double gam = (pc.Lam * p0 - pM1) * pc.inv1mL2;
                            s_ext[par][0] = pc.G0 * lam * fin + alpha * lamA;
                            s_ext[par][1] = pc.G0 * lam * bin + gam * lamB;
                        } else {
                            s_ext[par][0] = lam * fin;
                            s_ext[par][1] = 0.0;
                        }
                    }
                }
                __syncthreads();
                EL = s_ext[par][0];
                ER = s_ext[par][1];
            }
#pragma unroll
            for (int v = 0; v < NPT; ++v) {
                if (KIND == SK_TRIDIAG)
                    x[v] = fma(pc.G0, Fv[v] + Bv[v] - tile[v][k], fma(EL, lamq[v], ER * lamR[v]));
                else
                    x[v] = fma(EL, lamq[v], Fv[v]);
            }
        }
        // in-leaf history: push x into the remaining steps of the leaf (padding
        // nodes beyond the slab stay exactly zero)
#pragma unroll
        for (int v = 0; v < NPT; ++v) {
            if (tid * NPT + v >= mreal) x[v] = 0.0;
            tile[v][k] = x[v];
#pragma unroll
            for (int k2 = k + 1; k2 < L; ++k2) tile[v][k2] = fma(-cw[k2 - k], x[v], tile[v][k2]);
        }
    }

#pragma unroll
    for (int v = 0; v < NPT; ++v) {
        const int q = tid * NPT + v;
        if (q < mreal) {
            double* dst = a.X + (uint64_t)(pb * a.nodes + slab0 + q) * N + a.t0;
#pragma unroll
            for (int k = 0; k < L; ++k)
                if (k < len) dst[k] = tile[v][k];
        }
    }
}

// ---- host launch -------------------------------------------------------------

template <int KIND, int NPT, int L, bool MULTI>
static cudaError_t launch_leaf_t(const LeafArgs& a, int ctas, int threads, cudaStream_t st) {
    if (MULTI) {
        void* args[] = {(void*)&a};
        return cudaLaunchCooperativeKernel((const void*)leaf_kernel<KIND, NPT, L, MULTI>, dim3(ctas),
                                           dim3(threads), args, 0, st);
    }
    leaf_kernel<KIND, NPT, L, MULTI><<<ctas, threads, 0, st>>>(a);
    return cudaGetLastError();
}

// Supported (NPT, L) pairs: tile of NPT*L doubles per thread.
cudaError_t launch_leaf(int kind, int npt, int L, bool multi, const LeafArgs& a, int ctas,
                        int threads, cudaStream_t st) {
#define FTB_LEAF_CASE(K_, NPT_, L_)                                                      \
    if (kind == K_ && npt == NPT_ && L == L_)                                             \
        return multi ? launch_leaf_t<K_, NPT_, L_, true>(a, ctas, threads, st)            \
                     : launch_leaf_t<K_, NPT_, L_, false>(a, ctas, threads, st);
    FTB_LEAF_CASE(SK_DIAG, 1, 32)
    FTB_LEAF_CASE(SK_TRIDIAG, 1, 32)
    FTB_LEAF_CASE(SK_TRIDIAG, 2, 32)
    FTB_LEAF_CASE(SK_TRIDIAG, 4, 16)
    FTB_LEAF_CASE(SK_TRIDIAG, 8, 8)
    FTB_LEAF_CASE(SK_UPWIND, 1, 32)
    FTB_LEAF_CASE(SK_UPWIND, 2, 32)
    FTB_LEAF_CASE(SK_UPWIND, 4, 16)
    FTB_LEAF_CASE(SK_UPWIND, 8, 8)
#undef FTB_LEAF_CASE
    return cudaErrorInvalidValue;
}

}  // namespace ftb
