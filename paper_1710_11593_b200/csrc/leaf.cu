// leaf.cu -- the leaf of the time-axis divide-and-conquer: L consecutive time
// steps, each a spatial solve of the step operator, with the in-leaf history
// (lags < L) applied exactly in registers.
//
// Step operator solve: instead of the reference's Thomas
// sweep (src/schemes.cpp:453-461), sequential over nodes and ~1e-10 relative
// off on the cfg4 operator, the constant tridiagonal operator
// d I - b (S + S^T) with Dirichlet ends is inverted through its Green's
// function   x = G0 (F + B - r) + alpha lam^i + gam lam^(n+1-i)   where F and B
// are forward / backward lam-decay scans of r (thread, warp shuffle,
// cross-warp).  The upwind operator of Scheme 3 (src/schemes.cpp:345-351) is the
// forward scan alone; the ODE is a scalar divide.
//
// Problems wider than one CTA are split into slabs (one CTA each) and solved
// in three phases per leaf, with ONE cross-CTA exchange per leaf instead of
// one per step (space-time SPIKE):
//   1 (leaf_kernel<..., LOCAL>) every slab marches L steps with zero
//     inter-slab carries, recording the two carries it would export per step;
//   2 (leaf_correct) every CTA replays the small reduced recursion over all
//     slabs' carries (lag responses h*), giving its own slab's injections
//     EL_k, ER_k;
//   3 (leaf_correct) the slab's solution is corrected with precomputed
//     space-time response tables GL, GR: x += sum_l GL(l) EL_(k-l) + GR(l) ER_(k-l).
#include <mutex>

#include "internal.cuh"

#ifndef FT_LEAF_WREG
#define FT_LEAF_WREG 0  // 1: batched plans copy the in-leaf weights into registers (old path)
#endif
#ifndef FT_LEAF_UNROLL
#define FT_LEAF_UNROLL 1  // step-loop unroll: 1 measured 403 ms vs 408 (2) and 412 (4) on cfg4 (instruction fetch)
#endif

namespace ftb {

constexpr int kLeafUnroll = FT_LEAF_UNROLL;
#ifndef FT_STAGE_U
#define FT_STAGE_U 8
#endif
constexpr int kStageU = FT_STAGE_U;  // 16-byte loads in flight per thread staging a leaf tile
                                     // (16: cfg4 +3 ms -- the 128 CTAs staging at once are HBM-bound)

// in-leaf history weights col[1..L) of batched plans (B > 1), read through the
// constant cache with a CTA-uniform index (measured: config 5 97.2 -> 92.3 ms vs
// registers, ~95 ms through __ldg).  One bank per device, shared by every plan:
// leaf_bank_acquire / _release (below) give it to one plan at a time in stream
// order, so concurrent plans on distinct streams never read each other's weights.
// (Single-problem plans pass their weights as kernel parameters, LeafArgs::kc.)
__constant__ double c_leafcol[kMaxLeafProblems][32];


template <int NPT>
struct ScanConsts {
    double lam;
    double pwF[5], pwB[5];  // masked lane multipliers lam^(NPT 2^d) (0 where the partner is out of range)
    double lamv1[NPT], lamNv[NPT];
    double lamLaneF, lamLaneB, lamW;  // lam^(NPT lane), lam^(NPT (31-lane)), lam^(32 NPT)
    double exFmask, exBmask;
};

template <int NPT>
__device__ __forceinline__ void scan_consts(ScanConsts<NPT>& sc, const double* lp, int lp_stride, double lam,
                                            int lane) {
    sc.lam = lam;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const double p = lp[min(NPT << d, lp_stride - 1)];
        sc.pwF[d] = lane >= (1 << d) ? p : 0.0;
        sc.pwB[d] = lane + (1 << d) < 32 ? p : 0.0;
    }
#pragma unroll
    for (int v = 0; v < NPT; ++v) {
        sc.lamv1[v] = lp[v + 1];
        sc.lamNv[v] = lp[NPT - v];
    }
    sc.lamLaneF = lp[min(NPT * lane, lp_stride - 1)];
    sc.lamLaneB = lp[min(NPT * (31 - lane), lp_stride - 1)];
    sc.lamW = lp[min(32 * NPT, lp_stride - 1)];
    sc.exFmask = lane > 0 ? 1.0 : 0.0;
    sc.exBmask = lane < 31 ? 1.0 : 0.0;
}

// Leaf constants seen through one interface.  PC = false: per-problem values
// (constant-memory leaf weights, lam^k table) loaded into registers.  PC = true
// (single-problem plans): the kernel-parameter copy LeafArgs::kc, read as
// constant-bank operands -- no registers for the 31 weights and the uniform
// scan multipliers, only the two lane-dependent powers (the register file of
// the 255-register step loop otherwise spills, ncu).
template <bool PC, int NPT, int L>
struct LeafConsts;

template <int NPT, int L>
struct LeafConsts<false, NPT, L> {
    ScanConsts<NPT> sc;
#if FT_LEAF_WREG
    double w[L];
#else
    const double* w;  // this problem's row of c_leafcol: read per use through the constant cache
                      // (CTA-uniform index; 31 weights in registers spilled)
#endif
    __device__ __forceinline__ LeafConsts(const LeafArgs& a, int pb, const double* lp, double lam, int lane) {
        scan_consts<NPT>(sc, lp, a.lp_stride, lam, lane);
        const double* cc = c_leafcol[pb < kMaxLeafProblems ? pb : 0];
#if FT_LEAF_WREG
#pragma unroll
        for (int j = 0; j < L; ++j) w[j] = cc[j];
#else
        w = cc;
#endif
    }
    __device__ __forceinline__ double cw(int j) const { return w[j]; }
    __device__ __forceinline__ double lam() const { return sc.lam; }
    __device__ __forceinline__ double stepF(int d, double y, double S, int) const { return fma(sc.pwF[d], y, S); }
    __device__ __forceinline__ double stepB(int d, double y, double S, int) const { return fma(sc.pwB[d], y, S); }
    __device__ __forceinline__ double exF(double y, int) const { return sc.exFmask * y; }
    __device__ __forceinline__ double exB(double y, int) const { return sc.exBmask * y; }
    __device__ __forceinline__ double lamW() const { return sc.lamW; }
    __device__ __forceinline__ double lamv1(int v) const { return sc.lamv1[v]; }
    __device__ __forceinline__ double lamNv(int v) const { return sc.lamNv[v]; }
    __device__ __forceinline__ double laneF() const { return sc.lamLaneF; }
    __device__ __forceinline__ double laneB() const { return sc.lamLaneB; }
};

template <int NPT, int L>
struct LeafConsts<true, NPT, L> {
    const LeafArgs& a;
    double lamLaneF, lamLaneB;
    double pwF[5], pwB[5];  // lane-masked shuffle-scan multipliers (0 where the partner is out of range):
                            // one DFMA per round instead of DFMA + two selects
    __device__ __forceinline__ LeafConsts(const LeafArgs& a_, int, const double* lp, double, int lane) : a(a_) {
        lamLaneF = lp[min(NPT * lane, a.lp_stride - 1)];
        lamLaneB = lp[min(NPT * (31 - lane), a.lp_stride - 1)];
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            pwF[d] = lane >= (1 << d) ? a.kc[kKcPow + d] : 0.0;
            pwB[d] = lane + (1 << d) < 32 ? a.kc[kKcPow + d] : 0.0;
        }
    }
    __device__ __forceinline__ double cw(int j) const { return a.kc[j]; }
    __device__ __forceinline__ double lam() const { return a.kc[kKcLam]; }
    __device__ __forceinline__ double stepF(int d, double y, double S, int) const { return fma(pwF[d], y, S); }
    __device__ __forceinline__ double stepB(int d, double y, double S, int) const { return fma(pwB[d], y, S); }
    __device__ __forceinline__ double exF(double y, int lane) const { return lane > 0 ? y : 0.0; }
    __device__ __forceinline__ double exB(double y, int lane) const { return lane < 31 ? y : 0.0; }
    __device__ __forceinline__ double lamW() const { return a.kc[kKcLamW]; }
    __device__ __forceinline__ double lamv1(int v) const { return a.kc[kKcV1 + v]; }
    __device__ __forceinline__ double lamNv(int v) const { return a.kc[kKcNv + v]; }
    __device__ __forceinline__ double laneF() const { return lamLaneF; }
    __device__ __forceinline__ double laneB() const { return lamLaneB; }
};

// dst[q][k] (row stride L+1) = src[(row0 + q) * N + t0 + k] for q < rows, k < len;
// consecutive threads read consecutive steps of a node row, 8 loads in flight.
// radd (optional, same layout as src): added element-wise -- the streamed host
// path keeps the caller's R out of X until the leaf that solves those steps.
// sub (vector path only): dst holds values to subtract -- dst = src - dst (the leaf-pair
// kernel leaves the level-0 history product of the previous leaf there).
template <int L, bool LEAN = false>
__device__ __forceinline__ void stage_rows(double* dst, const double* src, const double* radd, uint64_t row0,
                                           uint64_t N, uint64_t t0, int rows, int len, bool sub = false) {
    // 16-byte loads when rows are 16-byte aligned and whole (the common case:
    // even N, full leaf); kStageU double2 in flight per thread.  LEAN (host-checked:
    // even N, full leaves, no radd): only this path is compiled.
    if (LEAN) radd = nullptr;
    if (LEAN || (len == L && (N & 1) == 0 && (t0 & 1) == 0)) {
        constexpr int HL = L / 2;
        const int total = rows * HL;
        for (int e0 = 0; e0 < total; e0 += kStageU * kLeafThreads) {
            double2 v[kStageU];
#pragma unroll
            for (int u = 0; u < kStageU; ++u) {
                const int e = e0 + u * kLeafThreads + threadIdx.x;
                const int q = e / HL, k2 = e - q * HL;
                v[u] = (e < total && src) ? __ldcg(reinterpret_cast<const double2*>(src + (row0 + q) * N + t0) + k2)
                                          : make_double2(0.0, 0.0);
            }
            if (radd) {
#pragma unroll
                for (int u = 0; u < kStageU; ++u) {
                    const int e = e0 + u * kLeafThreads + threadIdx.x;
                    const int q = e / HL, k2 = e - q * HL;
                    if (e < total) {
                        const double2 r = __ldcs(reinterpret_cast<const double2*>(radd + (row0 + q) * N + t0) + k2);
                        v[u].x += r.x;
                        v[u].y += r.y;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kStageU; ++u) {
                const int e = e0 + u * kLeafThreads + threadIdx.x;
                const int q = e / HL, k2 = e - q * HL;
                if (e < total) {
                    double* d = dst + q * (L + 1) + 2 * k2;
                    if (sub) {
                        d[0] = v[u].x - d[0];
                        d[1] = v[u].y - d[1];
                    } else {
                        d[0] = v[u].x;
                        d[1] = v[u].y;
                    }
                }
            }
        }
        return;
    }
    const int total = rows * len;
    for (int e0 = 0; e0 < total; e0 += 8 * kLeafThreads) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * kLeafThreads + threadIdx.x;
            const int q = e / len, k = e - q * len;
            v[u] = e < total ? (src ? src[(row0 + q) * N + t0 + k] : 0.0) + (radd ? radd[(row0 + q) * N + t0 + k] : 0.0)
                             : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * kLeafThreads + threadIdx.x;
            const int q = e / len, k = e - q * len;
            if (e < total) dst[q * (L + 1) + k] = v[u];
        }
    }
}

// X[row0 + q][t0 + k] = src[q][k] (row stride L+1), 16-byte stores when aligned
template <int L, bool LEAN = false>
__device__ __forceinline__ void store_rows(double* X, const double* src, uint64_t row0, uint64_t N, uint64_t t0,
                                           int rows, int len, int tid, int nth) {
    if (LEAN || (len == L && (N & 1) == 0 && (t0 & 1) == 0)) {
        constexpr int HL = L / 2;
        for (int e = tid; e < rows * HL; e += nth) {
            const int q = e / HL, k2 = e - q * HL;
            const double2 v = make_double2(src[q * (L + 1) + 2 * k2], src[q * (L + 1) + 2 * k2 + 1]);
            reinterpret_cast<double2*>(X + (row0 + q) * N + t0)[k2] = v;
        }
        return;
    }
    for (int e = tid; e < rows * len; e += nth) {
        const int q = e / len, k = e - q * len;
        X[(row0 + q) * N + t0 + k] = src[q * (L + 1) + k];
    }
}

// Forward (and, for TRIDIAG, backward) lam-decay scans over the CTA's nodes
// with zero carry in at both ends.  Fv/Bv: scans at this thread's nodes;
// totF: F at the CTA's last (possibly padding) node; totB: B at its first.
// FULL = true: every thread gets totF / totB (single-CTA mode, Dirichlet
// correction).  FULL = false (slab mode): warp w chains only the warp totals it
// needs, as warp-uniform predicated DFMAs (same order, so bitwise the same
// carries; no selects): totF is the CTA total in the last warp, totB in warp 0
// -- their only consumers are the exported slab carries.
template <int KIND, int NPT, bool FULL, class SC>
__device__ __forceinline__ void cta_scan(const double (&in)[NPT], const SC& sc,
                                         double (*s_wt)[2], int lane, int w, double (&Fv)[NPT],
                                         double (&Bv)[NPT], double& totF, double& totB, double& Fpv) {
    constexpr int nw = kLeafThreads / 32;
    constexpr bool TRI = KIND == SK_TRIDIAG;
    double f[NPT], bl[NPT];
    double acc = in[0];  // (no 0 * lam + in on the step's critical path)
    f[0] = acc;
#pragma unroll
    for (int v = 1; v < NPT; ++v) {
        acc = fma(sc.lam(), acc, in[v]);
        f[v] = acc;
    }
    double SF = acc, SB = 0.0;
    if (TRI) {
        double accb = in[NPT - 1];
        bl[NPT - 1] = accb;
#pragma unroll
        for (int v = NPT - 2; v >= 0; --v) {
            accb = fma(sc.lam(), accb, in[v]);
            bl[v] = accb;
        }
        SB = accb;
    }
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const double yF = __shfl_up_sync(0xffffffffu, SF, 1 << d);
        SF = sc.stepF(d, yF, SF, lane);
        if (TRI) {
            const double yB = __shfl_down_sync(0xffffffffu, SB, 1 << d);
            SB = sc.stepB(d, yB, SB, lane);
        }
    }
    const double exF = sc.exF(__shfl_up_sync(0xffffffffu, SF, 1), lane);
    const double exB = TRI ? sc.exB(__shfl_down_sync(0xffffffffu, SB, 1), lane) : 0.0;
    if (lane == 31) s_wt[w][0] = SF;
    if (lane == 0) s_wt[w][1] = SB;
    __syncthreads();
    // cross-warp carries: short sequential chains over the 8 warp totals
    double CF = 0.0, CB = 0.0;
    if constexpr (FULL) {
        double runF = 0.0, runB = 0.0;
#pragma unroll
        for (int ww = 0; ww < nw; ++ww) {
            if (ww == w) CF = runF;
            runF = fma(sc.lamW(), runF, s_wt[ww][0]);
            if (TRI) {
                const int wb = nw - 1 - ww;
                if (wb == w) CB = runB;
                runB = fma(sc.lamW(), runB, s_wt[wb][1]);
            }
        }
        totF = runF;
        totB = runB;
    } else {
#pragma unroll
        for (int ww = 0; ww < nw; ++ww)
            if (ww < w) CF = fma(sc.lamW(), CF, s_wt[ww][0]);
        if (TRI) {
#pragma unroll
            for (int wb = nw - 1; wb >= 0; --wb)
                if (wb > w) CB = fma(sc.lamW(), CB, s_wt[wb][1]);
        }
        totF = fma(sc.lamW(), CF, s_wt[w][0]);
        totB = TRI ? fma(sc.lamW(), CB, s_wt[w][1]) : 0.0;
    }
    const double Fprev = fma(sc.laneF(), CF, exF);
    Fpv = Fprev;  // F at the node before this thread's first node (0 before node 0)
#pragma unroll
    for (int v = 0; v < NPT; ++v) Fv[v] = fma(sc.lamv1(v), Fprev, f[v]);
    if (TRI) {
        const double Bnext = fma(sc.laneB(), CB, exB);
#pragma unroll
        for (int v = 0; v < NPT; ++v) Bv[v] = fma(sc.lamNv(v), Bnext, bl[v]);
    }
}

// Level-0 history product (n = 64) of the previous leaf onto the next one, per node row of
// the calling thread: row[k] := sum_j col[32 + k - j] row[j] (lags 1..63), in place in the
// thread's own rows of s_out (which hold the previous leaf's U).  Rolled over output chunks
// (instruction footprint): the weights are constant-bank operands at a CTA-uniform runtime
// offset (kc[0 .. 2L) holds lags 0 .. 2L-1).
template <int NPT, int L>
__device__ __forceinline__ void level0_rows(const LeafArgs& a, double* s_out, int tid, int mreal) {
#pragma unroll 1
    for (int v = 0; v < NPT; ++v) {
        const int q = tid * NPT + v;
        if (q >= mreal) continue;
        double* row = s_out + q * (L + 1);
        double u[L];
#pragma unroll
        for (int jj = 0; jj < L; ++jj) u[jj] = row[jj];
        // 8 outputs at a time: each output sums jj ascending (bitwise equal to the
        // standalone direct product) with 8 independent FMA chains in flight
#pragma unroll 1
        for (int k0 = 0; k0 < L; k0 += 8) {
            const double* wp = a.kc + L + k0;  // wp[kk - jj]: weight of lag L + k0 + kk - jj
            double acc[8];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) acc[kk] = 0.0;
#pragma unroll
            for (int jj = 0; jj < L; ++jj) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) acc[kk] = fma(wp[kk - jj], u[jj], acc[kk]);
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) row[k0 + kk] = acc[kk];
        }
    }
}

// MODE 0 (SINGLE): the CTA spans the whole problem; the Dirichlet correction
//   x += kF_i F_M + kB_i B_1 (host-precomputed per node) makes the step exact.
// MODE 1 (LOCAL): phase 1 of the slab decomposition (zero inter-slab carries);
//   per step the slab's exported carries (F at its last node, B at its first)
//   are written to xch[cta][k][2].
// LEAN (host-checked in launch_fused_t: even N, full leaf, no radd / fused RHS / Scheme-2
// stencil): the generic staging, forcing and V paths are compiled out.  The slab leaf's code
// must stay inside the SM's 64 KB of instruction cache: ncu showed every instruction past
// that mark stalling on instruction fetch (30 % of the leaf's warp samples at 150 KB).
// PAIR (leaf_pair kernel): half = 1 is the second leaf of a pair whose first leaf's solution
// is still in s_out: the level-0 product is formed there and the staged R subtracts it.
// Chained upwind slabs (MODE 2): one 16-byte {value, tag} record per slab and step; a single
// vector store / load, so the tag never arrives without its value.  Relaxed gpu-scope accesses
// (a weak load in the wait loop may legally be hoisted by ptxas: it hung).
__device__ __forceinline__ double2 chain_load(const double2* p) {
    double2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void chain_store(double2* p, double x, double tag) {
    asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(x), "d"(tag));
}

// MODE 0: single slab (closed-form Dirichlet images); MODE 1: space-time SPIKE phase 1 (zero
// inter-slab carries, carries exported); MODE 2: chained upwind slabs -- the operator is lower
// bidiagonal in space, so slab s only needs the solution at the last node of slab s - 1 at the
// same step: it runs a step or two behind its left neighbour and adds lam^(q+1) x_left to its
// own scan, exactly (no correction phase, no grid barrier).
template <int KIND, int NPT, int L, int MODE, bool PC = false, bool LEAN = false, bool PAIR = false>
__device__ __forceinline__ void leaf_body(const LeafArgs& a, double* s_out, bool write_x, int half = 0) {
    // s_out: [slab nodes][L + 1] solution tile (stays resident for the fused leaf)
    __shared__ double s_wt[2][32][2];
    __shared__ double s_own[2];
    __shared__ double s_cx[L][2];

    const int cta = blockIdx.x;
    const int pb = cta / a.P_local, s = a.s_begin + (cta - pb * a.P_local);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const ProblemConst pc = a.pc[pb];
    const int slab0 = s * a.slab;
    const int mreal = min(a.slab, a.nodes - slab0);
    const uint64_t rowb = (uint64_t)pb * a.rows_pp + (slab0 - a.node_begin);  // X row of node slab0
    const bool padded = mreal != (int)blockDim.x * NPT;
    const uint64_t N = a.N;
    const double* colp = a.col + (uint64_t)pb * N;
    const double* lp = a.lampow + (uint64_t)pb * a.lp_stride;
    const int len = LEAN ? L : a.len;
    const uint64_t t0 = a.t0 + (PAIR ? (uint64_t)half * L : 0);

    (void)colp;

    // (chained slabs: the last slab is the critical path)
    const bool stamp = a.dbg_clk && blockIdx.x == ((MODE == 2 && !(a.dbg & 8)) ? gridDim.x - 1 : 0) && threadIdx.x == 0;
    const LeafConsts<PC, NPT, L> sc(a, pb, lp, pc.lam, lane);  // plan constants: before the dependency wait
    if (!PAIR || half == 0) pdl_wait();
    if (stamp) a.dbg_clk[8] = clock64();
    if (PAIR && half) {
        __syncthreads();  // the store of the first leaf's solution has read every row
        level0_rows<NPT, L>(a, s_out, tid, mreal);
        __syncthreads();
        if (stamp) a.dbg_clk[5] = clock64();
    }
    // input tile: coalesced row reads (a warp reads consecutive steps of one
    // node) staged through shared memory, then into the register window
    stage_rows<L, LEAN>(s_out, (PAIR && half) ? a.src2 : a.src, a.radd, rowb, N, t0, mreal, len, PAIR && half);
    __syncthreads();
    if (stamp) a.dbg_clk[15] = clock64();
    double tile[NPT][L];
#pragma unroll
    for (int v = 0; v < NPT; ++v) {
        const int q = tid * NPT + v;
        const bool valid = q < mreal;
#pragma unroll
        for (int k = 0; k < L; ++k) tile[v][k] = (valid && k < len) ? s_out[q * (L + 1) + k] : 0.0;
    }
    if constexpr (PC && MODE == 1 && !PAIR) {
        if (a.fuse0) {
            // level-0 history product (n = 64) of the previous leaf onto this one:
            // tile[v][k] -= sum_j col[32 + k - j] U[row][t0 - 32 + j] (lags 1..63), with the
            // previous leaf's U staged through s_out (free until the step loop writes it);
            // the sums go back to the thread's own rows and are subtracted from the window.
            __syncthreads();
            stage_rows<L, LEAN>(s_out, a.X, nullptr, rowb, N, t0 - L, mreal, L);
            __syncthreads();
            if (stamp) a.dbg_clk[5] = clock64();
            level0_rows<NPT, L>(a, s_out, tid, mreal);
            // (own rows only: no barrier)
#pragma unroll
            for (int v = 0; v < NPT; ++v) {
                const int q = tid * NPT + v;
                if (q < mreal) {
#pragma unroll
                    for (int k = 0; k < L; ++k) tile[v][k] -= s_out[q * (L + 1) + k];
                }
            }
        }
    }
    if (!LEAN && a.genA) {
        // fused separable RHS (ft_solve_fast_modes): tile += sum_j A[row][j] T[pb][t][j]
        // straight into the register window; T is warp-uniform (broadcast loads)
        const int J = a.genJ;
        const double* Tb = a.genT + ((uint64_t)pb * N + t0) * J;
        constexpr int kMaxJ = 16;
        __shared__ double s_T[kMaxJ][L];  // this leaf's step factors, [j][k] (broadcast reads)
        for (int e = tid; e < kMaxJ * L; e += blockDim.x) {
            const int j = e / L, k = e - j * L;
            s_T[j][k] = (j < J && k < len) ? __ldg(&Tb[(uint64_t)k * J + j]) : 0.0;
        }
        __syncthreads();
#pragma unroll 1
        for (int j = 0; j < J; ++j) {
            double av[NPT];
#pragma unroll
            for (int v = 0; v < NPT; ++v) {
                const int q = tid * NPT + v;
                av[v] = q < mreal ? __ldg(&a.genA[(rowb + q) * J + j]) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < L; k += 2) {
                const double2 t2 = *reinterpret_cast<const double2*>(&s_T[j][k]);
#pragma unroll
                for (int v = 0; v < NPT; ++v) {
                    tile[v][k] = fma(av[v], t2.x, tile[v][k]);
                    tile[v][k + 1] = fma(av[v], t2.y, tile[v][k + 1]);
                }
            }
        }
    }
    __syncthreads();
    if (stamp) a.dbg_clk[9] = clock64();
    // Dirichlet correction coefficients (SINGLE mode)
    double kF[NPT], kB[NPT];
#pragma unroll
    for (int v = 0; v < NPT; ++v) {
        const int q = tid * NPT + v;
        const bool valid = q < mreal;
        kF[v] = (MODE == 0 && KIND == SK_TRIDIAG && valid) ? a.kcoef[(uint64_t)pb * 2 * a.nodes + q] : 0.0;
        kB[v] = (MODE == 0 && KIND == SK_TRIDIAG && valid) ? a.kcoef[(uint64_t)pb * 2 * a.nodes + a.nodes + q] : 0.0;
    }
    const int own_t = (mreal - 1) / NPT, own_v = (mreal - 1) - own_t * NPT;
    double vmask[NPT];
#pragma unroll
    for (int v = 0; v < NPT; ++v) vmask[v] = (tid * NPT + v < mreal) ? 1.0 : 0.0;
    double* outp = s_out + tid * NPT * (L + 1);
    // chained upwind slabs: lam^(q+1) per node, the neighbour's record of the next step in flight
    double lq[NPT];
    const bool chain_in = MODE == 2 && s > 0, chain_out = MODE == 2 && s + 1 < a.P;
    const double2* cin_p = MODE == 2 ? a.chain + ((uint64_t)pb * a.P + (s > 0 ? s - 1 : 0)) * L : nullptr;
    double2* cout_p = MODE == 2 ? a.chain + ((uint64_t)pb * a.P + s) * L : nullptr;
    // (two records in flight: the load of step k + 2 is issued during step k, ~2 steps before its
    // use -- an L2 round trip to a line another SM just wrote is most of a step)
    double2 cnx = make_double2(0.0, 0.0), cnx1 = make_double2(0.0, 0.0);
    if (MODE == 2) {
#pragma unroll
        for (int v = 0; v < NPT; ++v) lq[v] = lp[min(tid * NPT + v + 1, a.lp_stride - 1)];
        if (chain_in) {  // every lane of every warp polls the same record (one transaction per warp): the
                         // wait loop below is warp-uniform by a vote, so the scan's shuffles stay convergent
                         // (a thread-0-only wait loop sent them through WARPSYNC.COLLECTIVE: +250 cycles per step)
            cnx = chain_load(cin_p);
            cnx1 = chain_load(cin_p + (len > 1 ? 1 : 0));
        }
    }
    // Rolling window: tile[v][i] holds the right-hand side of step k + i; each
    // step shifts it down by one register while pushing the new solution into
    // the remaining in-leaf steps (no unrolling over k: the body stays small
    // enough for the instruction cache -- unrolling by 2 or 4 measured slower).
#pragma unroll kLeafUnroll
    for (int k = 0; k < len; ++k) {
        const int par = k & 1;
        double x[NPT];
        double xleft = 0.0;  // upwind: solution at the node left of this thread's first node
        if (KIND == SK_DIAG) {
#pragma unroll
            for (int v = 0; v < NPT; ++v) x[v] = tile[v][0] * pc.G0;  // G0 = 1/d (a DDIV is ~430 cycles)
        } else {
            double in[NPT];
#pragma unroll
            // upwind: r / d as r * (1/d) -- a division on the step's critical path costs ~430 cycles
            // on B200 (measured), the product 8; same rounding model as the host tables (local_solve_ld)
            for (int v = 0; v < NPT; ++v) in[v] = (KIND == SK_UPWIND) ? tile[v][0] * pc.G0 : tile[v][0];
            double Fv[NPT], Bv[NPT], totF, totB;
            double cin = 0.0;
            if (MODE == 2 && chain_in) {  // the left slab's boundary value of this step (normally already here)
                while (__any_sync(0xffffffffu, cnx.y != a.chain_tag)) cnx = chain_load(cin_p + k);
                cin = cnx.x;
                cnx = cnx1;  // rotate; the record of step k + 2 goes in flight
                if (k + 2 < len) cnx1 = chain_load(cin_p + k + 2);
            }
            cta_scan<KIND, NPT, MODE == 0>(in, sc, s_wt[par], lane, w, Fv, Bv, totF, totB, xleft);
            double cF = totF;
            if (MODE != 2 && padded) {  // F at the last real node (padding nodes carry zeros)
                if (tid == own_t) {
#pragma unroll
                    for (int v = 0; v < NPT; ++v)
                        if (v == own_v) s_own[par] = Fv[v];
                }
                __syncthreads();
                cF = s_own[par];
            }
            if (MODE == 1) {  // exported carries: F at the slab's last node, B at its first
                if (padded ? tid == 0 : (w == kLeafThreads / 32 - 1 && lane == 31)) s_cx[k][0] = cF;
                if (tid == 0) s_cx[k][1] = totB;
            }
#pragma unroll
            for (int v = 0; v < NPT; ++v) {
                if (KIND == SK_TRIDIAG) {
                    const double base = pc.G0 * (Fv[v] + Bv[v] - in[v]);
                    x[v] = MODE == 0 ? fma(kF[v], cF, fma(kB[v], totB, base)) : base;
                } else {
                    x[v] = MODE == 2 ? fma(lq[v], cin, Fv[v]) : Fv[v];
                }
            }
        }
#pragma unroll
        for (int v = 0; v < NPT; ++v) {
            if (padded) x[v] *= vmask[v];  // padding nodes stay exactly zero
            outp[v * (L + 1)] = x[v];
        }
        if (MODE == 2 && chain_out && tid == own_t) {  // this slab's last node: the right neighbour's input
#pragma unroll
            for (int v = 0; v < NPT; ++v)
                if (v == own_v) chain_store(cout_p + k, x[v], a.chain_tag);
        }
        // Scheme 2: the history acts on U_i + U_(i-1) (the left neighbour's solution)
        double xs[NPT];
#pragma unroll
        for (int v = 0; v < NPT; ++v)  // (compile-time false for the tridiagonal operator: x stays on the fast path)
            xs[v] = (KIND == SK_UPWIND && !LEAN && a.stencil) ? x[v] + (v > 0 ? x[v - 1] : xleft) : x[v];
        // push x_k into the remaining in-leaf steps; chunks whose first entry lies past
        // the leaf end (k + 1 + c >= len) are dead and skipped (one warp-uniform test per chunk)
#pragma unroll
        for (int c = 0; c + 1 < L; c += 8) {
            if (c == 0 || k + 1 + c < len) {
#pragma unroll
                for (int v = 0; v < NPT; ++v)
#pragma unroll
                    for (int i = c; i < c + 8 && i + 1 < L; ++i) tile[v][i] = fma(-sc.cw(i + 1), xs[v], tile[v][i + 1]);
            }
        }
#pragma unroll
        for (int v = 0; v < NPT; ++v) tile[v][L - 1] = 0.0;
        ++outp;
    }

    __syncthreads();
    if (stamp) a.dbg_clk[10] = clock64();
    // coalesced store of the solution tile: consecutive threads write consecutive steps of a row
    if (write_x) store_rows<L, LEAN>(a.X, s_out, rowb, N, t0, mreal, len, tid, blockDim.x);
    if (!LEAN && MODE == 0 && a.V) {  // Scheme 2 product sources V = U_i + U_(i-1) (single-slab problems)
        for (int e = tid; e < mreal * len; e += blockDim.x) {
            const int q = e / len, k = e - q * len;
            const double up = q > 0 ? s_out[(q - 1) * (L + 1) + k] : 0.0;
            a.V[(rowb + q) * N + t0 + k] = s_out[q * (L + 1) + k] + up;
        }
    }
    if (MODE == 1) {
        double* xo = a.xsend + (uint64_t)cta * L * 2 + (PAIR ? (uint64_t)half * gridDim.x * L * 2 : 0);
        for (int i = tid; i < 2 * len; i += blockDim.x) xo[i] = (&s_cx[0][0])[i];
    }
    if (stamp) a.dbg_clk[11] = clock64();
}

template <int KIND, int NPT, int L, int MODE, bool PC>
__global__ void __launch_bounds__(kLeafThreads, 1) leaf_kernel(LeafArgs a) {
    pdl_launch_dependents(a.pdl_trigger);
    extern __shared__ __align__(16) double s_dyn0[];
    leaf_body<KIND, NPT, L, MODE, PC>(a, s_dyn0, true);
}

// Phase 2 reduced recursion (see file header): warps < ceil(P/32) of the
// calling CTA, one slab per lane; `cin(sl, k, side)` supplies slab sl's
// phase-1 carry of step k, `out(sl, k, EL, ER)` receives every active slab's
// injections.  Used once per plan with unit impulses to tabulate the
// injection response W (leaf_wbuild below); the per-leaf phase 2 is then a
// matvec with W (correct_body).  Exact linear superposition of this recursion.
template <int KIND, int L, class Cin, class Out>
__device__ __forceinline__ void phase2_rec(const LeafArgs& a, int pb, int len, const double (*s_h)[L][4],
                                           double (*s_part)[8][2], double* s_tot, Cin cin, Out out) {
    constexpr bool TRI = KIND == SK_TRIDIAG;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int P = a.P;
    const int nw2 = (P + 31) >> 5;
    const ProblemConst pc = a.pc[pb];
    const double lam = pc.lam;
    const double* lp = a.lampow + (uint64_t)pb * a.lp_stride;
    const int m = a.slab;
    const int mlast = a.nodes - (P - 1) * m;
    const int sl = w * 32 + lane;          // slab owned by this lane
    const bool act = sl < P;
    const int ht = (sl == P - 1) ? 1 : 0;  // response table of this slab
    const double mu = lp[min(m, a.lp_stride - 1)];          // lam^m between slab ends
    const double mu_last = lp[min(mlast, a.lp_stride - 1)];
    double pw[5], pwb[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const double p = lp[min(m << d, a.lp_stride - 1)];
        pw[d] = lane >= (1 << d) ? p : 0.0;
        pwb[d] = lane + (1 << d) < 32 ? p : 0.0;
    }
    const double muW = lp[min(32 * m, a.lp_stride - 1)];
    const double exm = lane > 0 ? 1.0 : 0.0, exbm = lane < 31 ? 1.0 : 0.0;
    const double lamA = act ? lp[min(sl * m + 1, a.lp_stride - 1)] : 0.0;
    const int last_s = act ? min(sl * m + m, a.nodes) - 1 : 0;
    const double lamB = act ? lp[min(a.nodes - last_s, a.lp_stride - 1)] : 0.0;
    const double lmF = lp[min(m * lane, a.lp_stride - 1)];
    const double lmB = lp[min(m * (31 - lane), a.lp_stride - 1)];
    // rolling accumulators: accF[i], accB[i] collect the lag responses
    // destined for step k + i
    double accF[L], accB[L];
#pragma unroll
    for (int i = 0; i < L; ++i) {
        accF[i] = 0.0;
        accB[i] = 0.0;
    }
    const int nth2 = nw2 * 32;
#pragma unroll 2
    for (int k = 0; k < len; ++k) {
        double cF = act ? cin(sl, k, 0) + accF[0] : 0.0;
        double cB = act ? cin(sl, k, 1) + accB[0] : 0.0;
        // inclusive scans over slabs (uniform multiplier lam^m)
        double SF = cF, SB = cB;
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            SF = fma(pw[d], __shfl_up_sync(0xffffffffu, SF, 1 << d), SF);
            if (TRI) SB = fma(pwb[d], __shfl_down_sync(0xffffffffu, SB, 1 << d), SB);
        }
        const double exF = exm * __shfl_up_sync(0xffffffffu, SF, 1);
        const double exB = TRI ? exbm * __shfl_down_sync(0xffffffffu, SB, 1) : 0.0;
        double (*part)[2] = s_part[k & 1];
        if (lane == 31) part[w][0] = SF;
        if (lane == 0) part[w][1] = SB;
        asm volatile("bar.sync 1, %0;" ::"r"(nth2) : "memory");
        double CF = 0.0, runF = 0.0, CB = 0.0, runB = 0.0;
        for (int ww = 0; ww < nw2; ++ww) {
            if (ww == w) CF = runF;
            runF = fma(muW, runF, part[ww][0]);
            if (TRI) {
                const int wb = nw2 - 1 - ww;
                if (wb == w) CB = runB;
                runB = fma(muW, runB, part[wb][1]);
            }
        }
        // exclusive carries into this slab: F at the node before it, B after it
        const double FLin = fma(lmF, CF, exF);
        const double BRin = TRI ? fma(lmB, CB, exB) : 0.0;
        double* tot = s_tot;
        if (sl == P - 1) tot[0] = fma(mu_last, FLin, cF);  // F at node n-1
        if (sl == 0) tot[1] = fma(mu, BRin, cB);            // B at node 0
        asm volatile("bar.sync 1, %0;" ::"r"(nth2) : "memory");
        double EL, ER;
        if (TRI) {
            const double p0 = pc.G0 * lam * tot[1], pM1 = pc.G0 * lam * tot[0];
            const double alpha = (pc.Lam * pM1 - p0) * pc.inv1mL2;
            const double gam = (pc.Lam * p0 - pM1) * pc.inv1mL2;
            EL = fma(pc.G0 * lam, FLin, alpha * lamA);
            ER = fma(pc.G0 * lam, BRin, gam * lamB);
        } else {
            EL = a.stencil ? FLin : lam * FLin;  // Scheme 2: the boundary value itself (see slab_responses)
            ER = 0.0;
        }
        if (act) out(sl, k, EL, ER);
#pragma unroll
        for (int c = 0; c < L; c += 8) {
            if (c == 0 || k + 1 + c < len) {  // dead entries (k + 1 + i >= len) skipped in chunks
#pragma unroll
                for (int i = c; i < c + 8 && i + 1 < L; ++i) {
                    const double2 hF = *reinterpret_cast<const double2*>(&s_h[ht][i + 1][0]);
                    accF[i] = fma(hF.x, EL, fma(hF.y, ER, accF[i + 1]));
                    if (TRI) {
                        const double2 hB = *reinterpret_cast<const double2*>(&s_h[ht][i + 1][2]);
                        accB[i] = fma(hB.x, EL, fma(hB.y, ER, accB[i + 1]));
                    }
                }
            }
        }
        accF[L - 1] = 0.0;
        accB[L - 1] = 0.0;
        // s_tot / s_part are rewritten next step only after its first barrier,
        // which every reader of this step has passed
    }
}

// Injection response table W[b][s][side][lag][j] (j = 2 s' + side'): slab s's
// injection (EL: side 0, ER: side 1) at step `lag` caused by a unit phase-1
// carry of slab s' (F: side' 0, B: side' 1) at step 0.  The reduced system is
// time-invariant inside a leaf, so EL/ER_k = sum_{l<=k} sum_j W[.][k-l][j] c_l[j].
// Grid (2P, B), block ceil(P/32) warps.
template <int KIND, int L>
__global__ void __launch_bounds__(kMaxSlabs / 32 * 32 + 32) leaf_wbuild(LeafArgs a, double* W) {
    __shared__ __align__(16) double s_h[2][L][4];
    __shared__ double s_part[2][8][2];
    __shared__ double s_tot[2];
    const int j = blockIdx.x, pb = blockIdx.y;
    const int P = a.P;
    const double* hsrc = a.resp_h + (uint64_t)pb * 2 * L * 4;
    for (int i = threadIdx.x; i < 2 * L * 4; i += blockDim.x) (&s_h[0][0][0])[i] = hsrc[i];
    __syncthreads();
    const int js = j >> 1, jside = j & 1;
    double* Wb = W + (uint64_t)pb * P * 2 * L * 2 * P;
    phase2_rec<KIND, L>(
        a, pb, L, s_h, s_part, s_tot,
        [&](int sl, int k, int side) { return (sl == js && k == 0 && side == jside) ? 1.0 : 0.0; },
        [&](int sl, int k, double EL, double ER) {
            Wb[(((uint64_t)sl * 2 + 0) * L + k) * 2 * P + j] = EL;
            Wb[(((uint64_t)sl * 2 + 1) * L + k) * 2 * P + j] = ER;
        });
}

// Phase 2 + 3 of the slab decomposition (see file header).  One CTA per slab.
// Phase 2 is a matvec with the tabulated injection response (leaf_wbuild):
// every thread owns source carries j, accumulates the 2 x L injections of its
// own slab over them, and a butterfly reduce-scatter + cross-warp sum folds
// the 256 partial vectors (fixed order: bitwise reproducible, independent of
// how slabs are partitioned over ranks).
template <int KIND, int NPT, int L, bool LEAN = false, bool PAIR = false>
__device__ __forceinline__ void correct_body(const LeafArgs& a, double* s_c0, double* s_x, bool x_resident,
                                             int half = 0) {
    // s_c0: carries of every slab transposed to [L][2P + 1]; s_x: [m][L+1] phase-1 solution tile
    __shared__ double s_inj[L][2];          // this slab's EL_k, ER_k
    __shared__ double s_red[kLeafThreads / 32][2 * L];

    constexpr bool TRI = KIND == SK_TRIDIAG;
    const int cta = blockIdx.x;
    const int pb = cta / a.P_local, s = a.s_begin + (cta - pb * a.P_local);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int P = a.P;
    const int len = LEAN ? L : a.len;
    const int m = a.slab;
    const int JS = 2 * P + 1;

    const bool stamp = a.dbg_clk && blockIdx.x == 0 && threadIdx.x == 0;
    if (stamp) a.dbg_clk[0] = clock64();
    // load the carries of every slab of this problem (transposed) and the phase-1 tile
    const uint64_t t0 = a.t0 + (PAIR ? (uint64_t)half * L : 0);
    // (pair kernel: the second leaf's carries use the other half of the double-sized buffer, so
    // a fast CTA's phase 1 never overwrites carries a slow CTA is still reading)
    const double* xin = a.xch + (uint64_t)pb * P * L * 2 + (PAIR ? (uint64_t)half * gridDim.x * L * 2 : 0);
    {   // 16-byte loads (one step's two carries of a slab), 16 in flight per thread
        const double2* xin2 = reinterpret_cast<const double2*>(xin);
        const int total2 = P * L;
        for (int i0 = 0; i0 < total2; i0 += 16 * kLeafThreads) {
            double2 v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int i = i0 + u * kLeafThreads + tid;
                v[u] = i < total2 ? __ldcg(&xin2[i]) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int i = i0 + u * kLeafThreads + tid;
                if (i < total2) {
                    const int sp = i / L, l = i - sp * L;
                    s_c0[l * JS + 2 * sp] = v[u].x;
                    s_c0[l * JS + 2 * sp + 1] = v[u].y;
                }
            }
        }
    }
    const int slab0 = s * m;
    const int mreal = min(m, a.nodes - slab0);
    const uint64_t rowb = (uint64_t)pb * a.rows_pp + (slab0 - a.node_begin);  // X row of node slab0
    if (!x_resident) {
        constexpr int HL = L / 2;
        const bool vec = len == L && (a.N & 1) == 0 && (a.t0 & 1) == 0;
        const int total = vec ? mreal * HL : mreal * len;
        for (int e0 = 0; e0 < total; e0 += 8 * kLeafThreads) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * kLeafThreads + tid;
                if (vec) {
                    const int q = e / HL, k2 = e - q * HL;
                    v[u] = e < total ? __ldcg(reinterpret_cast<const double2*>(a.X + (rowb + q) * a.N + a.t0) + k2)
                                     : make_double2(0.0, 0.0);
                } else {
                    const int q = e / len, k = e - q * len;
                    v[u] = make_double2(e < total ? a.X[(rowb + q) * a.N + a.t0 + k] : 0.0, 0.0);
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * kLeafThreads + tid;
                if (e >= total) continue;
                if (vec) {
                    const int q = e / HL, k2 = e - q * HL;
                    s_x[q * (L + 1) + 2 * k2] = v[u].x;
                    s_x[q * (L + 1) + 2 * k2 + 1] = v[u].y;
                } else {
                    const int q = e / len, k = e - q * len;
                    s_x[q * (L + 1) + k] = v[u].x;
                }
            }
        }
    }
    __syncthreads();
    if (stamp) a.dbg_clk[1] = clock64();

    // ---- phase 2: EL/ER_k = sum_{l<=k} sum_j W[k-l][j] c_l[j] ----
    // One side at a time (rolled: instruction footprint, see leaf_body): every thread owns
    // source carries j and accumulates the L injections of its slab over them; a butterfly
    // reduce-scatter (lane keeps output `lane`) + cross-warp sum folds the partial vectors
    // (fixed order: bitwise reproducible, independent of the rank partition).
    if (!(a.dbg & 1)) {
        const double* Ws = a.resp_w + ((uint64_t)pb * P + s) * 2 * L * 2 * P;
        if (!TRI) {
            for (int i = tid; i < (kLeafThreads / 32) * L; i += kLeafThreads) s_red[i / L][L + (i & (L - 1))] = 0.0;
        }
#pragma unroll 1
        for (int side = 0; side < (TRI ? 2 : 1); ++side) {
            double acc[L];
#pragma unroll
            for (int o = 0; o < L; ++o) acc[o] = 0.0;
#pragma unroll 1
            for (int j = tid; j < 2 * P; j += kLeafThreads) {
                double wv[L];
#pragma unroll
                for (int l = 0; l < L; ++l) wv[l] = __ldg(&Ws[((uint64_t)side * L + l) * 2 * P + j]);
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    const double cv = l < len ? s_c0[l * JS + j] : 0.0;
#pragma unroll
                    for (int k = l; k < L; ++k) acc[k] = fma(wv[k - l], cv, acc[k]);
                }
            }
#pragma unroll
            for (int st = 0; st < 5; ++st) {
                const int off = 16 >> st, half = (L / 2) >> st;
                const bool up = (lane & off) != 0;
#pragma unroll
                for (int i = 0; i < half; ++i) {
                    const double send = up ? acc[i] : acc[i + half];
                    const double keep = up ? acc[i + half] : acc[i];
                    acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                }
            }
            s_red[w][side * L + lane] = acc[0];
        }
        __syncthreads();
        if (tid < 2 * L) {
            double v = 0.0;
#pragma unroll
            for (int ww = 0; ww < kLeafThreads / 32; ++ww) v += s_red[ww][tid];
            s_inj[tid & (L - 1)][tid / L] = v;
        }
    } else if (tid < 2 * L) {
        s_inj[tid & (L - 1)][tid / L] = 0.0;
    }
    __syncthreads();

    if (stamp) a.dbg_clk[2] = clock64();
    // ---- phase 3: x = x0 + sum_l GL(l) EL_(k-l) + GR(l) ER_(k-l) ----
    // Rolled: win[i] collects the responses to the injections of step st at step st + i; the
    // finished correction of step st leaves at win[0].  Segments of 4 steps with a static
    // window length (entries that would land past the leaf end are never formed).
    const int tsel = (s == P - 1) ? 1 : 0;
    // tables are time-major [side][l][q]: lanes (consecutive q) read coalesced
    const double* GT = a.resp_g + ((uint64_t)pb * 2 + tsel) * 2 * (uint64_t)m * L;
    if (TRI && a.paired_g) {
        // Mirror pairs: x_q += S (EL + ER) + D (EL - ER), x_(mreal-1-q) += S (EL + ER) - D (EL - ER)
        // with S = (GL_q + GR_q) / 2, D = (GL_q - GR_q) / 2 (GR_q = GL_(mreal-1-q) by symmetry):
        // one table and one window per pass, half the products and half the table traffic of
        // the unpaired form (17.1 k -> 13.5 k cycles per leaf; what remains is mostly the 128 CTAs
        // pulling the same 64 KB table from L2 at once -- fetching it earlier, across phase 2,
        // cost more in step-loop spills than it saved).
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
            const double sgn = pass ? -1.0 : 1.0;
#pragma unroll 1
            for (int q = tid; q < (mreal + 1) / 2; q += blockDim.x) {
                const int q2 = mreal - 1 - q;
                double g[L], win[L];
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    g[l] = GT[((uint64_t)pass * L + l) * m + q];
                    win[l] = 0.0;
                }
                double* xq = s_x + q * (L + 1);
                double* xq2 = s_x + q2 * (L + 1);
                const bool two = q2 != q;
                // the injection of the next step is fetched one iteration ahead and the tile values
                // before the window products, so no step waits on shared memory
                double e_next = fma(sgn, s_inj[0][1], s_inj[0][0]);  // EL + ER, EL - ER
#pragma unroll
                for (int sg = 0; sg < L / 4; ++sg) {
#pragma unroll 1
                    for (int st = 4 * sg; st < 4 * sg + 4; ++st) {
                        if (st >= len) break;
                        const double e = e_next;
                        const double xv = xq[st], xv2 = xq2[st];
                        const int sn = st + 1 < L ? st + 1 : st;
                        e_next = fma(sgn, s_inj[sn][1], s_inj[sn][0]);
                        const double c = fma(g[0], e, win[0]);
#pragma unroll
                        for (int i = 0; i < L - 1 - 4 * sg; ++i) win[i] = fma(g[i + 1], e, win[i + 1]);
                        xq[st] = xv + c;
                        if (two) xq2[st] = fma(sgn, c, xv2);
                    }
                }
            }
        }
    } else
#pragma unroll 1
    for (int q = tid; q < mreal; q += blockDim.x) {
        double gL[L], gR[TRI ? L : 1], win[L];
#pragma unroll
        for (int l = 0; l < L; ++l) {
            gL[l] = GT[(uint64_t)l * m + q];
            if (TRI) gR[l] = GT[((uint64_t)L + l) * m + q];
            win[l] = 0.0;
        }
        double* xq = s_x + q * (L + 1);
#pragma unroll
        for (int sg = 0; sg < L / 4; ++sg) {
            constexpr int dummy = 0;
            (void)dummy;
#pragma unroll 1
            for (int st = 4 * sg; st < 4 * sg + 4; ++st) {
                if (st >= len) break;
                const double el = s_inj[st][0];
                const double er = TRI ? s_inj[st][1] : 0.0;
                xq[st] += fma(gL[0], el, TRI ? fma(gR[0], er, win[0]) : win[0]);
                // targets st + 1 + i <= L - 1; blocks of 8 so that the two dependent products of an
                // entry are 8 independent DFMAs apart (back to back they exposed the pipe latency)
#pragma unroll
                for (int i0 = 0; i0 < L - 1 - 4 * sg; i0 += 8) {
                    double t8[8];
#pragma unroll
                    for (int i = i0; i < i0 + 8 && i < L - 1 - 4 * sg; ++i)
                        t8[i - i0] = TRI ? fma(gR[TRI ? i + 1 : 0], er, win[i + 1]) : win[i + 1];
#pragma unroll
                    for (int i = i0; i < i0 + 8 && i < L - 1 - 4 * sg; ++i) win[i] = fma(gL[i + 1], el, t8[i - i0]);
                }
            }
        }
    }
    __syncthreads();
    if (stamp) a.dbg_clk[3] = clock64();
    store_rows<L, LEAN>(a.X, s_x, rowb, a.N, t0, mreal, len, tid, blockDim.x);
    if (!LEAN && a.V) {  // Scheme 2 product sources V = U_i + U_(i-1); the slab's left neighbour value is EL
        for (int e = tid; e < mreal * len; e += blockDim.x) {
            const int q = e / len, k = e - q * len;
            const double left = q > 0 ? s_x[(q - 1) * (L + 1) + k] : s_inj[k][0];
            a.V[(rowb + q) * a.N + t0 + k] = s_x[q * (L + 1) + k] + left;
        }
    }
    if (stamp) a.dbg_clk[4] = clock64();
}

template <int KIND, int NPT, int L>
__global__ void __launch_bounds__(kLeafThreads, 1) leaf_correct(LeafArgs a) {
    pdl_launch_dependents(a.pdl_trigger);
    pdl_wait();
    extern __shared__ __align__(16) double s_dyn[];
    correct_body<KIND, NPT, L>(a, s_dyn, s_dyn + (uint64_t)L * (2 * a.P + 1), false);
}

// L2 prefetch (evict_last) of the phase-2/3 tables this slab will read: its
// rows of the injection response W and a share of the response table G, so
// they arrive from L2 instead of HBM after the history products streamed
// through the cache (ncu: long-scoreboard stalls in phases 2/3).
__device__ __forceinline__ void prefetch_l2_last(const void* ptr) {
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(ptr));
}

template <int L>
__device__ __forceinline__ void prefetch_correct_tables(const LeafArgs& a) {
    if (!a.resp_w || (a.dbg & 16)) return;
    const int cta = blockIdx.x;
    const int pb = cta / a.P_local, s = a.s_begin + (cta - pb * a.P_local);
    const int P = a.P, m = a.slab;
    const char* w = reinterpret_cast<const char*>(a.resp_w + ((uint64_t)pb * P + s) * 2 * L * 2 * P);
    const int wbytes = 2 * L * 2 * P * 8;
    for (int o = threadIdx.x * 128; o < wbytes; o += blockDim.x * 128) prefetch_l2_last(w + o);
    // G tables [side][l][q] of the two slab kinds: lines spread over the CTAs of the problem
    const char* g = reinterpret_cast<const char*>(a.resp_g + (uint64_t)pb * 2 * 2 * (uint64_t)m * L);
    const int gbytes = 2 * 2 * m * L * 8;
    const int c0 = cta - pb * a.P_local, nc = a.P_local;
    for (int o = (c0 * blockDim.x + threadIdx.x) * 128; o < gbytes; o += nc * blockDim.x * 128) prefetch_l2_last(g + o);
}

// Single-GPU slab leaf in ONE cooperative kernel: phase 1, publish carries, a
// grid barrier (all slabs co-resident), phases 2 + 3 on the resident tile.
template <int KIND, int NPT, int L, bool PC, bool LEAN>
__global__ void __launch_bounds__(kLeafThreads, 1) leaf_fused(LeafArgs a) {
    extern __shared__ __align__(16) double s_dyn[];
    double* s_c0 = s_dyn;
    double* s_x = s_dyn + (uint64_t)L * (2 * a.P + 1);
    const bool stamp = a.dbg_clk && blockIdx.x == 0 && threadIdx.x == 0;
    if (stamp) a.dbg_clk[12] = clock64();
    prefetch_correct_tables<L>(a);
    leaf_body<KIND, NPT, L, 1, PC, LEAN>(a, s_x, false);
    __syncthreads();
    if (stamp) a.dbg_clk[14] = clock64();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(a.bar, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
        } while (v < a.bar_target);
    }
    __syncthreads();
    if (stamp) a.dbg_clk[13] = clock64();
    correct_body<KIND, NPT, L, LEAN>(a, s_c0, s_x, true);
}

// Chained upwind slabs (config 3, Scheme 3 problems of 2 .. 4 slabs): one cooperative kernel per
// leaf (co-residency makes the per-step waits safe), no correction phase.
template <int KIND, int NPT, int L, bool PC, bool LEAN>
__global__ void __launch_bounds__(kLeafThreads, 1) leaf_chain(LeafArgs a) {
    extern __shared__ __align__(16) double s_dyn[];
    leaf_body<KIND, NPT, L, 2, PC, LEAN>(a, s_dyn, true);
}

// Two consecutive slab leaves in one cooperative kernel (single-GPU plans whose level-0
// history products fold into the leaf: between leaves 2i and 2i+1 the schedule has no other
// product).  The first leaf's solution stays in shared memory, so the level-0 product reads
// it there (no re-staging of U from global memory), the second leaf's R tile is prefetched
// into L2 while the first leaf runs, and one launch per pair disappears.  The body is a
// rolled loop over the two leaves: the instruction footprint is that of one leaf.
template <int KIND, int NPT, int L>
__global__ void __launch_bounds__(kLeafThreads, 1) leaf_pair(LeafArgs a) {
    extern __shared__ __align__(16) double s_dyn[];
    double* s_c0 = s_dyn;
    double* s_x = s_dyn + (uint64_t)L * (2 * a.P + 1);
    const bool stamp = a.dbg_clk && blockIdx.x == 0 && threadIdx.x == 0;
    if (stamp) a.dbg_clk[12] = clock64();
    prefetch_correct_tables<L>(a);
    {   // the second leaf's R tile (final since the last product kernel): into L2 now
        const int cta = blockIdx.x;
        const int pb = cta / a.P_local, s = a.s_begin + (cta - pb * a.P_local);
        const int slab0 = s * a.slab;
        const int mreal = min(a.slab, a.nodes - slab0);
        const uint64_t rowb = (uint64_t)pb * a.rows_pp + (slab0 - a.node_begin);
        for (int e = threadIdx.x; e < 2 * mreal; e += blockDim.x)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.src2 + (rowb + (e >> 1)) * a.N + a.t0 + L + (e & 1) * 16));
    }
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
        leaf_body<KIND, NPT, L, 1, true, true, true>(a, s_x, false, half);
        __syncthreads();
        if (stamp) a.dbg_clk[14] = clock64();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(a.bar, 1u);
            const unsigned target = a.bar_target + (unsigned)half * gridDim.x;
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
            } while (v < target);
        }
        __syncthreads();
        if (stamp) a.dbg_clk[13] = clock64();
        correct_body<KIND, NPT, L, true, true>(a, s_c0, s_x, true, half);
    }
}

// Partitioned slab leaf with the carry exchange done by the kernel itself over
// NVLink peer memory (opt-in, ft_p2p_connect): phase 1; every CTA stores its
// slab's 2L carries into every rank's receive buffer (parity = leaf index & 1,
// so a fast rank never overwrites carries a slow rank is still reading: it
// cannot pass the next leaf's barrier before that rank arrives), fences at
// system scope and bumps every rank's arrival counter; one thread per CTA
// waits until its own counter shows all world x P_local slabs of this leaf;
// phases 2/3 read the gathered carries locally.  Counters are cumulative over
// solves (epoch kernel at each solve start), so no reset race exists.
template <int KIND, int NPT, int L, bool PC>
__global__ void __launch_bounds__(kLeafThreads, 1) leaf_fused_p2p(LeafArgs a) {
    extern __shared__ __align__(16) double s_dyn[];
    double* s_c0 = s_dyn;
    double* s_x = s_dyn + (uint64_t)L * (2 * a.P + 1);
    leaf_body<KIND, NPT, L, 1, PC>(a, s_x, false);  // carries -> a.xsend[cta] (local)
    __syncthreads();
    const int cta = blockIdx.x, s = a.s_begin + cta;
    const double* mine = a.xsend + (uint64_t)cta * L * 2;
    const size_t par_off = (size_t)(a.p2p_leaf & 1) * a.P * L * 2;
    for (int r = 0; r < a.p2p_world; ++r) {
        double* dst = reinterpret_cast<double*>(a.p2p_peers[r] + kP2pHeader) + par_off + (uint64_t)s * L * 2;
        for (int i = threadIdx.x; i < 2 * L; i += blockDim.x) dst[i] = __ldcg(&mine[i]);
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int r = 0; r < a.p2p_world; ++r)
            atomicAdd_system(reinterpret_cast<unsigned long long*>(a.p2p_peers[r]), 1ull);
        const unsigned epoch = *a.p2p_epoch;  // 1-based: solves started on this rank
        const unsigned long long per_leaf = (unsigned long long)a.p2p_world * a.P_local;
        const unsigned long long target =
            ((unsigned long long)(epoch - 1) * a.p2p_leaves + a.p2p_leaf + 1) * per_leaf;
        const unsigned long long* own = reinterpret_cast<const unsigned long long*>(a.p2p_peers[a.s_begin / a.P_local]);
        unsigned long long v;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(own) : "memory");
        } while (v < target);
    }
    __syncthreads();
    correct_body<KIND, NPT, L>(a, s_c0, s_x, true);  // a.xch = this rank's receive buffer (parity)
}

__global__ void p2p_epoch_kernel(unsigned* epoch) { *epoch += 1u; }

cudaError_t launch_p2p_epoch(unsigned* epoch, cudaStream_t st) {
    p2p_epoch_kernel<<<1, 1, 0, st>>>(epoch);
    return cudaGetLastError();
}

// ---- host launch -------------------------------------------------------------

template <int KIND, int NPT, int L>
static cudaError_t launch_leaf_t(const LeafArgs& a, int ctas, int threads, bool multi, cudaStream_t st) {
    const size_t osmem = sizeof(double) * (size_t)kLeafThreads * NPT * (L + 1);
    static DeviceOnce oattr;
    if (oattr.first()) {
        const int mx = (int)(sizeof(double) * kLeafThreads * NPT * (L + 1));
        cudaFuncSetAttribute(leaf_kernel<KIND, NPT, L, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(leaf_kernel<KIND, NPT, L, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(leaf_kernel<KIND, NPT, L, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(leaf_kernel<KIND, NPT, L, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        oattr.done();
    }
    const dim3 blk(KIND == SK_DIAG ? threads : kLeafThreads);
    if (!multi) {
        return a.kc_valid ? launch_ex(leaf_kernel<KIND, NPT, L, 0, true>, dim3(ctas), blk, osmem, st, 1, a)
                          : launch_ex(leaf_kernel<KIND, NPT, L, 0, false>, dim3(ctas), blk, osmem, st, 1, a);
    }
    return a.kc_valid ? launch_ex(leaf_kernel<KIND, NPT, L, 1, true>, dim3(ctas), dim3(kLeafThreads), osmem, st, 1, a)
                      : launch_ex(leaf_kernel<KIND, NPT, L, 1, false>, dim3(ctas), dim3(kLeafThreads), osmem, st, 1, a);
}

template <int KIND, int NPT, int L>
static cudaError_t launch_correct_t(const LeafArgs& a, int ctas, cudaStream_t st) {
    const size_t smem = sizeof(double) * ((size_t)L * (2 * a.P + 1) + (size_t)a.slab * (L + 1));
    static DeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(leaf_correct<KIND, NPT, L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double) * (L * (2 * kMaxSlabs + 1) + kLeafThreads * NPT * (L + 1))));
        attr.done();
    }
    return launch_ex(leaf_correct<KIND, NPT, L>, dim3(ctas), dim3(kLeafThreads), smem, st, 1, a);
}

template <int KIND, int NPT, int L>
static cudaError_t launch_fused_t(const LeafArgs& a, int ctas, cudaStream_t st) {
    const size_t smem = sizeof(double) * ((size_t)L * (2 * a.P + 1) + (size_t)kLeafThreads * NPT * (L + 1));
    static DeviceOnce attr;
    const int mx = (int)(sizeof(double) * (L * (2 * kMaxSlabs + 1) + kLeafThreads * NPT * (L + 1)));
    if (attr.first()) {
        cudaFuncSetAttribute(leaf_fused<KIND, NPT, L, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(leaf_fused<KIND, NPT, L, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(leaf_fused<KIND, NPT, L, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(leaf_fused<KIND, NPT, L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        attr.done();
    }
    // the common case (whole leaves of an even-N problem, R from an array) runs the lean
    // instantiation: generic staging / streamed-R / fused-RHS / Scheme-2 paths compiled out
    static const bool no_lean = getenv("FT_NO_LEAN") != nullptr;
    const bool lean = !no_lean && a.len == L && (a.N & 1) == 0 && !a.radd && !a.genA && !a.V && !a.stencil;
    // cooperative attribute through cudaLaunchKernelEx: capturable into the solve's CUDA graph
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kLeafThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute coop[1];
    coop[0].id = cudaLaunchAttributeCooperative;
    coop[0].val.cooperative = 1;
    cfg.attrs = coop;
    cfg.numAttrs = 1;
    if (lean)
        return a.kc_valid ? cudaLaunchKernelEx(&cfg, leaf_fused<KIND, NPT, L, true, true>, a)
                          : cudaLaunchKernelEx(&cfg, leaf_fused<KIND, NPT, L, false, true>, a);
    return a.kc_valid ? cudaLaunchKernelEx(&cfg, leaf_fused<KIND, NPT, L, true, false>, a)
                      : cudaLaunchKernelEx(&cfg, leaf_fused<KIND, NPT, L, false, false>, a);
}

template <int KIND, int NPT, int L>
static cudaError_t launch_pair_t(const LeafArgs& a, int ctas, cudaStream_t st) {
    const size_t smem = sizeof(double) * ((size_t)L * (2 * a.P + 1) + (size_t)kLeafThreads * NPT * (L + 1));
    static DeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(leaf_pair<KIND, NPT, L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double) * (L * (2 * kMaxSlabs + 1) + kLeafThreads * NPT * (L + 1))));
        attr.done();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kLeafThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute coop[1];
    coop[0].id = cudaLaunchAttributeCooperative;
    coop[0].val.cooperative = 1;
    cfg.attrs = coop;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, leaf_pair<KIND, NPT, L>, a);
}

template <int KIND, int NPT, int L>
static cudaError_t launch_p2p_t(const LeafArgs& a, int ctas, cudaStream_t st) {
    const size_t smem = sizeof(double) * ((size_t)L * (2 * a.P + 1) + (size_t)kLeafThreads * NPT * (L + 1));
    static DeviceOnce attr;
    if (attr.first()) {
        const int mx = (int)(sizeof(double) * (L * (2 * kMaxSlabs + 1) + kLeafThreads * NPT * (L + 1)));
        cudaFuncSetAttribute(leaf_fused_p2p<KIND, NPT, L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(leaf_fused_p2p<KIND, NPT, L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        attr.done();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kLeafThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute coop[1];
    coop[0].id = cudaLaunchAttributeCooperative;  // every slab CTA of this rank co-resident
    coop[0].val.cooperative = 1;
    cfg.attrs = coop;
    cfg.numAttrs = 1;
    return a.kc_valid ? cudaLaunchKernelEx(&cfg, leaf_fused_p2p<KIND, NPT, L, true>, a)
                      : cudaLaunchKernelEx(&cfg, leaf_fused_p2p<KIND, NPT, L, false>, a);
}

cudaError_t launch_leaf_p2p(int kind, int npt, int L, const LeafArgs& a, int ctas, cudaStream_t st) {
    if (npt == 2 && L == 32) {
        if (kind == SK_TRIDIAG) return launch_p2p_t<SK_TRIDIAG, 2, 32>(a, ctas, st);
        if (kind == SK_UPWIND) return launch_p2p_t<SK_UPWIND, 2, 32>(a, ctas, st);
    }
    return cudaErrorInvalidValue;
}

// both leaves whole, even N, R from arrays, single-problem constants: see leaf_pair
bool leaf_pair_ok(const LeafArgs& a, int L) {
    static const bool off = getenv("FT_NO_PAIR") != nullptr || getenv("FT_NO_LEAN") != nullptr;
    return !off && a.kc_valid && a.len == L && (a.N & 1) == 0 && !a.radd && !a.genA && !a.V && !a.stencil;
}

cudaError_t launch_leaf_pair(int kind, int npt, int L, const LeafArgs& a, int ctas, cudaStream_t st) {
    if (npt == 2 && L == 32) {
        if (kind == SK_TRIDIAG) return launch_pair_t<SK_TRIDIAG, 2, 32>(a, ctas, st);
        if (kind == SK_UPWIND) return launch_pair_t<SK_UPWIND, 2, 32>(a, ctas, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_leaf_fused(int kind, int npt, int L, const LeafArgs& a, int ctas, cudaStream_t st) {
    if (npt == 2 && L == 32) {
        if (kind == SK_TRIDIAG) return launch_fused_t<SK_TRIDIAG, 2, 32>(a, ctas, st);
        if (kind == SK_UPWIND) return launch_fused_t<SK_UPWIND, 2, 32>(a, ctas, st);
    }
    return cudaErrorInvalidValue;
}

template <int NPT, int L>
static cudaError_t launch_chain_t(const LeafArgs& a, int ctas, cudaStream_t st) {
    const size_t smem = sizeof(double) * (size_t)kLeafThreads * NPT * (L + 1);
    static DeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(leaf_chain<SK_UPWIND, NPT, L, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(leaf_chain<SK_UPWIND, NPT, L, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(leaf_chain<SK_UPWIND, NPT, L, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(leaf_chain<SK_UPWIND, NPT, L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr.done();
    }
    static const bool no_lean = getenv("FT_NO_LEAN") != nullptr;
    const bool lean = !no_lean && a.len == L && (a.N & 1) == 0 && !a.radd && !a.genA && !a.V && !a.stencil;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kLeafThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute coop[1];
    coop[0].id = cudaLaunchAttributeCooperative;
    coop[0].val.cooperative = 1;
    cfg.attrs = coop;
    cfg.numAttrs = 1;
    if (lean)
        return a.kc_valid ? cudaLaunchKernelEx(&cfg, leaf_chain<SK_UPWIND, NPT, L, true, true>, a)
                          : cudaLaunchKernelEx(&cfg, leaf_chain<SK_UPWIND, NPT, L, false, true>, a);
    return a.kc_valid ? cudaLaunchKernelEx(&cfg, leaf_chain<SK_UPWIND, NPT, L, true, false>, a)
                      : cudaLaunchKernelEx(&cfg, leaf_chain<SK_UPWIND, NPT, L, false, false>, a);
}

cudaError_t launch_leaf_chain(int kind, int npt, int L, const LeafArgs& a, int ctas, cudaStream_t st) {
    if (npt == 2 && L == 32 && kind == SK_UPWIND) return launch_chain_t<2, 32>(a, ctas, st);
    return cudaErrorInvalidValue;
}

cudaError_t launch_leaf_correct(int kind, int npt, int L, const LeafArgs& a, int ctas, cudaStream_t st) {
    if (npt == 2 && L == 32) {
        if (kind == SK_TRIDIAG) return launch_correct_t<SK_TRIDIAG, 2, 32>(a, ctas, st);
        if (kind == SK_UPWIND) return launch_correct_t<SK_UPWIND, 2, 32>(a, ctas, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_leaf_wbuild(int kind, int L, const LeafArgs& a, int B, double* W, cudaStream_t st) {
    const dim3 grid(2 * a.P, B);
    const int threads = ((a.P + 31) / 32) * 32;
    if (L != 32) return cudaErrorInvalidValue;
    if (kind == SK_TRIDIAG) leaf_wbuild<SK_TRIDIAG, 32><<<grid, threads, 0, st>>>(a, W);
    else if (kind == SK_UPWIND) leaf_wbuild<SK_UPWIND, 32><<<grid, threads, 0, st>>>(a, W);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

// ---- the constant bank of batched plans' leaf weights --------------------------
namespace {
struct LeafBank {
    std::mutex mu;
    const void* owner[64] = {};
    cudaEvent_t done[64] = {};
};
LeafBank& leaf_bank() {
    static LeafBank b;
    return b;
}
}  // namespace

cudaError_t leaf_bank_acquire(const void* plan, const double* cols_host, int problems, cudaStream_t st) {
    LeafBank& b = leaf_bank();
    b.mu.lock();  // held until leaf_bank_release: the solve is enqueued under the lock
    const int d = DeviceOnce::dev();
    if (b.owner[d] == plan) return cudaSuccess;
    if (b.done[d]) {  // the previous owner's last solve has finished reading the bank
        cudaError_t e = cudaStreamWaitEvent(st, b.done[d], 0);
        if (e != cudaSuccess) {
            b.mu.unlock();
            return e;
        }
    }
    cudaError_t e = cudaMemcpyToSymbolAsync(c_leafcol, cols_host, sizeof(double) * 32 * problems, 0,
                                            cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) {
        b.mu.unlock();
        return e;
    }
    b.owner[d] = plan;
    return cudaSuccess;
}

cudaError_t leaf_bank_release(const void* plan, cudaStream_t st) {
    LeafBank& b = leaf_bank();
    const int d = DeviceOnce::dev();
    cudaError_t e = cudaSuccess;
    if (b.owner[d] == plan) {
        if (!b.done[d]) e = cudaEventCreateWithFlags(&b.done[d], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(b.done[d], st);
    }
    b.mu.unlock();
    return e;
}

void leaf_bank_forget(const void* plan) {  // ft_destroy: a new plan at the same address must upload
    LeafBank& b = leaf_bank();
    std::lock_guard<std::mutex> g(b.mu);
    for (auto& o : b.owner)
        if (o == plan) o = nullptr;
}

// Supported (kind, NPT, L): register tile of NPT*L doubles per thread.
cudaError_t launch_leaf(int kind, int npt, int L, bool multi, const LeafArgs& a, int ctas,
                        int threads, cudaStream_t st) {
#define FTB_LEAF_CASE(K_, NPT_, L_) \
    if (kind == K_ && npt == NPT_ && L == L_) return launch_leaf_t<K_, NPT_, L_>(a, ctas, threads, multi, st);
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
