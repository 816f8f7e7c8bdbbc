// api.cu -- C ABI (include/fractime_b200.h): scheme setup on the host
// (bit-identical to the reference: same libm calls, same expression order,
// no FMA contraction in host code), device-resident plan, and the
// divide-and-conquer driver.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fractime_b200.h"
#include "internal.cuh"

using namespace ftb;

namespace {

thread_local std::string g_err;
int g_leaf_dbg = getenv("FT_LEAF_DBG") ? atoi(getenv("FT_LEAF_DBG")) : 0;
bool g_no_kc = getenv("FT_NO_KC") != nullptr;  // A/B switch: leaf constants from constant memory

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define FT_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return set_err(FT_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                         " at " #call);                                      \
    } while (0)

struct Level {
    int n, m, K, G, groups;
    uint64_t spec_off;  // in cplx, per level block [B][K][m]
};

enum OpKind { OP_LEAF, OP_MP };
struct Op {
    OpKind kind;
    uint64_t t0;   // leaf: first step; mp: lo
    int len;       // leaf steps
    int level;     // mp level index
    uint64_t mid, hi;
    bool first;    // reads R from the caller's rhs (first touch)
};

// NCCL, bound at run time from the library the process already has (torch's libnccl.so.2) so
// the solver has no link-time dependency on it: only the calls the carry all-gather needs.
struct NcclId {
    char bytes[128];  // ncclUniqueId
};
struct NcclApi {
    int (*GetUniqueId)(NcclId*) = nullptr;
    int (*CommInitRank)(void**, int, NcclId, int) = nullptr;
    int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    bool ok = false;
};
const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        const char* names[] = {getenv("FT_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            if (!n) continue;
            void* h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (!h) continue;
            a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
            a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
            a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
            a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
            a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
            a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.CommDestroy && a.GetErrorString;
            if (a.ok) break;
        }
        return a;
    }();
    return api;
}
constexpr int kNcclFloat64 = 8;  // ncclDataType_t ncclFloat64 / ncclDouble

}  // namespace

struct ft_plan {
    int scheme = 0;
    int B = 1;
    uint64_t N = 0;
    uint64_t cells = 0;
    int nodes = 1;
    double h = 0, tau = 0;
    int rhs_mode = 0;
    bool custom = false;  // ft_setup_toeplitz plan (caller's columns, no RHS assembly)
    bool stencil = false; // Scheme 2: history products and in-leaf history act on U_i + U_(i-1)
    bool last_fuse0 = false;  // the last run_fast folded the n = 64 products into the leaves
    double* vsrc_d = nullptr;  // Scheme 2: V = U_i + U_(i-1) (product sources), rows x N
    int J = 1;
    int device = 0;
    std::vector<double> gamma;
    std::vector<double> mu, c;
    std::vector<double> col_h;   // [B][N]
    std::vector<double> wts_h;   // [B][N+1] G or M weights
    std::vector<ProblemConst> pc_h;
    // leaf configuration
    int kind = SK_DIAG;
    int L = 32, npt = 1, threads = 32, slab = 1, P = 1;
    bool multi = false;
    // slab partition across ranks (ft_setup_partitioned); single-rank: whole problem
    int part_rank = 0, part_world = 1;
    int node_begin = 0, local_nodes = 1, P_local = 1;
    ft_exchange_fn exchange = nullptr;
    void* exchange_user = nullptr;
    double* xsend_d = nullptr;  // caller-provided (partitioned) phase-1 carry buffer
    bool own_xch = true;
    // device-side exchange over NVLink peer memory (ft_p2p_handle / ft_p2p_connect)
    void* nccl_comm = nullptr;                 // ft_nccl_init: the carry all-gather is ncclAllGather on the plan's stream
    bool p2p = false;
    void* p2p_block = nullptr;                 // this rank's exchange block (kP2pHeader + receive buffers)
    std::vector<void*> p2p_opened;             // peers' blocks mapped through CUDA IPC
    unsigned long long* p2p_peers_d = nullptr; // [world] block bases, device array
    unsigned* bar_d = nullptr;  // fused slab leaf grid barrier
    cplx* mpscratch_d = nullptr;  // split K-branch history products
    bool split_k = true;
    int split_min_k = 8;        // K-branch levels with K >= this use the split (scratch) path
    long long* dbgclk_d = nullptr;
    bool fused_leaf = true;
    // levels
    std::vector<Level> levels;
    std::vector<Op> ops;
    int logT = 4;
    // device state
    ProblemConst* pc_d = nullptr;
    double* col_d = nullptr;
    double* wts_d = nullptr;
    double* lampow_d = nullptr;
    int lp_stride = 0;
    double2* chain_d = nullptr;    // chained upwind slab leaves: [B][P][L] boundary records
    bool chain_leaf = false;
    bool report_residual = false;  // FT_OPT_REPORT_RESIDUAL
    bool paired_g = false;       // resp_g holds the mirror-pair tables (phase 3 of the slab leaf)
    cplx* tw_d = nullptr;
    cplx* spec_d = nullptr;
    double* xch_d = nullptr;      // multi-slab carries of the current leaf
    double* kcoef_d = nullptr;    // single-CTA Dirichlet coefficients
    double* respg_d = nullptr;    // multi-slab space-time response tables
    double* resph_d = nullptr;
    double* respw_d = nullptr;    // multi-slab phase-2 injection responses (leaf_wbuild)
    std::vector<long double> lamL, G0L;  // long-double scan parameters (tables)
    std::vector<double> leafcol_h;       // [B][32] col[0..32) (0 beyond N) for the leaf (batched plans:
                                         // uploaded to the constant bank by leaf_bank_acquire)
    double kc_h[kKcLen] = {};            // problem 0's leaf constants (LeafArgs::kc)
    double* dw_d = nullptr;       // direct weights [B][N]
    double* cprime_d = nullptr;   // [B][nodes]
    double* den_d = nullptr;
    double* scratch_d = nullptr;  // [B][nodes]
    unsigned* dmctr_d = nullptr;  // multi-CTA direct march step counters
    double* work_d = nullptr;     // staging for host buffers
    double* rdev_d = nullptr;     // streamed host solves: device copy of the caller's R
    cudaStream_t h2d_st = nullptr, d2h_st = nullptr;  // streamed host solves: copy engines
    std::vector<cudaEvent_t> h2d_ev, d2h_ev;
    // CUDA graph of the whole launch schedule (device buffers, single rank), keyed by buffers
    cudaGraphExec_t graph = nullptr;
    const void* graph_X = nullptr;
    const void* graph_src = nullptr;
    const void* graph_gen = nullptr;
    int graph_genJ = 0;
    cudaGraphExec_t apply_graph = nullptr;  // ft_apply's launch sequence, keyed by its buffers
    const void* apply_x = nullptr;
    const void* apply_y = nullptr;
    double* genA_d = nullptr;     // ft_solve_fast_modes tables
    double* genT_d = nullptr;
    size_t genA_bytes = 0, genT_bytes = 0;
    double* genArgs_d = nullptr;  // ft_solve_fast_modes argument block
    size_t genArgs_bytes = 0;
    double* oder_d = nullptr;     // ft_solve_fast_modes on single-node plans: the RHS array
    uint64_t graph_launches = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace {

uint64_t rows_of(const ft_plan* p) { return (uint64_t)p->B * (uint64_t)p->local_nodes; }

// The n = 64 history products fold into the next cooperative slab leaf (wide
// problems only: for config 3's two slabs the standalone product is cheaper,
// 100 vs 102 ms); device-buffer solves without fused RHS generation.
bool fuse0_plan(const ft_plan* p) {
    static const bool off = getenv("FT_NO_FUSE0") != nullptr;
    static const int min_p = getenv("FT_FUSE0_MIN_P") ? atoi(getenv("FT_FUSE0_MIN_P")) : 8;
    return !off && p->multi && p->part_world == 1 && p->fused_leaf && p->L == 32 && p->B == 1 && p->P >= min_p &&
           !p->stencil;
}

// Single-node (ODE / Toeplitz) plans short enough for the one-kernel march
// (ode_whole_kernel); FT_NO_ODE1 (read once) is the A/B switch back to the D&C.
bool ode_whole_plan(const ft_plan* p) {
    static const bool no_ode1 = getenv("FT_NO_ODE1") != nullptr;
    return !no_ode1 && p->kind == SK_DIAG && p->nodes == 1 && p->part_world == 1 && ode_whole_ok(p->N);
}

// ---- reference setup restated (weights.cpp / schemes.cpp) -------------------
double power_step(uint64_t k, double p) {  // weights.cpp:8-16
    if (k == 0) return 1.0;
    const double kd = (double)k;
    if (k > 1000000) return std::pow(kd, p) * std::expm1(p * std::log1p(1.0 / kd));
    return std::pow(kd + 1.0, p) - std::pow(kd, p);
}

int validate(const ft_problem& s) {  // schemes.cpp:58-78
    const bool wave = s.scheme == FT_SCHEME_WAVE;
    if (s.scheme != FT_SCHEME_ODE && s.scheme != FT_SCHEME_HYPERBOLIC && s.scheme != FT_SCHEME_WAVE &&
        s.scheme != FT_SCHEME_DIFFUSION)
        return set_err(FT_EINVAL, "solve: unknown scheme");
    if (wave) {
        if (!(s.gamma > 1.0 && s.gamma < 2.0))
            return set_err(FT_EINVAL, "ProblemSpec: wave scheme needs gamma in (1, 2)");
    } else if (!(s.gamma > 0.0 && s.gamma < 1.0)) {
        return set_err(FT_EINVAL, "ProblemSpec: scheme needs gamma in (0, 1)");
    }
    if (s.time_steps < 1) return set_err(FT_EINVAL, "ProblemSpec: need at least 1 time step");
    if (s.scheme != FT_SCHEME_ODE && s.space_cells < 2)
        return set_err(FT_EINVAL, "ProblemSpec: need at least 2 space cells");
    if (!(s.time_length > 0.0) || (s.scheme != FT_SCHEME_ODE && !(s.space_length > 0.0)))
        return set_err(FT_EINVAL, "ProblemSpec: domain lengths must be positive");
    return FT_OK;
}

// Constant tridiagonal / upwind operator -> scan parameters (long double).
void scan_params(ft_plan* p, int b, std::vector<double>& lampow) {
    ProblemConst& pc = p->pc_h[b];
    long double lam = 0.0L, phi = 0.0L;
    if (p->kind == SK_TRIDIAG) {
        const long double bb = (long double)pc.off;
        const long double shift = (long double)pc.d - 2.0L * bb;  // exact
        const long double delta = shift / (2.0L * bb);
        phi = 2.0L * asinhl(sqrtl(delta / 2.0L));
        lam = expl(-phi);
        const long double one_m = -expm1l(-phi);
        pc.lam = (double)lam;
        p->G0L[b] = lam / (bb * one_m * (1.0L + lam));
        pc.G0 = (double)p->G0L[b];
        const long double Lam = expl(-phi * (long double)(p->nodes + 1));
        pc.Lam = (double)Lam;
        pc.inv1mL2 = (double)(1.0L / (1.0L - Lam * Lam));
    } else if (p->kind == SK_UPWIND) {
        lam = (long double)pc.off / (long double)pc.d;
        pc.lam = (double)lam;
        p->G0L[b] = 1.0L / (long double)pc.d;
        pc.G0 = (double)p->G0L[b];
        pc.Lam = 0.0;
        pc.inv1mL2 = 1.0;
    } else {
        pc.lam = 0.0;
        pc.G0 = 1.0 / pc.d;
        pc.Lam = 0.0;
        pc.inv1mL2 = 1.0;
    }
    p->lamL[b] = lam;
    double* lp = lampow.data() + (uint64_t)b * p->lp_stride;
    for (int k = 0; k < p->lp_stride; ++k) {
        long double v;
        if (p->kind == SK_TRIDIAG) v = expl(-phi * (long double)k);
        else if (p->kind == SK_UPWIND) v = powl(lam, (long double)k);
        else v = k == 0 ? 1.0L : 0.0L;
        lp[k] = (double)v;
    }
}

// Single-CTA Dirichlet correction  x_i += kF_i F_M + kB_i B_1  (i = q+1):
// alpha lam^i + gam lam^(n+1-i) with alpha, gam from p0 = G0 lam B_1, pM1 = G0 lam F_M.
void dirichlet_coefs(const ft_plan* p, int b, double* kF, double* kB) {
    const int n = p->nodes;
    const long double lam = p->lamL[b], G0 = p->G0L[b];
    const long double phi = -logl(lam);
    const long double Lam = expl(-phi * (long double)(n + 1));
    const long double inv = 1.0L / (1.0L - Lam * Lam);
    for (int q = 0; q < n; ++q) {
        const long double li = expl(-phi * (long double)(q + 1));
        const long double lr = expl(-phi * (long double)(n - q));
        kF[q] = (double)(G0 * lam * inv * (Lam * li - lr));
        kB[q] = (double)(G0 * lam * inv * (Lam * lr - li));
    }
}

// Zero-carry local solve of one slab (long double) -> x, exported carries.
void local_solve_ld(const ft_plan* p, int b, const std::vector<long double>& r, std::vector<long double>& x,
                    long double& cF, long double& cB) {
    const int ms = (int)r.size();
    const long double lam = p->lamL[b], G0 = p->G0L[b];
    std::vector<long double> F(ms), Bk(ms);
    long double acc = 0.0L;
    const bool tri = p->kind == SK_TRIDIAG;
    for (int q = 0; q < ms; ++q) {
        acc = lam * acc + (tri ? r[q] : r[q] * G0);  // upwind: G0 = 1/d
        F[q] = acc;
    }
    acc = 0.0L;
    for (int q = ms - 1; q >= 0; --q) {
        acc = lam * acc + r[q];
        Bk[q] = acc;
    }
    x.resize(ms);
    for (int q = 0; q < ms; ++q) x[q] = tri ? G0 * (F[q] + Bk[q] - r[q]) : F[q];
    cF = F[ms - 1];
    cB = Bk[0];
}

// Space-time responses of a slab of ms nodes to unit left / right injections
// (shapes lam^q, lam^(ms-1-q)) at lag 0: GL, GR [ms][L]; carry responses
// h = (hFL, hFR, hBL, hBR)[L] (lag 0 entries are zero).
void slab_responses(const ft_plan* p, int b, int ms, double* G /*[2][L][m]*/, double* H /*[L][4]*/) {
    const int L = p->L, m = p->slab;
    const double* col = p->col_h.data() + (uint64_t)b * p->N;
    const long double lam = p->lamL[b];
    // Scheme 2 (stencil): the injection is the left neighbour's boundary value itself
    // (EL = F before the slab, not lam F): same-step response lam^(q+1), and the history of
    // the slab's first node also sees that value (B~_j = -A~_j: U_i + U_(i-1))
    const bool st = p->stencil;
    for (int side = 0; side < 2; ++side) {
        std::vector<std::vector<long double>> g(L, std::vector<long double>(ms));
        for (int q = 0; q < ms; ++q)
            g[0][q] = powl(lam, (long double)(side == 0 ? q + (st ? 1 : 0) : ms - 1 - q));
        H[0 * 4 + side] = 0.0;
        H[0 * 4 + 2 + side] = 0.0;
        for (int l = 1; l < L; ++l) {
            std::vector<long double> dr(ms, 0.0L);
            for (int lp = 0; lp < l; ++lp) {
                const long double c = (uint64_t)(l - lp) < p->N ? (long double)col[l - lp] : 0.0L;
                for (int q = 0; q < ms; ++q) dr[q] -= c * g[lp][q];
                if (st) {  // stencil: + the left neighbour of every node (boundary value 1 at lag 0)
                    for (int q = 1; q < ms; ++q) dr[q] -= c * g[lp][q - 1];
                    if (lp == 0 && side == 0) dr[0] -= c;
                }
            }
            long double cF, cB;
            local_solve_ld(p, b, dr, g[l], cF, cB);
            H[l * 4 + side] = (double)cF;
            H[l * 4 + 2 + side] = (double)cB;
        }
        for (int l = 0; l < L; ++l)  // time-major [side][l][q] (coalesced over q on the device)
            for (int q = 0; q < m; ++q) G[((uint64_t)side * L + l) * m + q] = q < ms ? (double)g[l][q] : 0.0;
    }
}

void build_schedule(ft_plan* p) {
    const uint64_t N = p->N, L = (uint64_t)p->L;
    uint64_t Npad = L;
    while (Npad < N) Npad <<= 1;
    p->levels.clear();
    uint64_t off = 0;
    const int pairs = (p->local_nodes + 1) / 2 * p->B;
    for (uint64_t n = 2 * L; n <= Npad; n <<= 1) {
        Level lv;
        lv.n = (int)n;
        if (mp_is_single((int)n)) {  // one CTA per n-point transform, G row pairs per CTA
            lv.K = 1;
            lv.m = (int)n;
            lv.G = (int)n >= kMpTile ? 1 : kMpTile / (int)n;
        } else {
            // cluster split into K branches of m <= kMpBranchMax points
            lv.K = n <= 2 * (uint64_t)kMpBranchMax ? 2 : (int)(n / kMpBranchMax);
            lv.m = (int)(n / lv.K);
            lv.G = lv.m >= kMpTile ? 1 : kMpTile / lv.m;
        }
        if (lv.G > pairs) lv.G = pairs;
        lv.groups = (pairs + lv.G - 1) / lv.G;
        lv.spec_off = off;
        off += (uint64_t)p->B * n;
        p->levels.push_back(lv);
    }
    int logT = 4;
    while ((1ull << logT) < Npad) ++logT;
    p->logT = logT;
    p->ops.clear();
    for (uint64_t t0 = 0; t0 < N; t0 += L) {
        Op leaf{OP_LEAF, t0, (int)std::min<uint64_t>(L, N - t0), 0, 0, 0, t0 == 0};
        p->ops.push_back(leaf);
        const uint64_t t = t0 + L;
        if (t >= N) break;
        const uint64_t h = t & (~t + 1);  // lowest set bit
        int level = 0;
        while ((L << level) < h) ++level;
        Op mp{OP_MP, t - h, 0, level, t, t + h, t - h == 0};
        p->ops.push_back(mp);
    }
}

int alloc_copy(void** dst, const void* src, size_t bytes) {
    FT_CUDA(cudaMalloc(dst, bytes ? bytes : 8));
    if (bytes && src) FT_CUDA(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
    return FT_OK;
}

bool is_pinned_host(const void* ptr) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

bool is_device_ptr(const void* ptr) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int ensure_work(ft_plan* p) {
    if (!p->work_d) FT_CUDA(cudaMalloc(&p->work_d, sizeof(double) * rows_of(p) * p->N));
    return FT_OK;
}

int setup_impl(const ft_problem* probs, uint64_t count, const ft_options* opt, ft_plan** out, int rank = 0,
               int world = 1, const double* custom_cols = nullptr) {
    if (!probs || !out || count == 0) return set_err(FT_EINVAL, "ft_setup: null argument");
    *out = nullptr;
    for (uint64_t b = 0; b < count; ++b) {
        int rc = validate(probs[b]);
        if (rc) return rc;
        const ft_problem& a = probs[b];
        const ft_problem& z = probs[0];
        if (a.scheme != z.scheme || a.time_steps != z.time_steps ||
            (a.scheme != FT_SCHEME_ODE && a.space_cells != z.space_cells))
            return set_err(FT_EINVAL, "ft_setup_batch: problems must share scheme, N and M");
    }
    if (probs[0].time_steps > kMaxTimeSteps)  // history-product kernels exist up to n = 65536 (K <= 16 branches)
        return set_err(FT_ELENGTH, "ft_setup: at most " + std::to_string(kMaxTimeSteps) +
                                       " time steps per problem are supported");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(FT_ECUDA, "no CUDA device available (this library has no CPU path)");
    }
    ft_plan* p = new ft_plan();
    const ft_problem& z = probs[0];
    p->scheme = z.scheme;
    p->B = (int)count;
    p->N = z.time_steps;
    p->cells = z.scheme == FT_SCHEME_ODE ? 0 : z.space_cells;
    p->nodes = z.scheme == FT_SCHEME_ODE ? 1 : (int)(z.space_cells - 1);
    p->tau = z.time_length / (double)z.time_steps;
    p->h = z.scheme == FT_SCHEME_ODE ? 0.0 : z.space_length / (double)z.space_cells;
    p->rhs_mode = opt ? opt->rhs_mode : 0;
    p->report_residual = opt && (opt->flags & FT_OPT_REPORT_RESIDUAL);
    p->J = (opt && opt->near_field > 0) ? opt->near_field : (z.scheme == FT_SCHEME_WAVE ? 64 : 1);
    if (opt && opt->device >= 0) FT_CUDA(cudaSetDevice(opt->device));
    FT_CUDA(cudaGetDevice(&p->device));

    const uint64_t N = p->N;
    p->kind = z.scheme == FT_SCHEME_ODE ? SK_DIAG
              : (z.scheme == FT_SCHEME_WAVE || z.scheme == FT_SCHEME_HYPERBOLIC) ? SK_UPWIND
                                                                               : SK_TRIDIAG;
    p->stencil = z.scheme == FT_SCHEME_HYPERBOLIC;
    p->gamma.resize(count);
    p->mu.resize(count);
    p->c.resize(count);
    p->col_h.assign(count * N, 0.0);
    p->wts_h.assign(count * (N + 1), 0.0);
    p->pc_h.resize(count);
    std::vector<double> dw(count * N, 0.0), cprime, den;
    if (p->kind == SK_TRIDIAG) {
        cprime.assign(count * p->nodes, 0.0);
        den.assign(count * p->nodes, 0.0);
    }
    for (uint64_t b = 0; b < count; ++b) {
        const double g = probs[b].gamma;
        const double tau = probs[b].time_length / (double)probs[b].time_steps;
        const double h = p->h;
        p->gamma[b] = g;
        // SchemeConstants::for_spec (schemes.cpp:44-56)
        const double mu = std::pow(tau, -g) / std::tgamma(2.0 - g);
        double c = mu;
        if (p->scheme == FT_SCHEME_WAVE) c = std::pow(tau, -g) / std::tgamma(3.0 - g);
        if (p->scheme == FT_SCHEME_HYPERBOLIC) c = std::pow(tau, -g) / (2.0 * std::tgamma(2.0 - g));
        if (p->scheme == FT_SCHEME_DIFFUSION) c = std::pow(tau, -g) / std::tgamma(2.0 - g);
        p->mu[b] = mu;
        p->c[b] = c;
        double* col = p->col_h.data() + b * N;
        double* wv = p->wts_h.data() + b * (N + 1);
        ProblemConst& pc = p->pc_h[b];
        pc.c = c;
        pc.h = h;
        if (p->scheme == FT_SCHEME_WAVE) {
            // m_weights(gamma, N+1) and assemble_scheme3_reordered (schemes.cpp:277-287)
            for (uint64_t k = 0; k <= N; ++k) wv[k] = power_step(k, 2.0 - g);
            col[0] = 1.0 / h + c * wv[0];
            if (N > 1) col[1] = c * (wv[1] - 2.0 * wv[0]);
            for (uint64_t j = 2; j < N; ++j) col[j] = c * (wv[j - 2] - 2.0 * wv[j - 1] + wv[j]);
            pc.d = c * wv[0] + 1.0 / h;  // schemes.cpp:348 denominator
            pc.off = 1.0 / h;
            for (uint64_t j = 0; j < N; ++j) dw[b * N + j] = col[j];
        } else {
            // g_weights(gamma, N) (+1 spare for the RHS kernel)
            for (uint64_t k = 0; k <= N; ++k) wv[k] = power_step(k, 1.0 - g);
            if (p->scheme == FT_SCHEME_HYPERBOLIC) {
                // assemble_scheme2_reordered (schemes.cpp:160-165): A~ is the column; the
                // step is A~_0 U_i - B~_0 U_(i-1) = r and, since B~_j = -A~_j for j >= 1,
                // the history acts on U_i + U_(i-1) (the plan's source stencil)
                col[0] = 1.0 / h + c * wv[0];
                for (uint64_t j = 1; j < N; ++j) col[j] = c * (wv[j] - wv[j - 1]);
                pc.d = col[0];
                pc.off = 1.0 / h - c * wv[0];  // B~_0 (either sign)
                // direct path (schemes.cpp:215-217): w = c * (g[j-1] - g[j]), rounded as there
                for (uint64_t j = 1; j < N; ++j) dw[b * N + j] = c * (wv[j - 1] - wv[j]);
            } else if (p->scheme == FT_SCHEME_DIFFUSION) {
                col[0] = 2.0 / (h * h) + c * wv[0];  // schemes.cpp:394-396
                for (uint64_t j = 1; j < N; ++j) col[j] = c * (wv[j] - wv[j - 1]);
                pc.d = col[0];
                pc.off = 1.0 / (h * h);
                for (uint64_t j = 1; j < N; ++j) dw[b * N + j] = wv[j - 1] - wv[j];
                // Thomas factors, schemes.cpp:453-460 (same expressions, same order)
                const double diag = 2.0 / (h * h) + c * wv[0];
                const double off = -1.0 / (h * h);
                double denom = diag;
                cprime[b * p->nodes] = off / denom;
                den[b * p->nodes] = denom;
                for (int i = 1; i < p->nodes; ++i) {
                    denom = diag - off * cprime[b * p->nodes + i - 1];
                    cprime[b * p->nodes + i] = off / denom;
                    den[b * p->nodes + i] = denom;
                }
            } else {
                col[0] = 1.0 + mu * wv[0];  // SURVEY.md 3.4 composition
                for (uint64_t j = 1; j < N; ++j) col[j] = mu * (wv[j] - wv[j - 1]);
                pc.d = col[0];
                pc.off = 0.0;
                for (uint64_t j = 0; j < N; ++j) dw[b * N + j] = col[j];
            }
        }
    }

    if (custom_cols) {  // ft_setup_toeplitz: caller's lower-triangular columns, no scheme
        p->custom = true;
        for (uint64_t b = 0; b < count; ++b) {
            double* col = p->col_h.data() + b * N;
            std::memcpy(col, custom_cols + b * N, sizeof(double) * N);
            p->pc_h[b].d = col[0];
            p->pc_h[b].off = 0.0;
            for (uint64_t j = 0; j < N; ++j) dw[b * N + j] = col[j];
        }
    }

    // leaf configuration
    const int nodes = p->nodes;
    p->local_nodes = nodes;
    // problems at least this wide use the slab (SPIKE) leaf; narrower ones one CTA (tuning knob)
    // (513: config 3, 1024 nodes, 114 -> 92 ms as 2 slabs with L = 32 instead of one CTA with L = 16)
    const int slab_min = getenv("FT_SLAB_MIN") ? atoi(getenv("FT_SLAB_MIN")) : 513;
    if (p->kind == SK_DIAG) {
        p->npt = 1; p->L = 32; p->threads = 32; p->slab = 1; p->P = 1;
    } else if (nodes >= slab_min) {
        p->npt = 2; p->L = 32; p->threads = 256; p->slab = 512;
        p->P = (nodes + p->slab - 1) / p->slab;
        p->multi = true;
    } else if (nodes <= 256) {
        p->npt = 1; p->L = 32; p->threads = ((nodes + 31) / 32) * 32; p->slab = nodes; p->P = 1;
    } else if (nodes <= 512) {
        p->npt = 2; p->L = 32; p->threads = ((nodes + 63) / 64) * 32; p->slab = nodes; p->P = 1;
    } else if (nodes <= 1024) {
        p->npt = 4; p->L = 16; p->threads = ((nodes + 127) / 128) * 32; p->slab = nodes; p->P = 1;
    } else if (nodes <= 2048) {
        p->npt = 8; p->L = 8; p->threads = ((nodes + 255) / 256) * 32; p->slab = nodes; p->P = 1;
    } else {
        p->npt = 2; p->L = 32; p->threads = 256; p->slab = 512;
        p->P = (nodes + p->slab - 1) / p->slab;
        p->multi = true;
        if (p->P > kMaxSlabs) {
            delete p;
            return set_err(FT_EINVAL, "ft_setup: more than " + std::to_string(kMaxSlabs * 512) +
                                          " interior nodes per problem are not supported");
        }
    }
    p->P_local = p->P;
    if (world > 1) {
        if (!p->multi || count != 1 || p->P % world != 0 || rank < 0 || rank >= world) {
            delete p;
            return set_err(FT_EINVAL, "ft_setup_partitioned: needs one problem wider than 2048 nodes whose " +
                                          std::to_string(p->P) + " slabs divide evenly over " +
                                          std::to_string(world) + " ranks");
        }
        p->part_rank = rank;
        p->part_world = world;
        p->P_local = p->P / world;
        p->node_begin = rank * p->P_local * p->slab;
        p->local_nodes = std::min(nodes, (rank + 1) * p->P_local * p->slab) - p->node_begin;
    }
    if ((int)count > kMaxLeafProblems) {
        delete p;
        return set_err(FT_EINVAL, "ft_setup_batch: at most " + std::to_string(kMaxLeafProblems) +
                                      " problems per plan");
    }
    p->leafcol_h.assign(count * 32, 0.0);
    for (uint64_t b = 0; b < count; ++b)
        for (uint64_t j = 1; j < 32 && j < N; ++j) p->leafcol_h[b * 32 + j] = p->col_h[b * N + j];
    p->lp_stride = std::max(nodes + 2, 4098);
    std::vector<double> lampow((uint64_t)count * p->lp_stride);
    p->lamL.assign(count, 0.0L);
    p->G0L.assign(count, 0.0L);
    for (uint64_t b = 0; b < count; ++b) scan_params(p, (int)b, lampow);
    {  // LeafArgs::kc for single-problem plans (kKc* layout; same values as scan_consts reads)
        const double* lp0 = lampow.data();
        auto lpk = [&](int k) { return lp0[std::min(k, p->lp_stride - 1)]; };
        for (int j = 0; j < 32; ++j) p->kc_h[j] = p->leafcol_h[j];
        for (int j = 0; j < 32; ++j) p->kc_h[kKcCol2 + j] = (uint64_t)(32 + j) < N ? p->col_h[32 + j] : 0.0;
        for (int d = 0; d < 5; ++d) p->kc_h[kKcPow + d] = lpk(p->npt << d);
        p->kc_h[kKcLamW] = lpk(32 * p->npt);
        p->kc_h[kKcLam] = p->pc_h[0].lam;
        for (int v = 0; v < 8; ++v) {
            p->kc_h[kKcV1 + v] = v < p->npt ? lpk(v + 1) : 0.0;
            p->kc_h[kKcNv + v] = v < p->npt ? lpk(p->npt - v) : 0.0;
        }
    }
    build_schedule(p);

    // device copies
    const uint64_t B = count;
    int rc;
    if ((rc = alloc_copy((void**)&p->pc_d, p->pc_h.data(), sizeof(ProblemConst) * B))) return rc;
    if ((rc = alloc_copy((void**)&p->col_d, p->col_h.data(), sizeof(double) * B * N))) return rc;
    if ((rc = alloc_copy((void**)&p->wts_d, p->wts_h.data(), sizeof(double) * B * (N + 1)))) return rc;
    if ((rc = alloc_copy((void**)&p->lampow_d, lampow.data(), sizeof(double) * lampow.size()))) return rc;
    if ((rc = alloc_copy((void**)&p->dw_d, dw.data(), sizeof(double) * dw.size()))) return rc;
    if (p->kind == SK_TRIDIAG) {
        if ((rc = alloc_copy((void**)&p->cprime_d, cprime.data(), sizeof(double) * cprime.size()))) return rc;
        if ((rc = alloc_copy((void**)&p->den_d, den.data(), sizeof(double) * den.size()))) return rc;
    }
    if ((rc = alloc_copy((void**)&p->scratch_d, nullptr, sizeof(double) * 2 * B * nodes))) return rc;
    if ((rc = alloc_copy((void**)&p->dmctr_d, nullptr, 2 * sizeof(unsigned)))) return rc;
    if ((rc = alloc_copy((void**)&p->dbgclk_d, nullptr, sizeof(long long) * 16))) return rc;
    if (p->stencil && (rc = alloc_copy((void**)&p->vsrc_d, nullptr, sizeof(double) * rows_of(p) * N))) return rc;
    if (p->multi) {
        // (twice the carries of one leaf: the leaf-pair kernel double-buffers them)
        if ((rc = alloc_copy((void**)&p->xch_d, nullptr, sizeof(double) * 2 * 2 * B * p->P * p->L))) return rc;
        p->xsend_d = p->xch_d;
        if ((rc = alloc_copy((void**)&p->bar_d, nullptr, sizeof(unsigned)))) return rc;
        {
            // the fused leaf needs every slab CTA co-resident (cooperative launch)
            int dev_sms = 0, per_sm = 0;
            FT_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, p->device));
            per_sm = 1;
            // one cooperative kernel per leaf (phase 1, grid barrier, phases 2/3 on the
            // SMEM-resident tile): measured 407 -> 400 ms on cfg4 once the step loop
            // stopped spilling (kernel-parameter constants)
            p->fused_leaf = (int64_t)B * p->P_local <= (int64_t)dev_sms * per_sm && getenv("FT_NO_FUSED_LEAF") == nullptr;
        }
        {   // Scheme 3 problems of a few slabs: chained slabs instead of phase 1 / barrier / correction
            static const int chain_max = getenv("FT_CHAIN_MAX_P") ? atoi(getenv("FT_CHAIN_MAX_P")) : 4;
            p->chain_leaf = p->fused_leaf && p->kind == SK_UPWIND && !p->stencil && p->part_world == 1 &&
                            p->P <= chain_max && p->npt == 2 && p->L == 32;
            if (p->chain_leaf &&
                (rc = alloc_copy((void**)&p->chain_d, nullptr, sizeof(double2) * B * p->P * p->L)))
                return rc;
        }
        const uint64_t gsz = (uint64_t)2 * 2 * p->slab * p->L, hsz = (uint64_t)2 * p->L * 4;
        std::vector<double> G(B * gsz, 0.0), H(B * hsz, 0.0);
        const int mlast = nodes - (p->P - 1) * p->slab;
        for (uint64_t b = 0; b < B; ++b) {
            slab_responses(p, (int)b, p->slab, G.data() + b * gsz, H.data() + b * hsz);
            slab_responses(p, (int)b, mlast, G.data() + b * gsz + gsz / 2, H.data() + b * hsz + hsz / 2);
        }
        // Tridiagonal slabs are mirror symmetric (GR_q = GL_(ms-1-q)): phase 3 corrects the node
        // pair (q, ms-1-q) from the half-sum / half-difference tables
        //   S_q = (GL_q + GR_q) / 2 (side 0),  D_q = (GL_q - GR_q) / 2 (side 1),  q < (ms + 1) / 2,
        // with (EL + ER) and (EL - ER): half the products of the unpaired form (leaf.cu phase 3).
        p->paired_g = p->kind == SK_TRIDIAG && !p->stencil && getenv("FT_NO_PAIRED_G") == nullptr;
        if (p->paired_g) {
            const int m = p->slab, L = p->L;
            for (uint64_t b = 0; b < B; ++b)
                for (int kind = 0; kind < 2; ++kind) {
                    double* g = G.data() + b * gsz + (uint64_t)kind * (gsz / 2);
                    const int ms = kind == 0 ? m : mlast;
                    for (int l = 0; l < L; ++l) {
                        double* gl = g + (uint64_t)l * m;
                        double* gr = g + ((uint64_t)L + l) * m;
                        for (int q = 0; q < m; ++q) {
                            const double A = gl[q], Bv = gr[q];
                            const bool used = q < (ms + 1) / 2;
                            gl[q] = used ? 0.5 * (A + Bv) : 0.0;
                            gr[q] = used ? 0.5 * (A - Bv) : 0.0;
                        }
                    }
                }
        }
        if ((rc = alloc_copy((void**)&p->respg_d, G.data(), sizeof(double) * G.size()))) return rc;
        if ((rc = alloc_copy((void**)&p->resph_d, H.data(), sizeof(double) * H.size()))) return rc;
        // phase 2 as a matvec: tabulate the reduced recursion's response to unit carries
        const uint64_t wsz = B * (uint64_t)p->P * 2 * p->L * 2 * p->P;
        if ((rc = alloc_copy((void**)&p->respw_d, nullptr, sizeof(double) * wsz))) return rc;
        {
            LeafArgs wa{};
            wa.nodes = nodes;
            wa.slab = p->slab;
            wa.P = p->P;
            wa.pc = p->pc_d;
            wa.lampow = p->lampow_d;
            wa.lp_stride = p->lp_stride;
            wa.resp_h = p->resph_d;
            wa.stencil = p->stencil ? 1 : 0;
            FT_CUDA(launch_leaf_wbuild(p->kind, p->L, wa, (int)B, p->respw_d, 0));
            FT_CUDA(cudaDeviceSynchronize());
        }
    } else if (p->kind == SK_TRIDIAG) {
        std::vector<double> kc(B * 2 * nodes);
        for (uint64_t b = 0; b < B; ++b)
            dirichlet_coefs(p, (int)b, kc.data() + b * 2 * nodes, kc.data() + b * 2 * nodes + nodes);
        if ((rc = alloc_copy((void**)&p->kcoef_d, kc.data(), sizeof(double) * kc.size()))) return rc;
    }
    // multi-resolution twiddles tw[S + k] = exp(-2 pi i k / S), S = 1, 2, 4, ..., T (long double)
    {
        const uint64_t T = 1ull << p->logT;
        std::vector<cplx> tw(2 * T);
        const long double pi = 3.141592653589793238462643383279502884L;
        tw[0] = {1.0, 0.0};
        for (uint64_t S = 1; S <= T; S <<= 1)
            for (uint64_t k = 0; k < S; ++k) {
                const long double ang = 2.0L * pi * (long double)k / (long double)S;
                tw[S + k] = {(double)cosl(ang), (double)(-sinl(ang))};
            }
        if ((rc = alloc_copy((void**)&p->tw_d, tw.data(), sizeof(cplx) * 2 * T))) return rc;
    }
    FT_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    p->own_stream = true;
    FT_CUDA(cudaEventCreate(&p->ev0));
    FT_CUDA(cudaEventCreate(&p->ev1));
    // kernel spectra per level (embed_circulant equivalent)
    uint64_t spec_total = 0;
    for (auto& lv : p->levels) spec_total += (uint64_t)B * lv.n;
    if ((rc = alloc_copy((void**)&p->spec_d, nullptr, sizeof(cplx) * std::max<uint64_t>(spec_total, 1)))) return rc;
    for (auto& lv : p->levels) {
        if (lv.K == 1)
            FT_CUDA(launch_spectra_single(p->col_d, N, (int)B, lv.n, p->J, p->spec_d + lv.spec_off, p->tw_d,
                                          p->stream));
        else
            FT_CUDA(launch_spectra(p->col_d, N, (int)B, lv.n, lv.m, lv.K, p->J, p->spec_d + lv.spec_off,
                                   p->tw_d, p->logT, p->stream));
    }
    {
        bool needs = false;
        p->split_min_k = getenv("FT_SPLIT_MIN_K") ? atoi(getenv("FT_SPLIT_MIN_K")) : 8;  // tuning knob
        for (auto& lv : p->levels) needs = needs || lv.K >= p->split_min_k;
        p->split_k = getenv("FT_CLUSTER_K") == nullptr;
        if (needs && p->split_k)
            if ((rc = alloc_copy((void**)&p->mpscratch_d, nullptr, kMpScratchBytes))) return rc;
    }
    FT_CUDA(cudaStreamSynchronize(p->stream));
    *out = p;
    return FT_OK;
}

// Holds the batched-plan leaf weight bank for the enqueue of one solve.
struct BankScope {
    const ft_plan* p;
    bool on;
    cudaError_t err = cudaSuccess;
    BankScope(const ft_plan* plan, bool enable) : p(plan), on(enable) {
        if (on) {
            err = leaf_bank_acquire(p, p->leafcol_h.data(), p->B, p->stream);
            if (err != cudaSuccess) on = false;  // acquire unlocked on failure
        }
    }
    ~BankScope() {
        if (on) leaf_bank_release(p, p->stream);
    }
};

// Streamed host solve: the caller's R arrives in time chunks of C steps on a
// copy stream and is added by the leaf that solves those steps (history
// products accumulate into a zeroed X, linear in R); finished chunks of U
// leave on a second copy stream as soon as their last leaf is done.  PCIe
// traffic in both directions overlaps the solve.
struct GenRhs {                   // fused separable RHS (ft_solve_fast_modes)
    const double* A = nullptr;
    const double* T = nullptr;
    int J = 0;
};

struct StreamIO {
    uint64_t C = 0;               // chunk steps (multiple of the leaf length)
    bool defer = false;           // R streamed into rdev (leaves add it)
    const double* rdev = nullptr;
    double* u_host = nullptr;     // non-null: stream U chunks back
    uint64_t waited = 0;          // H2D chunks the compute stream has waited for
};

int run_fast(ft_plan* p, double* X, const double* rhs, uint64_t* launches,
             std::vector<cudaEvent_t>* evs = nullptr, StreamIO* io = nullptr, const GenRhs* gen = nullptr) {
    const cudaStream_t st = p->stream;
    const uint64_t N = p->N;
    // batched plans read their leaf weights from the per-device constant bank: own it for
    // the enqueue (a captured graph gets it from launch_fast at each replay)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    FT_CUDA(cudaStreamIsCapturing(st, &cap));
    BankScope bank(p, p->B > 1 && cap == cudaStreamCaptureStatusNone);
    if (bank.err != cudaSuccess) return set_err(FT_ECUDA, "leaf weight bank upload failed");
    uint64_t nl = 0;
    unsigned leaf_index = 0;
    // the n = 64 history products fold into the next (cooperative slab) leaf
    // (wide problems only: for config 3's two slabs the standalone product is cheaper, 100 vs 102 ms)
    const bool fuse0 = fuse0_plan(p) && !io && !gen;
    bool pend0 = false, pend0_first = false;
    p->last_fuse0 = fuse0;
    if (p->multi && p->part_world == 1 && p->fused_leaf) FT_CUDA(cudaMemsetAsync(p->bar_d, 0, sizeof(unsigned), st));
    const bool chain = p->chain_leaf && !p->p2p;
    if (chain) FT_CUDA(cudaMemsetAsync(p->chain_d, 0, sizeof(double2) * p->B * p->P * p->L, st));
    int leaves_total = 0;
    for (const Op& o : p->ops) leaves_total += o.kind == OP_LEAF ? 1 : 0;
    if (p->p2p) FT_CUDA(launch_p2p_epoch(reinterpret_cast<unsigned*>((char*)p->p2p_block + 8), st));
    for (size_t oi = 0; oi < p->ops.size(); ++oi) {
        const Op& op = p->ops[oi];
        if (evs) FT_CUDA(cudaEventRecord((*evs)[oi], st));
        if (op.kind == OP_LEAF) {
            LeafArgs a;
            a.X = X;
            a.V = p->stencil ? p->vsrc_d : nullptr;
            a.stencil = p->stencil ? 1 : 0;
            const bool defer = io && io->defer;
            a.src = (op.first && !defer) ? rhs : X;
            a.src2 = nullptr;
            a.radd = defer ? io->rdev : nullptr;
            a.fuse0 = (fuse0 && pend0) ? 1 : 0;
            if (a.fuse0 && pend0_first) a.src = rhs;  // the skipped product was this tile's first touch
            pend0 = false;
            a.genA = gen ? gen->A : nullptr;
            a.genT = gen ? gen->T : nullptr;
            a.genJ = gen ? gen->J : 0;
            if (gen && op.first) a.src = nullptr;  // nothing accumulated in X yet: history starts at zero
            if (defer) {  // this leaf's R chunk must have landed
                const uint64_t c = op.t0 / io->C;
                if (c >= io->waited) {
                    FT_CUDA(cudaStreamWaitEvent(st, p->h2d_ev[c], 0));
                    io->waited = c + 1;
                }
            }
            a.N = N;
            a.t0 = op.t0;
            a.len = op.len;
            a.nodes = p->nodes;
            a.slab = p->slab;
            a.P = p->P;
            a.pc = p->pc_d;
            a.col = p->col_d;
            a.lampow = p->lampow_d;
            a.lp_stride = p->lp_stride;
            a.kcoef = p->kcoef_d;
            a.xch = p->xch_d;
            a.xsend = p->xsend_d;
            a.chain = p->chain_d;
            a.chain_tag = (double)(leaf_index + 1);
            a.P_local = p->P_local;
            a.s_begin = p->part_rank * p->P_local;
            a.node_begin = p->node_begin;
            a.rows_pp = p->local_nodes;
            a.resp_g = p->respg_d;
            a.paired_g = p->paired_g ? 1 : 0;
            a.resp_h = p->resph_d;
            a.resp_w = p->respw_d;
            a.kc_valid = p->B == 1 && !g_no_kc;
            std::memcpy(a.kc, p->kc_h, sizeof(a.kc));
            a.pdl_trigger = pdl_mode() == 1;
            a.dbg = g_leaf_dbg;
            a.dbg_clk = (g_leaf_dbg & 4) ? p->dbgclk_d : nullptr;
            a.bar = p->bar_d;
            a.bar_target = (unsigned)(leaf_index + 1) * (unsigned)(p->B * p->P_local);
            ++leaf_index;
            a.p2p_peers = p->p2p_peers_d;
            a.p2p_epoch = p->p2p ? reinterpret_cast<const unsigned*>((const char*)p->p2p_block + 8) : nullptr;
            a.p2p_world = p->part_world;
            a.p2p_leaf = (int)leaf_index - 1;
            a.p2p_leaves = leaves_total;
            // leaves 2i and 2i+1 with only the (folded) level-0 product between them: one kernel
            bool pair = false;
            if (fuse0 && !a.fuse0 && !p->p2p && p->multi && p->part_world == 1 && p->fused_leaf &&
                oi + 2 < p->ops.size() && p->ops[oi + 1].kind != OP_LEAF && p->ops[oi + 1].level == 0 &&
                p->ops[oi + 2].kind == OP_LEAF && p->ops[oi + 2].len == p->L && leaf_pair_ok(a, p->L)) {
                a.src2 = p->ops[oi + 1].first ? rhs : X;  // the folded product was that tile's first touch
                pair = true;
            }
            if (pair) {
                FT_CUDA(launch_leaf_pair(p->kind, p->npt, p->L, a, p->B * p->P_local, st));
                ++leaf_index;
                if (evs) {  // per-op timing: the pair's time is charged to its first leaf
                    FT_CUDA(cudaEventRecord((*evs)[oi + 1], st));
                    FT_CUDA(cudaEventRecord((*evs)[oi + 2], st));
                }
                oi += 2;
            } else
            if (p->p2p) {  // exchange inside the kernel over peer memory: no hook, no second kernel
                a.xch = reinterpret_cast<double*>((char*)p->p2p_block + kP2pHeader) +
                        (size_t)(a.p2p_leaf & 1) * p->P * p->L * 2;
                FT_CUDA(launch_leaf_p2p(p->kind, p->npt, p->L, a, p->B * p->P_local, st));
            } else if (chain) {
                FT_CUDA(launch_leaf_chain(p->kind, p->npt, p->L, a, p->B * p->P_local, st));
            } else if (p->multi && p->part_world == 1 && p->fused_leaf) {
                FT_CUDA(launch_leaf_fused(p->kind, p->npt, p->L, a, p->B * p->P_local, st));
            } else {
                FT_CUDA(launch_leaf(p->kind, p->npt, p->L, p->multi, a, p->B * p->P_local, p->threads, st));
            }
            if (p->multi && !p->p2p && !(p->part_world == 1 && p->fused_leaf)) {
                if (p->nccl_comm) {  // one carry all-gather per leaf: NCCL on the plan's stream (graph-capturable)
                    const int nr = nccl_api().AllGather(p->xsend_d, p->xch_d, (size_t)p->P_local * p->L * 2,
                                                        kNcclFloat64, p->nccl_comm, st);
                    if (nr) return set_err(FT_ESOLVER, std::string("ncclAllGather: ") + nccl_api().GetErrorString(nr));
                } else if (p->part_world > 1) {  // the caller's collective
                    if (!p->exchange)
                        return set_err(FT_EINVAL, "partitioned plan: no exchange hook (ft_set_exchange / ft_nccl_init)");
                    const int rc = p->exchange(p->exchange_user, (uint64_t)p->P_local * p->L * 2, (void*)st);
                    if (rc) return set_err(FT_ESOLVER, "partitioned plan: exchange hook failed");
                }
                FT_CUDA(launch_leaf_correct(p->kind, p->npt, p->L, a, p->B * p->P_local, st));
                ++nl;
            }
            if (io && io->u_host) {  // a finished chunk of U goes back while the solve continues
                const uint64_t end = op.t0 + (uint64_t)op.len;
                if (end % io->C == 0 || end == N) {
                    const uint64_t c = (end - 1) / io->C, c0 = c * io->C, w = end - c0;
                    FT_CUDA(cudaEventRecord(p->d2h_ev[c], st));
                    FT_CUDA(cudaStreamWaitEvent(p->d2h_st, p->d2h_ev[c], 0));
                    FT_CUDA(cudaMemcpy2DAsync(io->u_host + c0, sizeof(double) * N, X + c0, sizeof(double) * N,
                                              sizeof(double) * w, rows_of(p), cudaMemcpyDeviceToHost, p->d2h_st));
                }
            }
        } else {
            if (fuse0 && op.level == 0 && oi + 1 < p->ops.size() && p->ops[oi + 1].kind == OP_LEAF) {
                pend0 = true;  // applied by the next leaf kernel
                pend0_first = op.first;
                continue;
            }
            const Level& lv = p->levels[op.level];
            MpArgs a;
            a.X = X;
            a.U = p->stencil ? p->vsrc_d : X;
            a.pdl_trigger = pdl_mode() == 1;
            a.rsrc = (op.first && !(io && io->defer)) ? rhs : X;
            if (gen && op.first) a.rsrc = nullptr;  // first touch of these targets: the history starts at zero
            a.N = N;
            a.lo = op.t0;
            a.mid = op.mid;
            a.hi = op.hi;
            a.n = lv.n;
            a.m = lv.m;
            a.K = lv.K;
            a.G = lv.G;
            a.rows = (int)rows_of(p);
            a.nodes = p->local_nodes;
            a.pairs_per_problem = (p->local_nodes + 1) / 2;
            a.spec = p->spec_d + lv.spec_off;
            a.tw = p->tw_d;
            a.logT = p->logT;
            a.col = p->col_d;
            a.J = p->J;
            a.scratch = (lv.K >= p->split_min_k && p->split_k) ? p->mpscratch_d : nullptr;  // K = 4: clusters measured faster
            a.pair_begin = 0;
            a.pair_count = 0;
            FT_CUDA(launch_mp(a, lv.groups, st));
            nl += mp_kernel_count(a) - 1;  // split levels launch several kernels per product
        }
        ++nl;
    }
    if (evs) FT_CUDA(cudaEventRecord(evs->back(), st));
    if (launches) *launches = nl;
    return FT_OK;
}

}  // namespace

extern "C" {

const char* ft_last_error(void) { return g_err.c_str(); }

int ft_setup_toeplitz(const double* first_cols, uint64_t n, uint64_t count, const ft_options* options,
                      ft_plan** out) {
    if (!first_cols || !out || n == 0 || count == 0) return set_err(FT_EINVAL, "ft_setup_toeplitz: bad argument");
    if (is_device_ptr(first_cols)) return set_err(FT_EINVAL, "ft_setup_toeplitz: host columns expected");
    for (uint64_t b = 0; b < count; ++b)  // toeplitz.cpp:175-176
        if (first_cols[b * n] == 0.0) return set_err(FT_ESOLVER, "lower_toeplitz_forward_solve: zero diagonal");
    std::vector<ft_problem> probs(count, ft_problem{FT_SCHEME_ODE, 0.5, n, 0, 1.0, 1.0});
    return setup_impl(probs.data(), count, options, out, 0, 1, first_cols);
}

// y = T x (or the block operator) for count vectors; col/row/x/y host or device
static int toeplitz_apply(const double* col, const double* row, uint64_t n, uint64_t count, const double* x,
                          double* y, double beta, int block_mode) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(FT_ECUDA, "no CUDA device available (this library has no CPU path)");
    }
    const cudaStream_t st = cudaStreamPerThread;
    const size_t vb = sizeof(double) * n * count, cb = sizeof(double) * n;
    double *dcol = nullptr, *drow = nullptr, *dx = nullptr, *dy = nullptr;
    auto cleanup = [&]() {
        if (dcol) cudaFree(dcol);
        if (drow) cudaFree(drow);
        if (dx && dx != x) cudaFree(dx);
        if (dy && dy != y) cudaFree(dy);
    };
    std::vector<double> lrow;
    if (!row) {  // ToeplitzOperator::lower_triangular (toeplitz.cpp:42-47)
        double c0 = 0.0;
        if (is_device_ptr(col)) {
            if (cudaMemcpy(&c0, col, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) return set_err(FT_ECUDA, "copy");
        } else {
            c0 = col[0];
        }
        lrow.assign(n, 0.0);
        lrow[0] = c0;
        row = lrow.data();
    }
    if (cudaMalloc(&dcol, cb) != cudaSuccess || cudaMalloc(&drow, cb) != cudaSuccess) {
        cleanup();
        return set_err(FT_ENOMEM, "toeplitz matvec: device allocation failed");
    }
    cudaMemcpyAsync(dcol, col, cb, cudaMemcpyDefault, st);
    cudaMemcpyAsync(drow, row, cb, cudaMemcpyDefault, st);
    double c0 = 0.0, r0 = 0.0;
    cudaMemcpyAsync(&c0, dcol, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&r0, drow, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (c0 != r0) {  // toeplitz.cpp:31-32
        cleanup();
        return set_err(FT_EINVAL, "ToeplitzOperator: first_col[0] must equal first_row[0]");
    }
    const bool xdev = is_device_ptr(x), ydev = is_device_ptr(y);
    dx = const_cast<double*>(x);
    dy = y;
    if (!xdev || x == y) {  // in place needs a copy of x (block mode reads neighbours)
        if (cudaMalloc(&dx, vb) != cudaSuccess) {
            dx = nullptr;
            cleanup();
            return set_err(FT_ENOMEM, "toeplitz matvec: device allocation failed");
        }
        cudaMemcpyAsync(dx, x, vb, cudaMemcpyDefault, st);
    }
    if (!ydev) {
        if (cudaMalloc(&dy, vb) != cudaSuccess) {
            dy = nullptr;
            cleanup();
            return set_err(FT_ENOMEM, "toeplitz matvec: device allocation failed");
        }
    }
    cudaError_t e = launch_toeplitz_matvec(dcol, drow, n, dx, dy, beta, block_mode, count, st);
    if (e == cudaSuccess && !ydev) e = cudaMemcpyAsync(y, dy, vb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cleanup();
    if (e != cudaSuccess) return set_err(FT_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e));
    return FT_OK;
}

int ft_toeplitz_matvec(const double* first_col, const double* first_row, uint64_t n, uint64_t count,
                       const double* x, double* y) {
    if (!first_col || !x || !y || count == 0) return set_err(FT_EINVAL, "ft_toeplitz_matvec: null argument");
    if (n == 0) return set_err(FT_EINVAL, "ToeplitzOperator: empty first column");
    return toeplitz_apply(first_col, first_row, n, count, x, y, 0.0, 0);
}

int ft_block_matvec(const double* first_col, const double* first_row, uint64_t n, uint64_t m_blocks,
                    double off_scale, const double* x, double* y) {
    if (!first_col || !x || !y) return set_err(FT_EINVAL, "ft_block_matvec: null argument");
    if (n == 0) return set_err(FT_EINVAL, "ToeplitzOperator: empty first column");
    if (m_blocks == 0) return set_err(FT_EINVAL, "BlockTridiagonalToeplitzOperator: need at least one block");
    return toeplitz_apply(first_col, first_row, n, m_blocks, x, y, off_scale, 1);
}

int ft_setup(const ft_problem* problem, const ft_options* options, ft_plan** out) {
    return setup_impl(problem, 1, options, out);
}

int ft_setup_batch(const ft_problem* problems, uint64_t count, const ft_options* options,
                   ft_plan** out) {
    return setup_impl(problems, count, options, out);
}

int ft_setup_partitioned(const ft_problem* problem, const ft_options* options, int rank, int world,
                         ft_plan** out) {
    return setup_impl(problem, 1, options, out, rank, world);
}

int ft_p2p_handle(ft_plan* p, void* handle_out) {
    if (!p || !handle_out) return set_err(FT_EINVAL, "ft_p2p_handle: null argument");
    if (p->part_world <= 1 || !p->multi || p->B != 1) return set_err(FT_EINVAL, "ft_p2p_handle: plan is not partitioned");
    FT_CUDA(cudaSetDevice(p->device));
    if (!p->p2p_block) {
        const size_t bytes = kP2pHeader + sizeof(double) * 2 * (size_t)p->P * p->L * 2;
        FT_CUDA(cudaMalloc(&p->p2p_block, bytes));
        FT_CUDA(cudaMemset(p->p2p_block, 0, bytes));
    }
    cudaIpcMemHandle_t h;
    FT_CUDA(cudaIpcGetMemHandle(&h, p->p2p_block));
    std::memcpy(handle_out, &h, sizeof(h));
    return FT_OK;
}

int ft_p2p_connect(ft_plan* p, const void* handles) {
    if (!p || !handles) return set_err(FT_EINVAL, "ft_p2p_connect: null argument");
    if (!p->p2p_block) return set_err(FT_EINVAL, "ft_p2p_connect: call ft_p2p_handle first");
    FT_CUDA(cudaSetDevice(p->device));
    std::vector<unsigned long long> bases(p->part_world);
    for (int r = 0; r < p->part_world; ++r) {
        if (r == p->part_rank) {
            bases[r] = (unsigned long long)(uintptr_t)p->p2p_block;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, (const char*)handles + (size_t)r * sizeof(h), sizeof(h));
        void* ptr = nullptr;
        FT_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        p->p2p_opened.push_back(ptr);
        bases[r] = (unsigned long long)(uintptr_t)ptr;
    }
    if (!p->p2p_peers_d) FT_CUDA(cudaMalloc(&p->p2p_peers_d, sizeof(unsigned long long) * p->part_world));
    FT_CUDA(cudaMemcpy(p->p2p_peers_d, bases.data(), sizeof(unsigned long long) * p->part_world,
                       cudaMemcpyHostToDevice));
    int dev_sms = 0;
    FT_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, p->device));
    if (p->P_local > dev_sms) return set_err(FT_EINVAL, "ft_p2p_connect: more slabs per rank than SMs");
    p->p2p = true;
    if (p->graph) cudaGraphExecDestroy(p->graph);
    p->graph = nullptr;
    return FT_OK;
}

int ft_nccl_unique_id(void* id128) {
    if (!id128) return set_err(FT_EINVAL, "ft_nccl_unique_id: null argument");
    if (!nccl_api().ok) return set_err(FT_ESOLVER, "NCCL not found (libnccl.so.2; set FT_NCCL_LIB)");
    NcclId id;
    const int nr = nccl_api().GetUniqueId(&id);
    if (nr) return set_err(FT_ESOLVER, std::string("ncclGetUniqueId: ") + nccl_api().GetErrorString(nr));
    std::memcpy(id128, id.bytes, sizeof(id.bytes));
    return FT_OK;
}

int ft_nccl_init(ft_plan* p, const void* id128, int rank, int world) {
    if (!p || !id128) return set_err(FT_EINVAL, "ft_nccl_init: null argument");
    if (!p->multi) return set_err(FT_EINVAL, "ft_nccl_init: the plan has no slab leaf (a single slab needs no exchange)");
    if (world != p->part_world || rank != p->part_rank)
        return set_err(FT_EINVAL, "ft_nccl_init: rank / world differ from the plan's partition");
    if (p->B != 1) return set_err(FT_EINVAL, "ft_nccl_init: single-problem plans only");
    if (p->p2p) return set_err(FT_EINVAL, "ft_nccl_init: the plan already exchanges over peer memory");
    if (!nccl_api().ok) return set_err(FT_ESOLVER, "NCCL not found (libnccl.so.2; set FT_NCCL_LIB)");
    FT_CUDA(cudaSetDevice(p->device));
    if (p->nccl_comm) {
        nccl_api().CommDestroy(p->nccl_comm);
        p->nccl_comm = nullptr;
    }
    NcclId id;
    std::memcpy(id.bytes, id128, sizeof(id.bytes));
    void* comm = nullptr;
    const int nr = nccl_api().CommInitRank(&comm, world, id, rank);
    if (nr) return set_err(FT_ESOLVER, std::string("ncclCommInitRank: ") + nccl_api().GetErrorString(nr));
    p->nccl_comm = comm;
    // in-place all-gather: this rank's phase-1 carries go straight into its block of the
    // gathered array (the plan's own buffer, [P][L][2], rank-major = slab-major)
    if (!p->own_xch) {
        p->xch_d = nullptr;
        const int rc = alloc_copy((void**)&p->xch_d, nullptr, sizeof(double) * 2 * 2 * p->B * p->P * p->L);
        if (rc) return rc;
        p->own_xch = true;
    }
    p->xsend_d = p->xch_d + (size_t)rank * p->P_local * p->L * 2;
    p->exchange = nullptr;
    // the collective sits between phase 1 and the correction: two kernels per leaf (also for
    // world = 1, which exercises this path on one GPU)
    p->fused_leaf = false;
    p->chain_leaf = false;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    return FT_OK;
}

int ft_set_exchange(ft_plan* p, ft_exchange_fn fn, void* user, double* send_device, double* recv_device) {
    if (!p || !fn || !send_device || !recv_device) return set_err(FT_EINVAL, "ft_set_exchange: null argument");
    if (p->part_world <= 1) return set_err(FT_EINVAL, "ft_set_exchange: plan is not partitioned");
    if ((reinterpret_cast<uintptr_t>(send_device) | reinterpret_cast<uintptr_t>(recv_device)) & 15)
        return set_err(FT_EINVAL, "ft_set_exchange: carry buffers must be 16-byte aligned");
    p->exchange = fn;
    p->exchange_user = user;
    p->xsend_d = send_device;
    if (p->xch_d) cudaFree(p->xch_d);
    p->xch_d = recv_device;
    p->own_xch = false;
    return FT_OK;
}

int ft_plan_get_info(const ft_plan* p, ft_plan_info* info) {
    if (!p || !info) return set_err(FT_EINVAL, "ft_plan_get_info: null argument");
    info->problems = p->B;
    info->nodes = p->nodes;
    info->time_steps = p->N;
    info->leaf = p->L;
    info->levels = p->levels.size();
    info->slabs = p->P;
    info->rank = p->part_rank;
    info->world = p->part_world;
    info->node_begin = p->node_begin;
    info->local_nodes = p->local_nodes;
    info->slabs_local = p->P_local;
    uint64_t f = 0;
    if (p->multi) f |= FT_PLAN_SLAB_LEAF;
    if (p->multi && p->part_world == 1 && p->fused_leaf) f |= FT_PLAN_FUSED_LEAF;
    if (fuse0_plan(p)) f |= FT_PLAN_FUSE0;
    for (const auto& lv : p->levels) {
        if (lv.K > 1 && !(lv.K >= p->split_min_k && p->split_k)) f |= FT_PLAN_CLUSTER_MP;
        if (lv.K >= p->split_min_k && p->split_k) f |= FT_PLAN_SPLIT_MP;
    }
    if (ode_whole_plan(p)) f |= FT_PLAN_ODE_WHOLE;
    info->flags = f;
    info->h = p->h;
    info->tau = p->tau;
    info->mu = p->mu[0];
    info->c = p->c[0];
    return FT_OK;
}

int ft_column(const ft_plan* p, uint64_t problem, double* col) {
    if (!p || !col || problem >= (uint64_t)p->B) return set_err(FT_EINVAL, "ft_column: bad argument");
    std::memcpy(col, p->col_h.data() + problem * p->N, sizeof(double) * p->N);
    return FT_OK;
}

int ft_set_stream(ft_plan* p, void* s) {
    if (!p) return set_err(FT_EINVAL, "ft_set_stream: null plan");
    if (p->own_stream) cudaStreamDestroy(p->stream);
    p->stream = (cudaStream_t)s;
    p->own_stream = false;
    return FT_OK;
}

// assemble_scheme4 rhs (schemes.cpp:401-408) / Scheme3Rhs (:300-306) / ODE
int ft_assemble_rhs(const ft_plan* p, ft_forcing_fn f, ft_initial_fn u0, ft_initial_fn phi,
                    void* user, double* rhs) {
    if (p && p->custom) return set_err(FT_EINVAL, "ft_assemble_rhs: plan from ft_setup_toeplitz has no scheme");
    if (!p || !rhs) return set_err(FT_EINVAL, "ft_assemble_rhs: null argument");
    if (!f) return set_err(FT_EINVAL, "ProblemSpec: forcing callback is required");
    const uint64_t N = p->N;
    for (int b = 0; b < p->B; ++b) {
        const double c = p->c[b], tau = p->tau, h = p->h;
        const double* w = p->wts_h.data() + (uint64_t)b * (N + 1);
        for (int i = 1; i <= p->nodes; ++i) {
            const double x = p->scheme == FT_SCHEME_ODE ? 0.0 : (double)i * h;
            const double u = u0 ? u0(x, user) : 0.0;
            const double ph = phi ? phi(x, user) : 0.0;
            double* r = rhs + ((uint64_t)b * p->nodes + (i - 1)) * N;
            if (p->scheme == FT_SCHEME_HYPERBOLIC) {  // Scheme2Rhs (schemes.cpp:176-187)
                const double us = (u0 ? u0((double)i * h, user) : 0.0) + (u0 ? u0((double)(i - 1) * h, user) : 0.0);
                const double x_half = ((double)i - 0.5) * h;
                for (uint64_t n = 1; n <= N; ++n) r[n - 1] = f(x_half, (double)n * tau, user) + c * w[n - 1] * us;
                continue;
            }
            for (uint64_t n = 1; n <= N; ++n) {
                if (p->scheme == FT_SCHEME_WAVE) {
                    const double t_half = ((double)n - 0.5) * tau;
                    double value = f(x, t_half, user) + c * tau * w[n - 1] * ph;
                    if (n >= 2) value -= c * (w[n - 2] - w[n - 1]) * u;
                    else if (p->rhs_mode == FT_RHS_CORRECTED_N1) value += c * w[0] * u;
                    r[n - 1] = value;
                } else {
                    r[n - 1] = f(x, (double)n * tau, user) + c * w[n - 1] * u;
                }
            }
        }
    }
    return FT_OK;
}

int ft_assemble_rhs_grid(const ft_plan* p, const double* F, const double* u0, const double* phi,
                         double* rhs) {
    if (p && p->custom) return set_err(FT_EINVAL, "ft_assemble_rhs: plan from ft_setup_toeplitz has no scheme");
    if (!p || !F || !rhs) return set_err(FT_EINVAL, "ft_assemble_rhs_grid: null argument");
    if (is_device_ptr(F) || is_device_ptr(rhs))
        return set_err(FT_EINVAL, "ft_assemble_rhs_grid: host arrays expected");
    const uint64_t N = p->N;
    for (int b = 0; b < p->B; ++b) {
        const double c = p->c[b], tau = p->tau;
        const double* w = p->wts_h.data() + (uint64_t)b * (N + 1);
        for (int i = 0; i < p->nodes; ++i) {
            const uint64_t row = (uint64_t)b * p->nodes + i;
            const double u = u0 ? u0[row] : 0.0;
            const double ph = phi ? phi[row] : 0.0;
            const double* Fr = F + row * N;
            double* r = rhs + row * N;
            if (p->scheme == FT_SCHEME_HYPERBOLIC) {  // u0 holds x_0..x_{cells-1} per problem
                const double* ub = u0 ? u0 + (uint64_t)b * (p->nodes + 1) : nullptr;
                const double us = ub ? ub[i + 1] + ub[i] : 0.0;
                for (uint64_t n = 1; n <= N; ++n) r[n - 1] = Fr[n - 1] + c * w[n - 1] * us;
                continue;
            }
            for (uint64_t n = 1; n <= N; ++n) {
                if (p->scheme == FT_SCHEME_WAVE) {
                    double value = Fr[n - 1] + c * tau * w[n - 1] * ph;
                    if (n >= 2) value -= c * (w[n - 2] - w[n - 1]) * u;
                    else if (p->rhs_mode == FT_RHS_CORRECTED_N1) value += c * w[0] * u;
                    r[n - 1] = value;
                } else {
                    r[n - 1] = Fr[n - 1] + c * w[n - 1] * u;
                }
            }
        }
    }
    return FT_OK;
}

int ft_assemble_rhs_modes(const ft_plan* p, int nmodes, const double* a, const double* k,
                          const double* pe, const int* trig, const double* u0amp,
                          const double* phiamp, double* rhs) {
    if (p && p->custom) return set_err(FT_EINVAL, "ft_assemble_rhs: plan from ft_setup_toeplitz has no scheme");
    if (!p || !rhs || nmodes < 0 || (nmodes && (!a || !k || !pe || !trig)))
        return set_err(FT_EINVAL, "ft_assemble_rhs_modes: bad argument");
    if (!is_device_ptr(rhs)) return set_err(FT_EINVAL, "ft_assemble_rhs_modes: rhs must be device memory");
    FT_CUDA(cudaSetDevice(p->device));
    const int B = p->B;
    std::vector<double> cv(B);
    for (int b = 0; b < B; ++b) cv[b] = p->c[b];
    double *a_d, *k_d, *p_d, *c_d, *u_d = nullptr, *f_d = nullptr;
    int* t_d;
    int rc;
    if ((rc = alloc_copy((void**)&a_d, a, sizeof(double) * B * nmodes))) return rc;
    if ((rc = alloc_copy((void**)&k_d, k, sizeof(double) * nmodes))) return rc;
    if ((rc = alloc_copy((void**)&p_d, pe, sizeof(double) * B * nmodes))) return rc;
    if ((rc = alloc_copy((void**)&t_d, trig, sizeof(int) * nmodes))) return rc;
    if ((rc = alloc_copy((void**)&c_d, cv.data(), sizeof(double) * B))) return rc;
    if (u0amp && (rc = alloc_copy((void**)&u_d, u0amp, sizeof(double) * B))) return rc;
    if (phiamp && (rc = alloc_copy((void**)&f_d, phiamp, sizeof(double) * B))) return rc;
    RhsModesArgs ra;
    ra.R = rhs;
    ra.N = p->N;
    ra.nodes = p->local_nodes;
    ra.B = B;
    ra.nmodes = nmodes;
    ra.scheme = p->scheme;
    ra.rhs_mode = p->rhs_mode;
    ra.node_begin = p->node_begin;
    ra.h = p->h;
    ra.tau = p->tau;
    ra.a = a_d;
    ra.k = k_d;
    ra.p = p_d;
    ra.trig = t_d;
    ra.u0amp = u_d;
    ra.phiamp = f_d;
    ra.wts = p->wts_d;
    ra.cvals = c_d;
    FT_CUDA(launch_rhs_modes(ra, p->stream));
    FT_CUDA(cudaStreamSynchronize(p->stream));
    cudaFree(a_d); cudaFree(k_d); cudaFree(p_d); cudaFree(t_d); cudaFree(c_d);
    if (u_d) cudaFree(u_d);
    if (f_d) cudaFree(f_d);
    return FT_OK;
}

// Fast solve with pinned host buffers: chunked H2D of R and D2H of U overlap
// the solve (StreamIO).  Pageable host buffers take the serial path below.
// Chunking and copy streams of the streamed host paths.
static int stream_setup(ft_plan* p, StreamIO& io) {
    const uint64_t N = p->N;
    // chunk: wide enough for efficient 2D DMA rows, small enough for a short fill/drain
    uint64_t C = getenv("FT_STREAM_CHUNK") ? (uint64_t)atoll(getenv("FT_STREAM_CHUNK")) : 2048;  // B200 PCIe: 16 KB rows best (measured 256..4096)
    C = std::max<uint64_t>((C + p->L - 1) / p->L * p->L, (uint64_t)p->L);
    io.C = std::min<uint64_t>(N, C);
    const uint64_t nch = (N + io.C - 1) / io.C;
    if (!p->h2d_st) {
        FT_CUDA(cudaStreamCreateWithFlags(&p->h2d_st, cudaStreamNonBlocking));
        FT_CUDA(cudaStreamCreateWithFlags(&p->d2h_st, cudaStreamNonBlocking));
    }
    while (p->h2d_ev.size() < nch) {
        cudaEvent_t e1, e2;
        FT_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
        FT_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
        p->h2d_ev.push_back(e1);
        p->d2h_ev.push_back(e2);
    }
    return FT_OK;
}

static int solve_streamed(ft_plan* p, const double* rhs, double* u, ft_report* rep, bool stream_rhs,
                          std::chrono::steady_clock::time_point t_start) {
    const uint64_t N = p->N, rows = rows_of(p);
    const size_t bytes = sizeof(double) * rows * N;
    const cudaStream_t st = p->stream;
    const bool u_dev = is_device_ptr(u);
    double* X = u;
    if (!u_dev) {
        int rc = ensure_work(p);
        if (rc) return rc;
        X = p->work_d;
    }
    StreamIO io;
    {
        int rc = stream_setup(p, io);
        if (rc) return rc;
    }
    const uint64_t nch = (N + io.C - 1) / io.C;
    FT_CUDA(cudaEventRecord(p->ev0, st));
    const double* src = rhs;
    if (stream_rhs) {
        if (!p->rdev_d) FT_CUDA(cudaMalloc(&p->rdev_d, bytes));
        io.defer = true;
        io.rdev = p->rdev_d;
        src = X;
        FT_CUDA(cudaStreamWaitEvent(p->h2d_st, p->ev0, 0));  // previous solves on this plan are done
        for (uint64_t c = 0; c < nch; ++c) {
            const uint64_t c0 = c * io.C, w = std::min<uint64_t>(N, c0 + io.C) - c0;
            FT_CUDA(cudaMemcpy2DAsync(p->rdev_d + c0, sizeof(double) * N, rhs + c0, sizeof(double) * N,
                                      sizeof(double) * w, rows, cudaMemcpyHostToDevice, p->h2d_st));
            FT_CUDA(cudaEventRecord(p->h2d_ev[c], p->h2d_st));
        }
        FT_CUDA(cudaMemsetAsync(X, 0, bytes, st));  // history accumulates into zero; leaves add R
    }
    io.u_host = u_dev ? nullptr : u;
    uint64_t launches = 0;
    int rc = run_fast(p, X, src, &launches, nullptr, &io);
    if (rc) return rc;
    FT_CUDA(cudaEventRecord(p->ev1, st));
    FT_CUDA(cudaStreamSynchronize(st));
    if (!u_dev) FT_CUDA(cudaStreamSynchronize(p->d2h_st));
    float ms = 0.f;
    FT_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    if (rep) {
        std::snprintf(rep->method, sizeof(rep->method), "%s", "fast");
        rep->iterations = 0;
        rep->residual = 0.0;
        rep->device_ms = ms;
        rep->kernel_launches = launches;
        rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    }
    return FT_OK;
}

// One fast solve on the plan's stream: replayed as a CUDA graph (single
// rank; keyed by the buffers and the fused-RHS tables), else launched directly.
static int launch_fast(ft_plan* p, double* X, const double* src, const GenRhs* gen, uint64_t* launches) {
    const cudaStream_t st = p->stream;
    // single-node (ODE) problems: the whole time march in one kernel per call
    if (!gen && ode_whole_plan(p)) {
        FT_CUDA(launch_ode_whole(X, src, p->col_d, p->pc_d, p->N, p->B, st));
        *launches = 1;
        return FT_OK;
    }
    const bool use_graph = (p->part_world == 1 || p->p2p || p->nccl_comm) && !getenv("FT_NO_GRAPH");
    if (!use_graph) return run_fast(p, X, src, launches, nullptr, nullptr, gen);
    const void* gkey = gen ? (const void*)gen->A : nullptr;
    const int gJ = gen ? gen->J : 0;
    if (!p->graph || p->graph_X != X || p->graph_src != src || p->graph_gen != gkey || p->graph_genJ != gJ) {
        if (p->graph) cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
        cudaStream_t cs;
        FT_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        FT_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        const cudaStream_t keep = p->stream;
        p->stream = cs;
        int rc = run_fast(p, X, src, &p->graph_launches, nullptr, nullptr, gen);
        p->stream = keep;
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(cs, &g);
        cudaStreamDestroy(cs);
        if (rc) return rc;
        FT_CUDA(ce);
        const cudaError_t ie = cudaGraphInstantiate(&p->graph, g, 0);
        cudaGraphDestroy(g);
        FT_CUDA(ie);
        p->graph_X = X;
        p->graph_src = src;
        p->graph_gen = gkey;
        p->graph_genJ = gJ;
    }
    {
        BankScope bank(p, p->B > 1);
        if (bank.err != cudaSuccess) return set_err(FT_ECUDA, "leaf weight bank upload failed");
        FT_CUDA(cudaGraphLaunch(p->graph, st));
    }
    *launches = p->graph_launches;
    return FT_OK;
}

static int solve_common(ft_plan* p, const double* rhs, double* u, ft_report* rep, bool fast) {
    if (!p || !rhs || !u) return set_err(FT_EINVAL, "ft_solve: null argument");
    if (!fast && p->part_world > 1) return set_err(FT_EINVAL, "ft_solve_direct: not available on partitioned plans");
    const auto t_start = std::chrono::steady_clock::now();
    FT_CUDA(cudaSetDevice(p->device));
    const uint64_t elems = rows_of(p) * p->N;
    const size_t bytes = sizeof(double) * elems;
    const bool rhs_dev = is_device_ptr(rhs), u_dev = is_device_ptr(u);
    const cudaStream_t st = p->stream;
    const bool stream_rhs = fast && !rhs_dev && is_pinned_host(rhs);
    const bool stream_u = fast && !u_dev && is_pinned_host(u);
    // single-node (ODE) plans move a few KB: one copy each way around the one-kernel march
    const bool ode1 = fast && ode_whole_plan(p);
    if ((stream_rhs || stream_u) && !ode1 && !getenv("FT_NO_STREAM"))
        return solve_streamed(p, rhs, u, rep, stream_rhs, t_start);
    double* X;
    const double* src;
    if (u_dev) {
        X = u;
        if (rhs_dev) {
            src = rhs;
        } else {
            FT_CUDA(cudaMemcpyAsync(X, rhs, bytes, cudaMemcpyHostToDevice, st));
            src = X;
        }
    } else {
        int rc = ensure_work(p);
        if (rc) return rc;
        X = p->work_d;
        if (rhs_dev) {
            src = rhs;
        } else {
            FT_CUDA(cudaMemcpyAsync(X, rhs, bytes, cudaMemcpyHostToDevice, st));
            src = X;
        }
    }
    uint64_t launches = 0;
    FT_CUDA(cudaEventRecord(p->ev0, st));
    if (fast) {
        int rc = launch_fast(p, X, src, nullptr, &launches);
        if (rc) return rc;
    } else {
        if (src != X) FT_CUDA(cudaMemcpyAsync(X, src, bytes, cudaMemcpyDeviceToDevice, st));
        DirectArgs da;
        da.X = X;
        da.N = p->N;
        da.nodes = p->nodes;
        da.kind = p->kind;
        da.w = p->dw_d;
        da.cprime = p->cprime_d;
        da.den = p->den_d;
        da.pc = p->pc_d;
        da.scratch = p->scratch_d;
        da.scratch2 = p->scratch_d + (uint64_t)p->B * p->nodes;
        da.stencil = p->stencil ? 1 : 0;
        da.ctr = p->dmctr_d;
        FT_CUDA(launch_direct(da, p->B, st));
        launches = 1;
    }
    FT_CUDA(cudaEventRecord(p->ev1, st));
    if (!u_dev) FT_CUDA(cudaMemcpyAsync(u, X, bytes, cudaMemcpyDeviceToHost, st));
    FT_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    FT_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    if (rep) {
        std::snprintf(rep->method, sizeof(rep->method), "%s", fast ? "fast" : "direct");
        rep->iterations = 0;
        rep->residual = 0.0;
        rep->device_ms = ms;
        rep->kernel_launches = launches;
        // FT_OPT_REPORT_RESIDUAL: measure max |A u - rhs| / max |rhs| through the plan's operator
        // (device buffers, rhs kept: one operator application, about the cost of the solve's products)
        if (p->report_residual && rhs_dev && u_dev && rhs != u && !p->stencil && p->part_world == 1) {
            double r = 0.0, m = 0.0;
            const int rc = ft_residual(p, rhs, u, nullptr, &r, &m);
            if (rc) return rc;
            rep->residual = m > 0.0 ? r / m : r;
        }
        rep->seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    }
    return FT_OK;
}

int ft_solve_fast(ft_plan* p, const double* rhs, double* u, ft_report* rep) {
    return solve_common(p, rhs, u, rep, true);
}

int ft_solve_direct(ft_plan* p, const double* rhs, double* u, ft_report* rep) {
    return solve_common(p, rhs, u, rep, false);
}

// Fast solve with the separable forcing generated inside the leaves (SURVEY 8f
// item 2): R is never materialised -- the history products accumulate into X
// from zero and each leaf adds sum_j A[row][j] T[n][j] while staging its tile.
int ft_solve_fast_modes(ft_plan* p, int nmodes, const double* a, const double* k, const double* pe,
                        const int* trig, const double* u0amp, const double* phiamp, double* u, ft_report* rep) {
    if (p && p->custom) return set_err(FT_EINVAL, "ft_solve_fast_modes: plan from ft_setup_toeplitz has no scheme");
    if (!p || !u || nmodes < 0 || (nmodes && (!a || !k || !pe || !trig)))
        return set_err(FT_EINVAL, "ft_solve_fast_modes: bad argument");
    const auto t_start = std::chrono::steady_clock::now();
    FT_CUDA(cudaSetDevice(p->device));
    const cudaStream_t st = p->stream;
    const int B = p->B;
    // small argument arrays in one plan-owned device block (no per-call cudaMalloc)
    const size_t nm = (size_t)std::max(1, nmodes);
    std::vector<double> hb;
    hb.reserve(2 * B * nm + nm + 3 * B + nm);
    auto put = [&](const double* x, size_t n) {
        const size_t off = hb.size();
        for (size_t i = 0; i < n; ++i) hb.push_back(x ? x[i] : 0.0);
        return off;
    };
    const size_t oa = put(nmodes ? a : nullptr, B * nm), ok = put(nmodes ? k : nullptr, nm),
                 op = put(nmodes ? pe : nullptr, B * nm);
    std::vector<double> cv(B);
    for (int b = 0; b < B; ++b) cv[b] = p->c[b];
    const size_t oc = put(cv.data(), B), ou = put(u0amp, B), of = put(phiamp, B);
    const size_t ot = hb.size();
    hb.resize(hb.size() + (nm + 1) / 2, 0.0);  // trig ids: nm contiguous ints in the tail
    {
        std::vector<int> tv(nm, 2);
        for (size_t i = 0; i < (size_t)nmodes; ++i) tv[i] = trig[i];
        std::memcpy(hb.data() + ot, tv.data(), sizeof(int) * nm);
    }
    int rc;
    if (hb.size() * sizeof(double) > p->genArgs_bytes) {
        if (p->genArgs_d) cudaFree(p->genArgs_d);
        p->genArgs_d = nullptr;
        if ((rc = alloc_copy((void**)&p->genArgs_d, nullptr, hb.size() * sizeof(double)))) return rc;
        p->genArgs_bytes = hb.size() * sizeof(double);
    }
    FT_CUDA(cudaMemcpyAsync(p->genArgs_d, hb.data(), hb.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    const double* gd = p->genArgs_d;
    const double *a_d = gd + oa, *k_d = gd + ok, *p_d = gd + op, *c_d = gd + oc;
    const double* u_d = u0amp ? gd + ou : nullptr;
    const double* f_d = phiamp ? gd + of : nullptr;
    const int* t_d = reinterpret_cast<const int*>(gd + ot);
    RhsModesArgs ra;
    ra.R = nullptr;
    ra.N = p->N;
    ra.nodes = p->local_nodes;
    ra.B = B;
    ra.nmodes = nmodes;
    ra.scheme = p->scheme;
    ra.rhs_mode = p->rhs_mode;
    ra.node_begin = p->node_begin;
    ra.h = p->h;
    ra.tau = p->tau;
    ra.a = a_d;
    ra.k = k_d;
    ra.p = p_d;
    ra.trig = t_d;
    ra.u0amp = u_d;
    ra.phiamp = f_d;
    ra.wts = p->wts_d;
    ra.cvals = c_d;
    const int J = std::max(1, gen_terms(ra));
    if (J > 16) return set_err(FT_EINVAL, "ft_solve_fast_modes: at most 14 forcing modes");
    if (ode_whole_plan(p)) {
        // single-node (ODE) plans: B x N right-hand sides are a few KB, so generate the
        // array (same device kernel as ft_assemble_rhs_modes) and run the one-kernel march
        if (!p->oder_d && (rc = alloc_copy((void**)&p->oder_d, nullptr, sizeof(double) * rows_of(p) * p->N)))
            return rc;
        const bool u_dev = is_device_ptr(u);
        double* X = u;
        if (!u_dev) {
            if ((rc = ensure_work(p))) return rc;
            X = p->work_d;
        }
        ra.R = p->oder_d;
        FT_CUDA(cudaEventRecord(p->ev0, st));
        FT_CUDA(launch_rhs_modes(ra, st));
        FT_CUDA(launch_ode_whole(X, p->oder_d, p->col_d, p->pc_d, p->N, p->B, st));
        FT_CUDA(cudaEventRecord(p->ev1, st));
        if (!u_dev) FT_CUDA(cudaMemcpyAsync(u, X, sizeof(double) * rows_of(p) * p->N, cudaMemcpyDeviceToHost, st));
        FT_CUDA(cudaStreamSynchronize(st));
        float ms = 0.f;
        FT_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
        if (rep) {
            std::snprintf(rep->method, sizeof(rep->method), "%s", "fast");
            rep->iterations = 0;
            rep->residual = 0.0;
            rep->device_ms = ms;
            rep->kernel_launches = 2;
            rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
        }
        return FT_OK;
    }
    const size_t ab = sizeof(double) * rows_of(p) * J, tb = sizeof(double) * (size_t)B * p->N * J;
    if (ab != p->genA_bytes || tb != p->genT_bytes) {
        // the captured graph bakes in the table pointers and J: a reallocation may hand
        // back the same address, so drop the graph rather than trust the pointer key
        if (p->graph) cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    if (ab != p->genA_bytes) {
        if (p->genA_d) cudaFree(p->genA_d);
        p->genA_d = nullptr;
        if ((rc = alloc_copy((void**)&p->genA_d, nullptr, ab))) return rc;
        p->genA_bytes = ab;
    }
    if (tb != p->genT_bytes) {
        if (p->genT_d) cudaFree(p->genT_d);
        p->genT_d = nullptr;
        if ((rc = alloc_copy((void**)&p->genT_d, nullptr, tb))) return rc;
        p->genT_bytes = tb;
    }
    if (gen_terms(ra) == 0) {  // homogeneous: all-zero tables
        FT_CUDA(cudaMemsetAsync(p->genA_d, 0, ab, st));
        FT_CUDA(cudaMemsetAsync(p->genT_d, 0, tb, st));
    } else {
        FT_CUDA(launch_gen_tables(ra, p->genA_d, p->genT_d, st));
    }
    GenRhs gen;
    gen.A = p->genA_d;
    gen.T = p->genT_d;
    gen.J = J;
    const bool u_dev = is_device_ptr(u);
    double* X = u;
    if (!u_dev) {
        if ((rc = ensure_work(p))) return rc;
        X = p->work_d;
    }
    uint64_t launches = 0;
    FT_CUDA(cudaEventRecord(p->ev0, st));
    if (!u_dev && is_pinned_host(u) && !getenv("FT_NO_STREAM")) {
        // pinned host output: finished chunks of U leave on the copy stream while the
        // solve continues (the only PCIe traffic of this call besides the mode arguments)
        StreamIO io;
        if ((rc = stream_setup(p, io))) return rc;
        io.u_host = u;
        if ((rc = run_fast(p, X, nullptr, &launches, nullptr, &io, &gen))) return rc;
        FT_CUDA(cudaEventRecord(p->ev1, st));
        FT_CUDA(cudaStreamSynchronize(st));
        FT_CUDA(cudaStreamSynchronize(p->d2h_st));
    } else {
        if ((rc = launch_fast(p, X, nullptr, &gen, &launches))) return rc;
        FT_CUDA(cudaEventRecord(p->ev1, st));
        if (!u_dev) FT_CUDA(cudaMemcpyAsync(u, X, sizeof(double) * rows_of(p) * p->N, cudaMemcpyDeviceToHost, st));
    }
    FT_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    FT_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    if (rep) {
        std::snprintf(rep->method, sizeof(rep->method), "%s", "fast");
        rep->iterations = 0;
        rep->residual = 0.0;
        rep->device_ms = ms;
        rep->kernel_launches = launches;
        rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    }
    return FT_OK;
}

// y = A x with A the plan's block lower-triangular Toeplitz system matrix (the matrix
// ft_solve_fast inverts): far history through the schedule's own FFT / direct products
// (O(M N log N)), in-leaf lags and the spatial stencil by apply_near_kernel.
static int apply_launches(ft_plan* p, const double* x, double* y, cudaStream_t st);
static int apply_impl(ft_plan* p, const double* x, double* y) {
    if (!p || !x || !y) return set_err(FT_EINVAL, "ft_apply: bad argument");
    if (p->stencil) return set_err(FT_EINVAL, "ft_apply: Scheme 2 (stencil history) plans are not supported");
    if (p->part_world != 1) return set_err(FT_EINVAL, "ft_apply: partitioned plans are not supported");
    if (!is_device_ptr(x) || !is_device_ptr(y) || x == y)
        return set_err(FT_EINVAL, "ft_apply: x and y must be distinct buffers, both on the device or both on the host");
    FT_CUDA(cudaSetDevice(p->device));
    // the launch sequence (up to ~2 N / L products) replays as one CUDA graph per buffer pair: a
    // Krylov caller applies the operator hundreds of times to the same device vectors
    if (!getenv("FT_NO_GRAPH")) {
        if (p->apply_graph && p->apply_x == x && p->apply_y == y) {
            FT_CUDA(cudaGraphLaunch(p->apply_graph, p->stream));
            return FT_OK;
        }
        if (p->apply_graph) cudaGraphExecDestroy(p->apply_graph);
        p->apply_graph = nullptr;
        cudaStream_t cs;
        FT_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        FT_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        const int rc = apply_launches(p, x, y, cs);
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(cs, &g);
        cudaStreamDestroy(cs);
        if (rc) return rc;
        FT_CUDA(ce);
        const cudaError_t ie = cudaGraphInstantiate(&p->apply_graph, g, 0);
        cudaGraphDestroy(g);
        FT_CUDA(ie);
        p->apply_x = x;
        p->apply_y = y;
        FT_CUDA(cudaGraphLaunch(p->apply_graph, p->stream));
        return FT_OK;
    }
    return apply_launches(p, x, y, p->stream);
}

static int apply_launches(ft_plan* p, const double* x, double* y, cudaStream_t st) {
    const uint64_t N = p->N;
    FT_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * rows_of(p) * N, st));
    for (const Op& op : p->ops) {
        if (op.kind == OP_LEAF) continue;
        const Level& lv = p->levels[op.level];
        MpArgs a;
        a.X = y;
        a.U = x;
        a.rsrc = y;
        a.pdl_trigger = 0;
        a.N = N;
        a.lo = op.t0;
        a.mid = op.mid;
        a.hi = op.hi;
        a.n = lv.n;
        a.m = lv.m;
        a.K = lv.K;
        a.G = lv.G;
        a.rows = (int)rows_of(p);
        a.nodes = p->local_nodes;
        a.pairs_per_problem = (p->local_nodes + 1) / 2;
        a.spec = p->spec_d + lv.spec_off;
        a.tw = p->tw_d;
        a.logT = p->logT;
        a.col = p->col_d;
        a.J = p->J;
        a.scratch = (lv.K >= p->split_min_k && p->split_k) ? p->mpscratch_d : nullptr;
        a.pair_begin = 0;
        a.pair_count = 0;
        FT_CUDA(launch_mp(a, lv.groups, st));
    }
    FT_CUDA(launch_apply_near(x, y, N, p->local_nodes, rows_of(p), p->pc_d, p->col_d, p->kind, p->L, st));
    return FT_OK;
}

int ft_apply(ft_plan* p, const double* x, double* y) {
    if (p && x && y && !is_device_ptr(x) && !is_device_ptr(y)) {
        // host vectors (the reference's LinearOperator::apply takes and returns host spans):
        // staged through two device buffers
        FT_CUDA(cudaSetDevice(p->device));
        const size_t bytes = sizeof(double) * rows_of(p) * p->N;
        double *xd = nullptr, *yd = nullptr;
        if (cudaMalloc(&xd, bytes) != cudaSuccess || cudaMalloc(&yd, bytes) != cudaSuccess) {
            cudaFree(xd);
            return set_err(FT_ENOMEM, "ft_apply: device staging buffers");
        }
        cudaError_t e = cudaMemcpyAsync(xd, x, bytes, cudaMemcpyHostToDevice, p->stream);
        // (temporary buffers: launched directly, not through the cached graph)
        int rc = e == cudaSuccess ? apply_launches(p, xd, yd, p->stream) : set_err(FT_ECUDA, cudaGetErrorString(e));
        if (!rc) {
            e = cudaMemcpyAsync(y, yd, bytes, cudaMemcpyDeviceToHost, p->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
            if (e != cudaSuccess) rc = set_err(FT_ECUDA, cudaGetErrorString(e));
        }
        cudaFree(xd);
        cudaFree(yd);
        return rc;
    }
    const int rc = apply_impl(p, x, y);
    if (rc) return rc;
    FT_CUDA(cudaStreamSynchronize(p->stream));
    return FT_OK;
}

int ft_residual(ft_plan* p, const double* rhs, const double* u, double* work, double* max_abs_residual,
                double* max_abs_rhs) {
    if (!p || !rhs || !u || !max_abs_residual || !max_abs_rhs) return set_err(FT_EINVAL, "ft_residual: bad argument");
    if (!is_device_ptr(rhs)) return set_err(FT_EINVAL, "ft_residual: device buffers expected");
    double* y = work;
    if (!y) {
        const int rc = ensure_work(p);
        if (rc) return rc;
        y = p->work_d;
    }
    const int rc = apply_impl(p, u, y);
    if (rc) return rc;
    unsigned long long* out = nullptr;
    FT_CUDA(cudaMalloc(&out, 2 * sizeof(unsigned long long)));
    cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), p->stream);
    cudaError_t e = launch_resid_max(y, rhs, rows_of(p) * p->N, out, p->stream);
    unsigned long long h[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    cudaFree(out);
    if (e != cudaSuccess) return set_err(FT_ECUDA, cudaGetErrorString(e));
    std::memcpy(max_abs_residual, &h[0], sizeof(double));
    std::memcpy(max_abs_rhs, &h[1], sizeof(double));
    return FT_OK;
}

// diagnostics: the clock64 stamps of the last slab leaf (FT_LEAF_DBG & 4)
int ft_debug_leaf_clocks(const ft_plan* p, long long* out16) {
    if (!p || !p->dbgclk_d) return set_err(FT_EINVAL, "no leaf clocks");
    FT_CUDA(cudaMemcpy(out16, p->dbgclk_d, sizeof(long long) * 16, cudaMemcpyDeviceToHost));
    return FT_OK;
}

int ft_schedule(uint64_t N, uint64_t L, ft_op_time* out, uint64_t cap, uint64_t* count) {
    if (!count || N == 0 || L == 0 || (L & (L - 1))) return set_err(FT_EINVAL, "ft_schedule: bad argument");
    ft_plan tmp;
    tmp.N = N;
    tmp.L = (int)L;
    tmp.nodes = 1;
    tmp.B = 1;
    build_schedule(&tmp);
    for (uint64_t i = 0; i < tmp.ops.size() && i < cap; ++i) {
        const Op& op = tmp.ops[i];
        ft_op_time& o = out[i];
        o.ms = 0.f;
        o.bytes = 0;
        if (op.kind == OP_LEAF) {
            o.kind = 0;
            o.level = -1;
            o.t0 = op.t0;
            o.len = (uint64_t)op.len;
        } else {
            o.kind = 1;
            o.level = op.level;
            o.t0 = op.mid;
            o.len = std::min<uint64_t>(op.hi, N) - op.mid;
        }
    }
    *count = tmp.ops.size();
    return FT_OK;
}

int ft_profile_fast(ft_plan* p, const double* rhs, double* u, ft_op_time* out, uint64_t cap,
                    uint64_t* count) {
    if (!p || !rhs || !u || !count) return set_err(FT_EINVAL, "ft_profile_fast: null argument");
    if (!is_device_ptr(rhs) || !is_device_ptr(u))
        return set_err(FT_EINVAL, "ft_profile_fast: device buffers expected");
    FT_CUDA(cudaSetDevice(p->device));
    std::vector<cudaEvent_t> evs(p->ops.size() + 1);
    for (auto& e : evs) FT_CUDA(cudaEventCreate(&e));
    uint64_t nl = 0;
    int rc = run_fast(p, u, rhs, &nl, &evs);
    if (rc) return rc;
    FT_CUDA(cudaStreamSynchronize(p->stream));
    const uint64_t rows = rows_of(p);
    const uint64_t n_ops = p->ops.size();
    for (uint64_t i = 0; i < n_ops && i < cap; ++i) {
        const Op& op = p->ops[i];
        ft_op_time& o = out[i];
        float ms = 0.f;
        FT_CUDA(cudaEventElapsedTime(&ms, evs[i], evs[i + 1]));
        o.ms = ms;
        if (op.kind == OP_LEAF) {
            o.kind = 0;
            o.level = -1;
            o.t0 = op.t0;
            o.len = (uint64_t)op.len;
            o.bytes = 16ull * rows * o.len;  // read R, write U
        } else {
            const uint64_t h = op.mid - op.t0;
            const uint64_t tend = std::min<uint64_t>(op.hi, p->N);
            o.kind = 1;
            o.level = op.level;
            o.t0 = op.mid;
            o.len = tend - op.mid;
            o.bytes = 8ull * rows * h + 16ull * rows * o.len;  // read U half, read+write R half
        }
    }
    if (p->last_fuse0) {  // folded n = 64 products: their bytes belong to the next leaf's launch
        for (uint64_t i = 0; i + 1 < n_ops && i + 1 < cap; ++i)
            if (p->ops[i].kind == OP_MP && p->ops[i].level == 0 && p->ops[i + 1].kind == OP_LEAF) {
                out[i + 1].bytes += out[i].bytes;
                out[i].bytes = 0;
            }
    }
    *count = n_ops;
    for (auto& e : evs) cudaEventDestroy(e);
    return FT_OK;
}

void ft_destroy(ft_plan* p) {
    if (!p) return;
    leaf_bank_forget(p);
    cudaSetDevice(p->device);
    if (!p->own_xch) p->xch_d = nullptr;
    void* ptrs[] = {p->pc_d, p->col_d, p->wts_d, p->lampow_d, p->tw_d, p->spec_d, p->xch_d,
                    p->kcoef_d, p->chain_d, p->respg_d, p->resph_d, p->respw_d, p->bar_d, p->mpscratch_d, p->dw_d, p->cprime_d, p->den_d, p->scratch_d, p->dmctr_d, p->work_d, p->vsrc_d, p->genA_d, p->genT_d, p->genArgs_d, p->oder_d};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    if (p->graph) cudaGraphExecDestroy(p->graph);
    if (p->apply_graph) cudaGraphExecDestroy(p->apply_graph);
    if (p->nccl_comm) nccl_api().CommDestroy(p->nccl_comm);
    if (p->rdev_d) cudaFree(p->rdev_d);
    for (void* q : p->p2p_opened) cudaIpcCloseMemHandle(q);
    if (p->p2p_block) cudaFree(p->p2p_block);
    if (p->p2p_peers_d) cudaFree(p->p2p_peers_d);
    for (cudaEvent_t e : p->h2d_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : p->d2h_ev) cudaEventDestroy(e);
    if (p->h2d_st) cudaStreamDestroy(p->h2d_st);
    if (p->d2h_st) cudaStreamDestroy(p->d2h_st);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
    delete p;
}

}  // extern "C"
