// internal.cuh -- shared definitions of the B200 fast BLTT solver.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

namespace ftb {

// Spatial operator of one time step (the diagonal block  col0*I + spatial part):
//   SK_DIAG    : d x = r                                  (one-sided ODE)
//   SK_UPWIND  : d x_i - s x_{i-1} = r_i,  x_0 = 0          (reference Scheme 3, s = 1/h)
//   SK_TRIDIAG : d x_i - b (x_{i-1} + x_{i+1}) = r_i, Dirichlet  (reference Scheme 4, b = 1/h^2)
enum SpaceKind { SK_DIAG = 0, SK_UPWIND = 1, SK_TRIDIAG = 2 };

// Per-problem constants of the step operator, in the form the scan solver
// uses.  TRIDIAG: x = G0 (F + B - r) + alpha lam^i + gam lam^(n+1-i)
// with F/B the forward/backward lam-decay scans of r.  UPWIND: x = F where F is
// the forward scan with multiplier lam = s/d of  r/d.
struct ProblemConst {
    double d;        // col[0]
    double off;      // b (tridiag) or s (upwind), positive
    double lam;      // decay multiplier
    double G0;       // tridiag Green normalisation (upwind: 1/d)
    double Lam;      // lam^(nodes+1)
    double inv1mL2;  // 1/(1-Lam^2)
    double c;        // scheme constant c (direct path)
    double h;        // mesh width (direct wave path divides by it, as the reference)
};

constexpr int kLeafThreads = 256;
constexpr uint64_t kMaxTimeSteps = 65536;  // N limit (FT_ELENGTH): history products up to n = 65536
// LeafArgs::kc layout (single-problem plans): col[0..64) (the in-leaf weights, lags < 32,
// and the far half of the level-0 history window fused into the leaf, contiguous so the
// rolled product indexes them at a runtime offset), then the uniform scan multipliers
// lam^(NPT 2^d) (d < 5), lam^(32 NPT), lam, lam^(v+1) and lam^(NPT-v) (v < 8).
constexpr int kKcCol2 = 32, kKcPow = 64, kKcLamW = 69, kKcLam = 70, kKcV1 = 72, kKcNv = 80, kKcLen = 88;
constexpr int kMaxSlabs = 160;
constexpr int kMaxLeafProblems = 128;  // problems per plan
constexpr int kMpThreads = 256;
constexpr int kMpTile = 4096;   // complex points per CTA (64 KiB of SMEM + pad)
constexpr int kMpDirectMaxH = 64;   // blocks n <= 128 use the direct Toeplitz kernel
constexpr int kMpSingleMaxN = 4096; // 256 <= n <= 4096: single-CTA n-point FFT kernel (n = 8192 as a
                                    // 2-CTA cluster: 32.0 vs 34.8 ms per level, 1 CTA/SM single)
constexpr int kMpBranchMax = 4096;  // larger n: K-CTA clusters of (n / K)-point branches (8192 measured slower: 1 CTA/SM)

struct __align__(16) cplx {
    double x, y;
};

__host__ __device__ inline cplx cmul(cplx a, cplx b) {
    return {fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}
__host__ __device__ inline cplx cmulc(cplx a, cplx b) {  // a * conj(b)
    return {fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y)};
}
__device__ __forceinline__ cplx ldgc(const cplx* p) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p));
    return {v.x, v.y};
}
__host__ __device__ inline cplx cadd(cplx a, cplx b) { return {a.x + b.x, a.y + b.y}; }
__host__ __device__ inline cplx csub(cplx a, cplx b) { return {a.x - b.x, a.y - b.y}; }

// Per-device one-time setup (cudaFuncSetAttribute applies to the current device
// only; plans may pick a device through ft_options.device).  Two threads racing
// both run the (idempotent) setup.
struct DeviceOnce {
    std::atomic<unsigned long long> mask{0};
    static int dev() {
        int d = 0;
        cudaGetDevice(&d);
        return d & 63;
    }
    bool first() const { return !((mask.load() >> dev()) & 1ull); }
    void done() { mask.fetch_or(1ull << dev()); }
};

// ---- programmatic dependent launch (PDL) ------------------------------------
// Every kernel of the fast-solve schedule is launched with programmatic stream
// serialization: it lets the next kernel's CTAs launch as soon as all CTAs of
// the running one have started, so launch latency and prologues overlap the
// predecessor's tail.  Each such kernel calls pdl_wait() before its first
// access to data another kernel of the solve writes or reads (every CTA calls
// it, so completion of kernel k implies completion of k-1: transitive).
__device__ __forceinline__ void pdl_launch_dependents(int on) {
    if (on) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// FT_PDL: unset/0 = off (measured: with an early trigger cfg4 went 420 -> 473 ms),
// 1 = trigger at kernel start, 2 = implicit trigger at CTA exit (launch latency only)
inline int pdl_mode() {
    static const int m = getenv("FT_PDL") ? atoi(getenv("FT_PDL")) : 0;
    return m;
}
inline bool pdl_enabled() { return pdl_mode() != 0; }

// cudaLaunchKernelEx with PDL (when enabled) and an optional cluster size
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             unsigned cluster, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cluster;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// ---- launch arguments ------------------------------------------------------

struct LeafArgs {
    double* X;                 // rows x N, node-major (U for solved steps, R after)
    const double* src;         // where this leaf's R tile is read from (X or the caller's rhs)
    const double* src2;        // leaf-pair kernel: the same for the second leaf of the pair
    const double* radd;        // streamed host solves: R added at staging (history in src), else null
    uint64_t N;                // row pitch = time steps
    uint64_t t0;               // first step of the leaf
    int len;                   // steps in this leaf (<= L)
    int nodes;                 // interior nodes per problem
    int slab;                  // nodes per CTA
    int P;                     // slabs (CTAs) per problem
    const ProblemConst* pc;    // [B]
    const double* col;         // [B][N] Toeplitz first columns
    const double* lampow;      // [B][lp_stride]: lam^k, k = 0..lp_stride-1
    int lp_stride;
    const double* kcoef;       // [B][2][nodes] single-CTA Dirichlet coefficients kF, kB
    double* xch;               // multi-slab carries of the current leaf, all slabs [B][P][L][2]
    double* xsend;             // phase-1 output [B*P_local][L][2] (== xch unless partitioned)
    double2* chain;            // chained upwind slabs: [B][P][L] {last-node solution, leaf tag} per step
    double chain_tag;          // tag of this leaf's entries (leaf index + 1; the buffer is zeroed per solve)
    int P_local;               // slabs (CTAs) per problem held by this plan / rank
    int s_begin;               // first slab of this rank
    int node_begin;            // first node of this rank (X row 0 of a problem)
    int rows_pp;               // X rows per problem held by this plan
    const double* resp_g;      // [B][2 slab kinds][2 (L,R)][slab][L] space-time responses
    int paired_g;              // resp_g holds mirror-pair tables S = (GL+GR)/2, D = (GL-GR)/2 (tridiagonal)
    const double* resp_h;      // [B][2 slab kinds][L][4] carry responses hFL hFR hBL hBR
    const double* resp_w;      // [B][P][2 (EL,ER)][L lag][2P source carries] injection responses
    int dbg;                   // diagnostics: bit0 skip phase 2, bit1 skip phase 3
    unsigned* bar;             // fused slab leaf: grid-barrier counter (zeroed per solve)
    unsigned bar_target;       // value the counter reaches when every CTA of this leaf arrived
    long long* dbg_clk;        // diagnostics: per-phase clock64 stamps of CTA 0 (null = off)
    int pdl_trigger;           // PDL: signal dependents at kernel start (pdl_mode() == 1)
    double* V;                 // Scheme 2 (single slab): V = U_i + U_(i-1) written next to U, else null
    int stencil;               // Scheme 2: in-leaf history acts on U_i + U_(i-1)
    const double* genA;        // fused separable RHS (ft_solve_fast_modes): [rows][genJ] node factors
    const double* genT;        //   [B][N][genJ] step factors; R = sum_j genA * genT added at staging
    int genJ;                  //   (null genA: R comes from src)
    // device-side carry exchange over NVLink peer memory (partitioned plans, opt-in):
    const unsigned long long* p2p_peers;  // [world] base of every rank's exchange block (peer-mapped)
    const unsigned* p2p_epoch;            // this rank's solve counter (incremented per solve)
    int p2p_world, p2p_leaf, p2p_leaves;  // ranks, leaf index in the solve, leaves per solve
    int fuse0;                 // slab leaf applies the n = 64 history product from the previous leaf
                               // (X[., t0-32, t0) -> this tile) itself; its launch is skipped
    int kc_valid;              // kc holds problem 0's leaf constants (single-problem plans)
    double kc[kKcLen];         // see kKc* (kernel parameter: constant-bank operands)
};

struct MpArgs {
    double* X;
    const double* U;           // source rows U[lo, mid) (== X; Scheme 2: V = U_i + U_(i-1))
    const double* rsrc;        // target R is read from here (== X except first touch; null = zero)
    uint64_t N;
    uint64_t lo, mid, hi;      // source [lo, mid), target [mid, min(hi, N))
    int n, m, K, G;            // block size, branch length, branches, row pairs per CTA
    int rows, nodes;           // total rows, nodes per problem
    int pairs_per_problem;
    const cplx* spec;          // spectra of this level: [B][K][m] digit-reversed, scaled 1/n
    const cplx* tw;            // twiddle table w_T^k = exp(-2 pi i k / T)
    int logT;
    const double* col;         // [B][N] (near field)
    int J;                     // near-field lags summed exactly: 1..J-1
    cplx* scratch;             // split K-branch levels: branch results [pairs][K][m]
    int pair_begin, pair_count;  // split K-branch levels: pairs of this launch
    int pdl_trigger;           // PDL: signal dependents at kernel start (pdl_mode() == 1)
};

struct DirectArgs {
    double* X;            // in: R (node-major), out: U; in place
    uint64_t N;
    int nodes;
    int kind;             // SK_*
    const double* w;      // [B][N]: S4 dg[j] = g[j-1]-g[j]; S3/ODE: col[j]
    const double* cprime; // [B][nodes] Thomas (S4)
    const double* den;    // [B][nodes] Thomas denominators (S4)
    const ProblemConst* pc;
    double* scratch;      // [B][nodes]
    double* scratch2;     // [B][nodes] (Scheme 2: per-node history of the current step)
    int stencil;          // Scheme 2 (kind SK_UPWIND)
    unsigned* ctr;        // multi-CTA march: [2] step counters (null: one CTA per problem)
};

struct RhsModesArgs {
    double* R;
    uint64_t N;
    int nodes, B, nmodes, scheme, rhs_mode;
    int node_begin;       // global index of this plan's first node (partitioned plans)
    double h, tau;
    const double* a;      // [B][nmodes]
    const double* k;      // [nmodes]
    const double* p;      // [B][nmodes]
    const int* trig;      // [nmodes]
    const double* u0amp;  // [B] or null
    const double* phiamp; // [B] or null
    const double* wts;    // [B][N+1]: g (S4/ODE) or m (S3) weights
    const double* cvals;  // [B] c (S3/S4) or mu (ODE)
};


struct SpecArgs;
size_t mp_smem_bytes(int G, int m);
bool mp_is_direct(int n);
bool mp_is_single(int n);
constexpr uint64_t kMpScratchBytes = 256ull << 20;  // split K-branch scratch (L2-sized batches)
cudaError_t launch_spectra_single(const double* col, uint64_t N, int B, int n, int J, cplx* spec,
                                  const cplx* tw, cudaStream_t st);
cudaError_t launch_mp(const MpArgs& a, int groups, cudaStream_t st);
int mp_kernel_count(const MpArgs& a);
cudaError_t launch_spectra(const double* col, uint64_t N, int B, int n, int m, int K, int J,
                           cplx* spec, const cplx* tw, int logT, cudaStream_t st);
cudaError_t launch_leaf(int kind, int npt, int L, bool multi, const LeafArgs& a, int ctas,
                        int threads, cudaStream_t st);
cudaError_t launch_leaf_correct(int kind, int npt, int L, const LeafArgs& a, int ctas, cudaStream_t st);
cudaError_t launch_leaf_wbuild(int kind, int L, const LeafArgs& a, int B, double* W, cudaStream_t st);
cudaError_t launch_leaf_fused(int kind, int npt, int L, const LeafArgs& a, int ctas, cudaStream_t st);
bool leaf_pair_ok(const LeafArgs& a, int L);
cudaError_t launch_leaf_pair(int kind, int npt, int L, const LeafArgs& a, int ctas, cudaStream_t st);
cudaError_t launch_leaf_chain(int kind, int npt, int L, const LeafArgs& a, int ctas, cudaStream_t st);
cudaError_t launch_leaf_p2p(int kind, int npt, int L, const LeafArgs& a, int ctas, cudaStream_t st);
cudaError_t launch_p2p_epoch(unsigned* epoch, cudaStream_t st);
// exchange block layout: [0] uint64 arrival counter, [8] uint32 solve epoch, [64..) receive
// buffers [2 parities][P][L][2] doubles
constexpr size_t kP2pHeader = 64;
cudaError_t launch_direct(const DirectArgs& a, int B, cudaStream_t st);
bool ode_whole_ok(uint64_t N);
cudaError_t launch_ode_whole(double* X, const double* R, const double* col, const ProblemConst* pc, uint64_t N,
                             int B, cudaStream_t st);
cudaError_t launch_rhs_modes(const RhsModesArgs& a, cudaStream_t st);
// batched plans' in-leaf weights live in one constant bank per device: acquire it (waits for
// the previous owner's last solve, uploads) before enqueueing a solve, release right after
cudaError_t leaf_bank_acquire(const void* plan, const double* cols_host, int problems, cudaStream_t st);
cudaError_t leaf_bank_release(const void* plan, cudaStream_t st);
void leaf_bank_forget(const void* plan);
int gen_terms(const RhsModesArgs& a);  // J of the separable RHS tables
cudaError_t launch_gen_tables(const RhsModesArgs& a, double* A, double* T, cudaStream_t st);
cudaError_t launch_toeplitz_matvec(const double* col, const double* row, uint64_t n, const double* x, double* y,
                                   double beta, int block_mode, uint64_t vectors, cudaStream_t st);
cudaError_t launch_apply_near(const double* x, double* y, uint64_t N, int nodes, uint64_t rows,
                              const ProblemConst* pc, const double* col, int kind, int L, cudaStream_t st);
cudaError_t launch_resid_max(const double* y, const double* r, uint64_t n, unsigned long long* out, cudaStream_t st);

}  // namespace ftb
