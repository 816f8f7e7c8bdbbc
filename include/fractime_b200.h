/*
 * fractime_b200.h -- C ABI of the B200-native fast solver for the block
 * lower-triangular Toeplitz (BLTT) systems of the L1 Caputo schemes
 * (arXiv 1710.11593).  Drop-in for the reference `fractime` solver entry
 * points (scheme setup, direct solve, fast solve); see INTEGRATION.md for the
 * ctypes / C++ bindings a maintainer adds on the reference side.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   ft_setup / ft_setup_batch  <- validate()                       src/schemes.cpp:58-78
 *                                 SchemeConstants::for_spec()       src/schemes.cpp:44-56
 *                                 g_weights()/m_weights()           src/weights.cpp:28-40
 *                                 assemble_scheme4() (column)       src/schemes.cpp:381-399
 *                                 assemble_scheme3_reordered()      src/schemes.cpp:272-288
 *                                 embed_circulant() (spectra)       src/toeplitz.cpp:84-96
 *   ft_column                  <- ToeplitzOperator::first_col()     include/fractime/toeplitz.hpp:38
 *                                 assemble_scheme2_reordered()      src/schemes.cpp:149-167
 *   ft_assemble_rhs            <- assemble_scheme4() rhs            src/schemes.cpp:401-408
 *                                 Scheme3Rhs::operator()            src/schemes.cpp:300-306
 *                                 Scheme2Rhs::operator()            src/schemes.cpp:183-187
 *   ft_solve_direct            <- solve(spec, SolveMethod::Direct)  src/schemes.cpp:434-463, :333-352,
 *                                                                    :210-232
 *                                 lower_toeplitz_forward_solve()    src/toeplitz.cpp:169-186
 *   ft_solve_fast              <- solve(spec, SolveMethod::Fast)    src/schemes.cpp:464-474, :353-369,
 *                                                                    :233-257
 *   ft_solve_fast_modes        <- the same, with the forcing callback evaluated inside the solve
 *                                 (schemes.cpp:401-408 / :300-306 / :183-187) for separable forcings
 *                                 (GMRES + FFT matvec, src/krylov.cpp:107-223, replaced by a
 *                                 time-axis divide-and-conquer; same system, same answer)
 *   ft_setup_toeplitz          <- ToeplitzOperator::lower_triangular() include/fractime/toeplitz.hpp:33
 *                                 + lower_toeplitz_forward_solve()  src/toeplitz.cpp:169-186
 *                                 (solved by the same D&C in O(n log^2 n); ft_solve_direct keeps
 *                                 the reference's O(n^2) substitution order)
 *   ft_toeplitz_matvec         <- embed_circulant() + toeplitz_matvec() src/toeplitz.cpp:84-115
 *                                 (make_toeplitz_operator, src/toeplitz.cpp:198-201)
 *   ft_block_matvec            <- BlockTridiagonalToeplitzOperator + block_matvec()
 *                                 src/toeplitz.cpp:117-167 (make_block_operator :203-208)
 *   ft_apply / ft_residual     <- make_block_operator() / make_toeplitz_operator() on the plan's own
 *                                 matrix (src/toeplitz.cpp:194-208: the operator the fast path's
 *                                 gmres_solve applies, src/schemes.cpp:464-474), through the plan's
 *                                 FFT history products; SolveReport::residual of a finished solve
 *   ft_setup_partitioned,      <- (no reference counterpart: the reference is single-process) slab
 *   ft_set_exchange,              partition of one wide problem over the GPUs of a node, the carry
 *   ft_nccl_*, ft_p2p_*           all-gather per leaf by the caller's collective, by ncclAllGather
 *                                 inside the captured graph, or by NVLink peer stores
 *   ft_last_error              <- the what() of the reference's std::exception
 *
 * Conventions
 *   - Layout: node-major, values[(i-1)*N + (n-1)] = U_i^n, i = 1..cells-1,
 *     n = 1..N (reference include/fractime/schemes.hpp:209-223).  Batched
 *     plans stack problems: problem b starts at b*(cells-1)*N.  The ODE has
 *     one "node".
 *   - Pointers passed to ft_assemble_rhs_grid / ft_solve_* may be host or
 *     device memory (detected per call).  Host buffers are staged through
 *     plan-owned device memory; device buffers are used in place.  rhs == u
 *     is allowed (in-place solve).
 *   - Errors: functions return FT_OK (0) or a negative FT_E* code; the
 *     message (reference wording where one exists) is in ft_last_error(),
 *     thread-local.  There is no CPU fallback: without a usable CUDA device
 *     every compute entry point fails with FT_ECUDA.
 *   - Threading: a plan is immutable after setup apart from its staging
 *     buffers; use one plan per host thread (distinct plans may run
 *     concurrently on distinct streams: every plan owns its device tables).
 *   - Limits: N <= 65536 time steps (FT_ELENGTH otherwise: the history-product
 *     kernels go up to n = 65536 points); at most 160 slabs of 512 nodes
 *     (81920 interior nodes) per problem and 128 problems per plan (FT_EINVAL);
 *     device memory ~ 2 x rows x N x 8 bytes for device-buffer solves.
 */
#ifndef FRACTIME_B200_H
#define FRACTIME_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Scheme ids follow the reference enum SchemeId (schemes.hpp:182):
 * Ode2Sided=0 (here: the one-sided fractional ODE of BASELINE config 1, built
 * from the reference Toeplitz API as in SURVEY.md 3.4), Hyperbolic=1
 * (reference Scheme 2, transport),
 * DiffusionWave=2 (reference Scheme 3), Diffusion=3 (Scheme 4). */
enum {
    FT_SCHEME_ODE = 0,
    FT_SCHEME_HYPERBOLIC = 1,
    FT_SCHEME_WAVE = 2,
    FT_SCHEME_DIFFUSION = 3
};

enum {
    FT_OK = 0,
    FT_EINVAL = -1,   /* std::invalid_argument */
    FT_EDOM = -2,     /* std::domain_error     */
    FT_ELENGTH = -3,  /* std::length_error     */
    FT_ESOLVER = -4,  /* std::runtime_error    */
    FT_ECUDA = -5,
    FT_ENOMEM = -6
};

/* Right-hand-side mode for the wave scheme (Scheme 3): the reference omits
 * the c*M_0*u0 term in the n = 1 row (schemes.cpp:304).  Mode 0 reproduces
 * the reference; mode 1 adds the term. */
enum { FT_RHS_REFERENCE = 0, FT_RHS_CORRECTED_N1 = 1 };

typedef struct ft_problem {
    int scheme;            /* FT_SCHEME_* */
    double gamma;          /* Caputo order: (0,1) ODE/diffusion, (1,2) wave */
    uint64_t time_steps;   /* N, tau = time_length / N */
    uint64_t space_cells;  /* reference M (cells); interior nodes = cells-1; ignored for ODE */
    double time_length;    /* T */
    double space_length;   /* L, h = L / cells */
} ft_problem;

typedef struct ft_options {
    int rhs_mode;          /* FT_RHS_*; wave scheme only */
    int near_field;        /* lags < near_field are summed exactly in every history
                              product (0 = default: 1 for ODE/diffusion, 64 for wave) */
    int device;            /* CUDA device ordinal (-1 = current) */
    int flags;             /* FT_OPT_* bits (0 = defaults) */
} ft_options;

enum {
    FT_OPT_REPORT_RESIDUAL = 1  /* ft_solve_fast / ft_solve_direct on device buffers (rhs != u) fill
                                   ft_report::residual with max |A u - rhs| / max |rhs|, measured by one
                                   application of the plan's operator (ft_residual); off by default
                                   because it costs about as much as the solve's history products */
};

typedef struct ft_report {
    char method[16];       /* "fast" / "direct" (SolveReport::method) */
    uint64_t iterations;   /* 0: both paths are direct methods (no Krylov matvecs) */
    double residual;       /* 0 by default: both paths are direct solves (no iteration, no residual
                              estimate), as the reference's Direct path reports 0 (SolveReport
                              defaults, schemes.hpp:58-63); with FT_OPT_REPORT_RESIDUAL the measured
                              max |A u - rhs| / max |rhs| (the reference's GMRES reports ||r||_2 / ||b||_2) */
    double seconds;        /* wall time of the call (SolveReport::seconds) */
    double device_ms;      /* device time of the solve proper (CUDA events) */
    uint64_t kernel_launches;  /* kernels this library launched for the call */
} ft_report;

typedef struct ft_plan_info {
    uint64_t problems;     /* batch size B */
    uint64_t nodes;        /* interior nodes per problem (1 for the ODE) */
    uint64_t time_steps;   /* N */
    uint64_t leaf;         /* D&C leaf length */
    uint64_t levels;       /* history-product levels */
    uint64_t slabs;        /* spatial slabs (CTAs) per problem in the leaf solve */
    double h, tau;
    double mu, c;          /* SchemeConstants of problem 0 */
    int rank, world;       /* slab partition of a partitioned plan (0, 1 otherwise) */
    uint64_t node_begin;   /* first interior node (0-based) held by this plan */
    uint64_t local_nodes;  /* nodes held by this plan (rows of its buffers per problem) */
    uint64_t slabs_local;  /* slabs (CTAs) of this rank */
    uint64_t flags;        /* FT_PLAN_* bits: which fast-path kernels the plan's device-buffer solve runs */
} ft_plan_info;

enum {
    FT_PLAN_SLAB_LEAF = 1,      /* multi-slab (space-time SPIKE) leaf */
    FT_PLAN_FUSED_LEAF = 2,     /* one cooperative kernel per leaf */
    FT_PLAN_FUSE0 = 4,          /* the n = 64 history products folded into the leaf */
    FT_PLAN_CLUSTER_MP = 8,     /* K-CTA cluster history products (n = 8192, 16384) */
    FT_PLAN_SPLIT_MP = 16,      /* split K-branch history products with a combine pass (n >= 32768) */
    FT_PLAN_ODE_WHOLE = 32      /* single-node plans: the one-kernel march */
};

typedef struct ft_plan ft_plan;

/* forcing(x, t, user) and initial data u0(x, user) / phi(x, user), evaluated
 * at the reference's points: diffusion/ODE (i h, n tau); wave (i h, (n-1/2) tau);
 * hyperbolic forcing ((i-1/2) h, n tau) and u0 at x_i and x_(i-1). */
typedef double (*ft_forcing_fn)(double x, double t, void* user);
typedef double (*ft_initial_fn)(double x, void* user);

int ft_setup(const ft_problem* problem, const ft_options* options, ft_plan** out);
int ft_setup_batch(const ft_problem* problems, uint64_t count, const ft_options* options,
                   ft_plan** out);
int ft_plan_get_info(const ft_plan* plan, ft_plan_info* info);

/* The carry all-gather as ncclAllGather on the plan's stream, issued by the library itself:
 * no host callback per leaf, and the whole solve (2048 leaves x {phase-1 kernel, all-gather,
 * correction kernel} + the history products) is captured into ONE CUDA graph like the
 * single-GPU solve.  NCCL is bound at run time from the process's libnccl.so.2 (torch's; or
 * FT_NCCL_LIB) -- no link-time dependency.  Rank 0 calls ft_nccl_unique_id and ships the 128
 * bytes to every rank by any transport; every rank then calls ft_nccl_init (collective) on its
 * ft_setup_partitioned plan.  world == 1 is allowed on any wide plan: the same two-kernel leaf
 * and collective run on one GPU (how the path is tested where only one GPU exists). */
int ft_nccl_unique_id(void* id128);
int ft_nccl_init(ft_plan* plan, const void* id128, int rank, int world);

/* Multi-GPU slab partition of one wide problem (BASELINE config 4): rank r of
 * `world` holds the contiguous nodes [node_begin, node_begin + local_nodes)
 * (ft_plan_info); its rhs / u buffers are [local_nodes][N].  History products
 * are node-local; the leaf exchanges its slabs' carries once per leaf through
 * the caller's collective: `exchange(user, count, stream)` must all-gather
 * `count` doubles per rank from every rank's send buffer into the recv buffer
 * (rank-major), ordered on `stream` -- e.g. ncclAllGather on that stream.  The
 * send/recv device buffers (16-byte aligned) are registered with ft_set_exchange. */
typedef int (*ft_exchange_fn)(void* user, uint64_t count_per_rank, void* cuda_stream);
int ft_setup_partitioned(const ft_problem* problem, const ft_options* options, int rank, int world,
                         ft_plan** out);
int ft_set_exchange(ft_plan* plan, ft_exchange_fn exchange, void* user, double* send_device,
                    double* recv_device);
/* Alternative to the hook (opt-in): the leaf kernel exchanges the carries itself
 * over NVLink peer memory.  Each rank allocates its exchange block and exports a
 * CUDA IPC handle (64 bytes) with ft_p2p_handle; the caller all-gathers the
 * handles (rank-major) and passes them to ft_p2p_connect on every rank.  From
 * then on every leaf is one cooperative kernel per rank: phase 1, stores of the
 * carries into every rank's block, a system-scope arrival counter, phases 2/3.
 * All ranks must run the same sequence of fast solves. */
int ft_p2p_handle(ft_plan* plan, void* handle_out);
int ft_p2p_connect(ft_plan* plan, const void* handles);
int ft_column(const ft_plan* plan, uint64_t problem, double* col_host);

int ft_assemble_rhs(const ft_plan* plan, ft_forcing_fn forcing, ft_initial_fn u0,
                    ft_initial_fn phi, void* user, double* rhs_host);
/* Same, from the forcing already sampled at the scheme's points (node-major
 * grid F) and initial data arrays (nodes per problem, NULL = 0; the hyperbolic
 * scheme's u0 holds nodes + 1 values per problem, x_0 .. x_{cells-1}). */
int ft_assemble_rhs_grid(const ft_plan* plan, const double* forcing_grid, const double* u0,
                         const double* phi, double* rhs);
/* Device generation of a separable forcing
 *   f_b(x, t) = sum_j a[b*nmodes+j] * trig_j(k_j pi x) * t^{p[b*nmodes+j]}
 * (trig 0 = sin, 1 = cos, 2 = 1, 3 = x(1-x), 4 = 1-2x), u0_b(x) = u0_amp[b] sin(pi x),
 * phi likewise. */
int ft_assemble_rhs_modes(const ft_plan* plan, int nmodes, const double* a, const double* k,
                          const double* p, const int* trig, const double* u0_amp,
                          const double* phi_amp, double* rhs_device);

int ft_solve_fast(ft_plan* plan, const double* rhs, double* u, ft_report* report);
/* Fast solve with the separable forcing of ft_assemble_rhs_modes generated
 * inside the leaf kernels: the right-hand side is never
 * materialised (no RHS array, no RHS read); the history products accumulate
 * from zero and each leaf adds sum_j A[node][j] T[step][j] while staging.  u:
 * host or device, [rows][N].  Same arguments as ft_assemble_rhs_modes. */
int ft_solve_fast_modes(ft_plan* plan, int nmodes, const double* a, const double* k, const double* p,
                        const int* trig, const double* u0_amp, const double* phi_amp, double* u,
                        ft_report* report);
int ft_solve_direct(ft_plan* plan, const double* rhs, double* u, ft_report* report);

/* y = A x, A the plan's block lower-triangular Toeplitz system matrix -- the operator the
 * reference's fast path hands to GMRES (make_block_operator / make_toeplitz_operator,
 * src/toeplitz.cpp:194-201, applied by block_matvec :150-167 through the FFT circulant
 * embedding :84-115) and the matrix ft_solve_fast inverts.  The far history runs through the
 * plan's own FFT / direct history products (O(M N log N), the level spectra cached at setup);
 * the in-leaf lags and the spatial stencil are added in the difference form
 * (d - 2b) x_i - b ((x_(i-1) - x_i) + (x_(i+1) - x_i)).  x, y: distinct buffers [rows][N], both
 * on the device or both on the host (staged).  Scheme 2 and partitioned plans: FT_EINVAL. */
int ft_apply(ft_plan* plan, const double* x_device, double* y_device);
/* max |A u - rhs| and max |rhs| over all unknowns (the reference's SolveReport::residual is
 * GMRES's; the D&C is direct, so ft_solve_fast reports 0 and this call measures it).  work:
 * a device buffer [rows][N] for A u, or NULL to use the plan's own work buffer. */
int ft_residual(ft_plan* plan, const double* rhs_device, const double* u_device, double* work_device,
                double* max_abs_residual, double* max_abs_rhs);

/* Diagnostics: one fast solve (device buffers only) with a CUDA event
 * between every launch; per-launch device times for roofline accounting.
 * kind 0 = leaf, 1 = history product (level = D&C level, n = 2L << level);
 * first/len give the time range written, rows the rows touched. */
typedef struct ft_op_time {
    int kind;
    int level;
    uint64_t t0;
    uint64_t len;
    uint64_t bytes;  /* algorithmic HBM bytes of the launch */
    float ms;
} ft_op_time;
int ft_profile_fast(ft_plan* plan, const double* rhs_device, double* u_device, ft_op_time* out,
                    uint64_t capacity, uint64_t* count);

/* Host-only (no CUDA needed): the divide-and-conquer launch schedule for N
 * steps and leaf length L -- kind 0 = leaf [t0, t0+len), kind 1 = history
 * product from source [t0 - h, t0) onto target [t0, t0 + len) (level =
 * log2(h / L)).  Used by the CPU test-suite to check the decomposition covers
 * every (source, target) pair of the Toeplitz history exactly once. */
int ft_schedule(uint64_t time_steps, uint64_t leaf, ft_op_time* out, uint64_t capacity,
                uint64_t* count);

/* Lower-triangular Toeplitz systems T_b x_b = r_b, b < count (ToeplitzOperator::
 * lower_triangular + lower_toeplitz_forward_solve, src/toeplitz.cpp:169-186):
 * first_cols[count][n] (host).  The plan solves with ft_solve_fast (the D&C,
 * one "node") or ft_solve_direct (the reference's forward substitution, same
 * summation order); buffers are [count][n].  col[0] == 0 fails with FT_ESOLVER
 * "lower_toeplitz_forward_solve: zero diagonal" like the reference.  The
 * ft_assemble_rhs* calls are rejected on such plans (no scheme). */
int ft_setup_toeplitz(const double* first_cols, uint64_t n, uint64_t count, const ft_options* options,
                      ft_plan** out);

/* y[b] = T x[b], b < count, T the n x n Toeplitz matrix with T(i,j) =
 * first_row[j-i] (j >= i) and first_col[i-j] (i > j); first_row == NULL means
 * lower triangular.  Replaces embed_circulant + toeplitz_matvec
 * (src/toeplitz.cpp:84-115); computed as a direct fp64 product on the GPU (no
 * circulant rounding).  first_col[0] != first_row[0] -> FT_EINVAL with the
 * reference's message (src/toeplitz.cpp:31-32).  All arrays host or device;
 * x == y allowed.  O(n^2) per vector and no setup: meant for one-off products.  A lower
 * triangular operator applied many times (a Krylov loop) should use a Toeplitz plan instead:
 * ft_setup_toeplitz caches the level spectra once and ft_apply(plan, x, y) runs the FFT
 * history products, O(n log n) per vector. */
int ft_toeplitz_matvec(const double* first_col, const double* first_row, uint64_t n, uint64_t count,
                       const double* x, double* y);

/* Block tridiagonal operator of m_blocks identical n x n Toeplitz diagonal
 * blocks and off_scale * I off-diagonal blocks (BlockTridiagonalToeplitzOperator
 * + block_matvec, src/toeplitz.cpp:117-167): y_b = T x_b + off_scale (x_{b-1} +
 * x_{b+1}), added left then right as the reference does.  x, y: [m_blocks][n]. */
int ft_block_matvec(const double* first_col, const double* first_row, uint64_t n, uint64_t m_blocks,
                    double off_scale, const double* x, double* y);

int ft_set_stream(ft_plan* plan, void* cuda_stream);
const char* ft_last_error(void);
void ft_destroy(ft_plan* plan);

#ifdef __cplusplus
}
#endif
#endif /* FRACTIME_B200_H */
