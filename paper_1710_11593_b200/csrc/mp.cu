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

#include "fft.cuh"
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace ftb {

__device__ __forceinline__ cplx conjc(cplx a) { return {a.x, -a.y}; }

__global__ void __launch_bounds__(kMpThreads) mp_kernel(MpArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx* buf = reinterpret_cast<cplx*>(smem_raw);
    cg::cluster_group cluster = cg::this_cluster();
    const int b = (int)cluster.block_rank();
    const int K = a.K, m = a.m, G = a.G, n = a.n;
    const int logm = __ffs(m) - 1, logn = __ffs(n) - 1, logK = __ffs(K) - 1;
    const int shT_n = a.logT - logn, shT_K = a.logT - logK;
    const int total = G * m;
    const int npairs = (a.rows / a.nodes) * a.pairs_per_problem;
    const int pair0 = blockIdx.y * G;
    const uint64_t N = a.N;

    // 1. fold the (zero-padded) source block into branch b and twist
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int g = idx >> logm, r = idx & (m - 1);
        const int rp = pair0 + g;
        cplx v = {0.0, 0.0};
        if (rp < npairs) {
            const int pb = rp / a.pairs_per_problem, lp = rp - pb * a.pairs_per_problem;
            const int i1 = 2 * lp;
            const bool has2 = i1 + 1 < a.nodes;
            const double* x1 = a.X + (uint64_t)(pb * a.nodes + i1) * N + a.lo;
            for (int q = 0; q < K / 2; ++q) {
                const int j = q * m + r;
                const cplx z = {x1[j], has2 ? x1[N + j] : 0.0};
                if (q == 0) {
                    v = cadd(v, z);
                } else {
                    const cplx zeta = conjc(ldgc(&a.tw[((b * q) & (K - 1)) << shT_K]));
                    v = cadd(v, cmul(z, zeta));
                }
            }
            if (b) v = cmulc(v, ldgc(&a.tw[(b * r) << shT_n]));  // * exp(+2 pi i b r / n)
        }
        buf[sphys(idx)] = v;
    }
    __syncthreads();

    // 2. branch convolution: forward FFT, multiply by the kernel spectrum, inverse FFT
    fft_forward(buf, total, logm, a.tw, a.logT);
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int g = idx >> logm, r = idx & (m - 1);
        const int rp = min(pair0 + g, npairs - 1);
        const int pb = rp / a.pairs_per_problem;
        const cplx s = ldgc(&a.spec[((uint64_t)pb * K + b) * m + r]);
        buf[sphys(idx)] = cmul(buf[sphys(idx)], s);
    }
    __syncthreads();
    fft_inverse(buf, total, logm, a.tw, a.logT);
    cluster.sync();

    // 3. inverse K-point DFT across the cluster's branches (DSMEM), near field, store
    const int slice = m / K;
    const int halfK = K / 2;
    const uint64_t tend = a.hi < N ? a.hi : N;
    const int work = G * slice * halfK;
    for (int idx = threadIdx.x; idx < work; idx += blockDim.x) {
        const int rr = idx % slice;
        const int tmp = idx / slice;
        const int qq = tmp % halfK;
        const int g = tmp / halfK;
        const int r = b * slice + rr;
        const int q = halfK + qq;
        const int rp = pair0 + g;
        if (rp >= npairs) continue;
        const uint64_t t = a.mid + (uint64_t)qq * m + r;
        if (t >= tend) continue;
        cplx y = {0.0, 0.0};
        for (int bb = 0; bb < K; ++bb) {
            const cplx* rb = cluster.map_shared_rank(buf, bb);
            const cplx w = rb[sphys(g * m + r)];
            const int e = (bb * (q * m + r)) & (n - 1);
            y = cadd(y, cmul(w, ldgc(&a.tw[e << shT_n])));
        }
        const int pb = rp / a.pairs_per_problem, lp = rp - pb * a.pairs_per_problem;
        const int i1 = 2 * lp;
        const bool has2 = i1 + 1 < a.nodes;
        const uint64_t row1 = (uint64_t)(pb * a.nodes + i1);
        const int tp = (int)(t - a.mid);
        if (tp < a.J - 1) {  // exact near field: lags t - j < J
            const double* cp = a.col + (uint64_t)pb * N;
            const double* x1 = a.X + row1 * N;
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
        a.X[row1 * N + t] = a.rsrc[row1 * N + t] - y.x;
        if (has2) a.X[(row1 + 1) * N + t] = a.rsrc[(row1 + 1) * N + t] - y.y;
    }
    cluster.sync();
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
    const int logm = __ffs(m) - 1, logn = __ffs(n) - 1, logK = __ffs(K) - 1;
    const double* col = a.col + (uint64_t)pb * a.N;
    const uint64_t kend = (uint64_t)n < a.N ? (uint64_t)n : a.N;
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
        cplx v = {0.0, 0.0};
        for (int q = 0; q < K; ++q) {
            const uint64_t k = (uint64_t)q * m + r;
            const double c = (k >= (uint64_t)a.J && k < kend) ? col[k] : 0.0;
            const cplx zeta = conjc(a.tw[((b * q) & (K - 1)) << (a.logT - logK)]);
            v = cadd(v, cplx{c * zeta.x, c * zeta.y});
        }
        v = cmulc(v, a.tw[(b * r) << (a.logT - logn)]);
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

cudaError_t launch_mp(const MpArgs& a, int groups, cudaStream_t st) {
    const size_t smem = mp_smem_bytes(a.G, a.m);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(mp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mp_smem_bytes(1, 8192));
        cudaFuncSetAttribute(mp_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.K, groups, 1);
    cfg.blockDim = dim3(kMpThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, mp_kernel, a);
}

cudaError_t launch_spectra(const double* col, uint64_t N, int B, int n, int m, int K, int J,
                           cplx* spec, const cplx* tw, int logT, cudaStream_t st) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(spectra_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mp_smem_bytes(1, 8192));
        attr_set = true;
    }
    SpecArgs a{col, N, n, m, K, J, spec, tw, logT};
    spectra_kernel<<<dim3(K, B), kMpThreads, mp_smem_bytes(1, m), st>>>(a);
    return cudaGetLastError();
}

}  // namespace ftb
