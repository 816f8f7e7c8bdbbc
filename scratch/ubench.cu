// microbenchmarks: dependent-chain latencies on B200 (sm_100a)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, long long* cyc, double a, int n) {
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = fma(x, a, 1e-9); x = fma(x, a, 1e-9); x = fma(x, a, 1e-9); x = fma(x, a, 1e-9); }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* out, long long* cyc, int n) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = __shfl_up_sync(~0u, x, 1) + 1.0; x = __shfl_up_sync(~0u, x, 1) + 1.0; }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl_only(int* out, long long* cyc, int n) {
    int x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = __shfl_xor_sync(~0u, x, 1); x = __shfl_xor_sync(~0u, x, 2); }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(double* out, long long* cyc, int n) {
    __shared__ double s[256];
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { s[threadIdx.x] = x; __syncthreads(); x = s[(threadIdx.x + 1) & 255] + 1.0; __syncthreads(); }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dfma_tput(double* out, long long* cyc, double a, int n) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        x0 = fma(x0, a, 1e-9); x1 = fma(x1, a, 1e-9); x2 = fma(x2, a, 1e-9); x3 = fma(x3, a, 1e-9);
        x4 = fma(x4, a, 1e-9); x5 = fma(x5, a, 1e-9); x6 = fma(x6, a, 1e-9); x7 = fma(x7, a, 1e-9);
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double* out; long long* cyc; int* io;
    cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8 * 1024); cudaMalloc(&io, 4096);
    long long h[4];
    int n = 10000;
    k_dfma<<<1, 32>>>(out, cyc, 0.999, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cyc\n", h[0] / (4.0 * n));
    k_shfl<<<1, 32>>>(out, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("SHFL(double)+DADD dependent: %.2f cyc per pair\n", h[0] / (2.0 * n));
    k_shfl_only<<<1, 32>>>(io, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("SHFL(int) dependent: %.2f cyc\n", h[0] / (2.0 * n));
    k_bar<<<1, 256>>>(out, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("STS+BAR+LDS+DADD+BAR (256 thr): %.2f cyc\n", h[0] / (1.0 * n));
    for (int thr : {32, 128, 256, 512, 1024}) {
        k_dfma_tput<<<148, thr>>>(out, cyc, 0.999, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA throughput %4d thr/SM: %.1f DFMA/clk/SM\n", thr, 8.0 * n * thr / h[0]);
    }
    return 0;
}
