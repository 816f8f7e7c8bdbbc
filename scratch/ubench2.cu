// microbenchmarks 2: SMEM / barrier handshake latencies on B200 (sm_100a)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void nsync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void narrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void k_lds_chase(int* out, long long* cyc, int n) {
    __shared__ int s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 33) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { p = s[p]; p = s[p]; p = s[p]; p = s[p]; }
    long long t1 = clock64();
    out[threadIdx.x] = p; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds_d(double* out, long long* cyc, int n) {
    __shared__ double s[64];
    s[threadIdx.x] = threadIdx.x;
    __syncwarp();
    double x = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { s[threadIdx.x] = x; __syncwarp(); x = s[threadIdx.x ^ 1] + 1.0; __syncwarp(); }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_clock(long long* out, long long* cyc, int n) {
    long long acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) acc += clock64();
    long long t1 = clock64();
    out[threadIdx.x] = acc; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// handshake: warp 0 produces x -> smem, arrive(1); warp 1 syncs(1), reads, writes y, arrive(2); warp 0 syncs(2)
__global__ void k_handshake(double* out, long long* cyc, int n) {
    __shared__ double a[32], b[32];
    double x = threadIdx.x;
    long long t0 = clock64();
    if (threadIdx.x < 32) {
        for (int i = 0; i < n; ++i) {
            a[threadIdx.x] = x;
            narrive(1, 64);
            nsync(2, 64);
            x = b[threadIdx.x] + 1.0;
        }
    } else {
        for (int i = 0; i < n; ++i) {
            nsync(1, 64);
            const double y = a[threadIdx.x - 32] * 0.5;
            b[threadIdx.x - 32] = y;
            narrive(2, 64);
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// 4-warp named barrier sync with smem exchange
__global__ void k_bar4(double* out, long long* cyc, int n) {
    __shared__ double s[128];
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { s[threadIdx.x] = x; nsync(3, 128); x = s[(threadIdx.x + 32) & 127] + 1.0; nsync(3, 128); }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// scan step like phase 2: 5 double shuffle rounds (F up, B down) with fma
__global__ void k_scan(double* out, long long* cyc, int n) {
    double SF = threadIdx.x, SB = threadIdx.x;
    const double p = 0.999;
    const int lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            const double pf = lane >= (1 << d) ? p : 0.0, pb = lane + (1 << d) < 32 ? p : 0.0;
            SF = fma(pf, __shfl_up_sync(~0u, SF, 1 << d), SF);
            SB = fma(pb, __shfl_down_sync(~0u, SB, 1 << d), SB);
        }
        SF = SF * 1e-3 + SB * 1e-3; SB = SF;
    }
    long long t1 = clock64();
    out[threadIdx.x] = SF + SB; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* out; long long* cyc; int* io; long long* lo;
    cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8 * 1024); cudaMalloc(&io, 4096); cudaMalloc(&lo, 8192);
    long long h[4];
    int n = 10000;
    k_lds_chase<<<1, 32>>>(io, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS.32 dependent (pointer chase): %.2f cyc\n", h[0] / (4.0 * n));
    k_lds_d<<<1, 32>>>(out, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("STS.64+syncwarp+LDS.64+DADD+syncwarp: %.2f cyc\n", h[0] / (1.0 * n));
    k_clock<<<1, 32>>>(lo, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("clock64 read: %.2f cyc\n", h[0] / (1.0 * n));
    k_handshake<<<1, 64>>>(out, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("arrive/sync handshake round trip (2 warps): %.2f cyc\n", h[0] / (1.0 * n));
    k_bar4<<<1, 128>>>(out, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("STS+namedbar(128)+LDS+DADD+namedbar: %.2f cyc\n", h[0] / (1.0 * n));
    k_scan<<<1, 32>>>(out, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("5-round F/B double shuffle scan: %.2f cyc\n", h[0] / (1.0 * n));
    k_scan<<<1, 128>>>(out, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("5-round F/B double shuffle scan (4 warps): %.2f cyc\n", h[0] / (1.0 * n));
    return 0;
}
