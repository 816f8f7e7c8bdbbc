// Do DFMA (FP64 pipe) and DMMA m8n8k4 (tensor) run concurrently on B200?  Three kernels:
// pure DFMA, pure DMMA, interleaved; aggregate TFLOP/s of each.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void __launch_bounds__(256) k(double* out, double a, double b) {
    double f[8], m[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { f[i] = threadIdx.x * 1e-3 + i; m[i][0] = i; m[i][1] = -i; }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE != 1) f[i] = fma(f[i], a, b);
            if (MODE == 1 || MODE == 2 || (MODE == 3 && i == 0) || (MODE == 4 && (i & 3) == 0)) dmma(m[i][0], m[i][1], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += f[i] + m[i][0] + m[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
double run(double* out, const char* name) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int grid = 148 * 8;
    k<MODE><<<grid, 256>>>(out, 0.999999, 1e-9);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<MODE><<<grid, 256>>>(out, 0.999999, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    const double thr = (double)grid * 256, per = (double)ITERS * 8;
    const double fl_fma = MODE != 1 ? thr * per * 2 : 0;                    // 2 flops per DFMA per thread
    const double frac = MODE == 3 ? 0.125 : MODE == 4 ? 0.25 : 1.0;
    const double fl_mma = MODE != 0 ? frac * (thr / 32) * per * (8 * 8 * 4 * 2) : 0;  // 512 flops per warp DMMA
    printf("%-12s %.3f ms  DFMA %.1f TFLOP/s  DMMA %.1f TFLOP/s  total %.1f\n", name, ms, fl_fma / ms / 1e9,
           fl_mma / ms / 1e9, (fl_fma + fl_mma) / ms / 1e9);
    return ms;
}
int main() {
    double* out; cudaMalloc(&out, 148 * 8 * 256 * 8);
    run<0>(out, "DFMA only"); run<1>(out, "DMMA only"); run<2>(out, "interleaved"); run<3>(out, "8 DFMA:1 DMMA"); run<4>(out, "4 DFMA:1 DMMA");
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
