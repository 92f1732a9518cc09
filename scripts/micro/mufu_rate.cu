// MUFU.EX2 and FMNMX3 throughput on one B200 (diagnostic): ops per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__global__ void k_ex2(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = ex2(a[i]) - 1.0f;
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
int main() {
    float* d; cudaMalloc(&d, 148 * 8 * 1024 * 4);
    int iters = 4096;
    for (int blocks_per_sm : {1, 2, 4, 8}) {
        k_ex2<<<148 * blocks_per_sm, 256>>>(d, iters);
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_ex2<<<148 * blocks_per_sm, 256>>>(d, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        float cyc; cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
        double ops = 148.0 * blocks_per_sm * 256 * iters * 8;
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("warps/SM %d: %.3f ms, ex2 per SM per clk (by event, %d MHz max) %.2f; block0 cycles %.0f -> per-SM rate %.2f\n",
               blocks_per_sm * 8, ms, clk / 1000, ops / 148 / (ms * 1e-3 * clk * 1e3), cyc,
               256.0 * blocks_per_sm * iters * 8 / cyc);
    }
    return 0;
}
