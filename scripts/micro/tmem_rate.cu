// tcgen05.ld throughput on one B200 (diagnostic): TMEM bytes read per SM per clock for
// several load shapes and numbers of loads in flight before tcgen05.wait::ld; NW warps per
// CTA, one CTA per SM, warp w reads lane quarter w % 4.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define R8(o) "=r"(v[o]), "=r"(v[o + 1]), "=r"(v[o + 2]), "=r"(v[o + 3]), "=r"(v[o + 4]), "=r"(v[o + 5]), "=r"(v[o + 6]), "=r"(v[o + 7])
template <int SHAPE>
__device__ __forceinline__ void ld(uint32_t a, uint32_t (&v)[32]) {
    if constexpr (SHAPE == 0)  // 32x32b.x32: 32 lanes x 32 cols = 4 KB
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : R8(0), R8(8), R8(16), R8(24) : "r"(a));
    else if constexpr (SHAPE == 1)  // 16x256b.x8: 16 lanes x 64 cols = 4 KB
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : R8(0), R8(8), R8(16), R8(24) : "r"(a));
    else  // 16x128b.x16: 16 lanes x 64 cols... = 16 x 16 B x 16 = 4 KB
        asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : R8(0), R8(8), R8(16), R8(24) : "r"(a));
}

template <int NW, int SHAPE, int INFL>
__global__ void __launch_bounds__(NW * 32, 1) k_tmem(float* out, int iters) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp / 4) * 128;
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; it += INFL) {
        uint32_t v[INFL][32];
#pragma unroll
        for (int u = 0; u < INFL; ++u) ld<SHAPE>(base + (u & 1) * 64, v[u]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < INFL; ++u) acc += __uint_as_float(v[u][0]) + __uint_as_float(v[u][31]);
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x * 2] = (float)(t1 - t0);
    out[1 + blockIdx.x * 2] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
template <int NW, int SHAPE, int INFL>
void run(float* d) {
    const int iters = 8000;
    k_tmem<NW, SHAPE, INFL><<<148, NW * 32>>>(d, iters);
    cudaDeviceSynchronize();
    k_tmem<NW, SHAPE, INFL><<<148, NW * 32>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    float cyc; cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
    const char* nm[] = {"32x32b.x32", "16x256b.x8", "16x128b.x16"};
    printf("%-12s in flight %d, %2d warps: %s, TMEM read %.1f B/clk/SM\n", nm[SHAPE], INFL, NW, cudaGetErrorString(e),
           (double)NW * iters * 4096 / cyc);
}
int main() {
    float* d; cudaMalloc(&d, 148 * 2 * 4);
    run<4, 0, 1>(d); run<4, 0, 2>(d); run<4, 0, 4>(d); run<8, 0, 2>(d); run<16, 0, 1>(d); run<16, 0, 2>(d);
    run<4, 1, 1>(d); run<4, 1, 2>(d); run<8, 1, 2>(d); run<16, 1, 2>(d);
    run<4, 2, 1>(d); run<4, 2, 2>(d); run<8, 2, 2>(d);
    return 0;
}
