// mbarrier round-trip latency between two warps of one CTA (diagnostic): warp 0 lane 0
// and warp 4 lane 0 ping-pong through two mbarriers N times; reported per one-way hop.
// Variants: try_wait loop (ptx::mbar_wait), test_wait spin, and a tcgen05.commit of one
// M128 N64 MMA as the "arrive" on one side (commit -> waiting warp latency).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2006_09503_b200/csrc/ptx.cuh"
using namespace p2bw;

__device__ __forceinline__ void spin_test(uint64_t* bar, uint32_t parity) {
    while (!ptx::mbar_test(bar, parity)) {
    }
}

template <int MODE>  // 0 try_wait both sides, 1 test_wait spin both sides, 2 MMA commit -> try_wait
__global__ void __launch_bounds__(256, 1) k_pp(long long* out, int n) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[2];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar[0], 1);
        ptx::mbar_init(&bar[1], 1);
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<512>(&slot);
    ptx::fence_proxy_async();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t a = ptx::smem_u32(smem), b = a + 16384;
    constexpr uint32_t id = ptx::idesc_bf16(128, 64, false, false);
    if (warp == 0 && lane == 0) {
        long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
            if (MODE == 2) {
                ptx::umma_bf16(tmem + 256, ptx::sdesc_sw128(a, 16, 1024), ptx::sdesc_sw128(b, 16, 1024), id, 0u);
                ptx::umma_commit(&bar[0]);
            } else {
                ptx::mbar_arrive(&bar[0]);
            }
            if (MODE == 1) spin_test(&bar[1], i & 1);
            else ptx::mbar_wait(&bar[1], i & 1);
        }
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    } else if (warp == 4 && lane == 0) {
        for (int i = 0; i < n; ++i) {
            if (MODE == 1) spin_test(&bar[0], i & 1);
            else ptx::mbar_wait(&bar[0], i & 1);
            ptx::mbar_arrive(&bar[1]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

template <int MODE>
void run(long long* d, const char* name) {
    const int n = 4000;
    cudaFuncSetAttribute(k_pp<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    k_pp<MODE><<<148, 256, 40000>>>(d, n);
    cudaDeviceSynchronize();
    k_pp<MODE><<<148, 256, 40000>>>(d, n);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%-44s %s: %.0f clk per round trip\n", name, cudaGetErrorString(e), (double)c / n);
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    run<0>(d, "arrive / try_wait, both sides");
    run<1>(d, "arrive / test_wait spin, both sides");
    run<2>(d, "1 MMA + tcgen05.commit / try_wait, arrive back");
    return 0;
}
