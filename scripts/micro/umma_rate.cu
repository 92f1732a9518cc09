// tcgen05.mma throughput on one B200 (diagnostic): cycles per 128 x N x 16 bf16 MMA for
// operands from SMEM (SS) or A from TMEM (TS), B K-major or MN-major, one CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2006_09503_b200/csrc/ptx.cuh"
using namespace p2bw;

template <int N, bool TS, bool BMN, int NACC = 1, int COMMIT = 0>
__global__ void __launch_bounds__(128, 1) k_mma(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::mbar_init(&bar2, 1); ptx::fence_mbar_init(); }
    if (warp == 0) ptx::tmem_alloc<512>(&slot);
    ptx::fence_proxy_async();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t a = ptx::smem_u32(smem), b = a + 32768;
        constexpr uint32_t id = ptx::idesc_bf16(128, N, false, BMN);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t bd = BMN ? ptx::sdesc_sw128(b + kk * 2048, 8192, 1024) : ptx::sdesc_sw128(b + (kk & 3) * 32, 16, 1024);
                // NACC independent accumulators, round robin (N <= 64: 4 x 64 columns at 256..511)
                const uint32_t acc = tmem + 256 + (kk % NACC) * (N <= 64 ? 64 : 128);
                if constexpr (TS) ptx::umma_bf16_ts(acc, tmem + kk * 8, bd, id, 1u);
                else ptx::umma_bf16(acc, ptx::sdesc_sw128(a + (kk & 3) * 32, 16, 1024), bd, id, 1u);
                // COMMIT > 0: a tcgen05.commit to a second mbarrier after every COMMIT MMAs (never waited)
                if constexpr (COMMIT > 0)
                    if ((kk + 1) % COMMIT == 0) ptx::umma_commit(&bar2);
            }
        }
        ptx::umma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}
template <int N, bool TS, bool BMN, int NACC = 1, int COMMIT = 0>
void run(long long* d) {
    const int iters = 2000;
    auto k = k_mma<N, TS, BMN, NACC, COMMIT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    k<<<148, 128, 70000>>>(d, iters);
    cudaDeviceSynchronize();
    k<<<148, 128, 70000>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("M128 N%-3d K16 %s B %s, %d accumulator(s), commit every %d: %s, %.1f clk per MMA (ideal %d)\n", N,
           TS ? "TS (A in TMEM)" : "SS", BMN ? "MN-major" : "K-major", NACC, COMMIT, cudaGetErrorString(e),
           (double)c / (iters * 8), 128 * N / 256);
}
int main() {
    long long* d; cudaMalloc(&d, 148 * 8);
    run<16, true, false>(d); run<16, false, false>(d); run<32, true, false>(d);
    run<64, false, false>(d); run<64, false, true>(d); run<64, true, true>(d); run<64, true, false>(d);
    run<128, false, false>(d); run<128, true, false>(d); run<256, false, false>(d); run<256, true, false>(d);
    // independent accumulators: is the ~45 clk floor of small-N MMAs a dependency chain?
    run<64, true, true, 2>(d); run<64, true, true, 4>(d); run<64, false, true, 4>(d); run<32, true, false, 4>(d);
    run<128, true, false, 2>(d);
    // commit cost: one tcgen05.commit per 8 / 4 / 2 MMAs
    run<64, false, false, 1, 8>(d); run<64, false, false, 1, 4>(d); run<64, false, false, 1, 2>(d);
    run<128, false, false, 1, 4>(d);
    return 0;
}
