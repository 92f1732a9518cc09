// The attention backward's per-tile MMA mix in isolation (diagnostic): one thread per SM
// issues, per 128-query tile, S^T / dP^T for two 64-query halves (SS, N 64, K-major),
// dV (TS, B MN-major) and dK (SS, B MN-major) per half and dQ (SS, A and B MN-major) per
// tile, with the kernel's SMEM offsets and a commit after every group, nothing waited.
// Prints clk per MMA for the whole mix and for each class alone.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2006_09503_b200/csrc/ptx.cuh"
using namespace p2bw;

constexpr int kTile = 16384;
template <int MASK>  // bit 0 S/dP, bit 1 dV/dK, bit 2 dQ; bit 3: tcgen05.fence::after_thread_sync before every group; bit 4: also an mbarrier wait (already complete) before every group
__global__ void __launch_bounds__(768, 1) k_mix(long long* out, int tiles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[5];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 12 * kTile / 4; i += blockDim.x) {
        // bit 7: pseudo-random bf16 operands in [-2, 2) instead of all 1.0
        uint32_t v = 0x3c003c00u;
        if (MASK & 128) {
            uint32_t x = (i + 1) * 2654435761u;
            x ^= x >> 13;
            x *= 0x5bd1e995u;
            const uint32_t lo = 0x3f80u | (x & 0x007fu) | ((x >> 8) & 0x8000u) | ((x >> 9) & 0x0080u);
            const uint32_t hi = 0x3f80u | ((x >> 16) & 0x007fu) | ((x >> 4) & 0x8000u) | ((x >> 20) & 0x0080u);
            v = lo | (hi << 16);
        }
        reinterpret_cast<uint32_t*>(smem)[i] = v;
    }
    if (threadIdx.x == 0) { for (int i = 0; i < 5; ++i) ptx::mbar_init(&bar[i], 1); ptx::fence_mbar_init(); }
    if (warp == 0) ptx::tmem_alloc<512>(&slot);
    ptx::fence_proxy_async();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t s = ptx::smem_u32(smem);
        const uint32_t aK = s, aV = s + 2 * kTile, aQ = s + 4 * kTile, aDO = s + 6 * kTile, aDS = s + 8 * kTile;
        constexpr uint32_t id_s = ptx::idesc_bf16(128, 64, false, false);
        constexpr uint32_t id_kv = ptx::idesc_bf16(128, 64, false, true);
        constexpr uint32_t id_q = ptx::idesc_bf16(128, 64, true, true);
        long long t0 = clock64();
        int n = 0;
        for (int t = 0; t < tiles; ++t) {
            for (int e = 0; e < 2; ++e) {
                if (MASK & 16) ptx::mbar_wait(&bar[3], 1);  // phase 0 still open: parity 1 is "complete"
                if (MASK & 8) ptx::tc_fence_after();
                if (MASK & 1) {
                    for (int kk = 0; kk < 4; ++kk)
                        ptx::umma_bf16(tmem + 64 * e, ptx::sdesc_sw128(aK + kk * 32, 16, 1024),
                                       ptx::sdesc_sw128(aQ + e * 8192 + kk * 32, 16, 1024), id_s, kk > 0);
                    for (int kk = 0; kk < 4; ++kk)
                        ptx::umma_bf16(tmem + 128 + 64 * e, ptx::sdesc_sw128(aV + kk * 32, 16, 1024),
                                       ptx::sdesc_sw128(aDO + e * 8192 + kk * 32, 16, 1024), id_s, kk > 0);
                    ptx::umma_commit(&bar[0]);
                    n += 8;
                }
                if (MASK & 16) ptx::mbar_wait(&bar[3], 1);
                if (MASK & 8) ptx::tc_fence_after();
                if (MASK & 2) {
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t b_off = (4 * e + kk) * 2048;
                        ptx::umma_bf16_ts(tmem + 256, tmem + 64 * e + 16 * kk, ptx::sdesc_sw128(aDO + b_off, 8192, 1024),
                                          id_kv, 1u);
                        ptx::umma_bf16(tmem + 320, ptx::sdesc_sw128(aDS + e * kTile + kk * 32, 16, 1024),
                                       ptx::sdesc_sw128(aQ + b_off, 8192, 1024), id_kv, 1u);
                    }
                    n += 8;
                }
                if ((MASK & 4) && e == 1) {
                    for (int kk = 0; kk < 8; ++kk)
                        ptx::umma_bf16(tmem + 384 + 64 * (t & 1), ptx::sdesc_sw128(aDS + kk * 2048, kTile, 1024),
                                       ptx::sdesc_sw128(aK + kk * 2048, 8192, 1024), id_q, kk > 0);
                    n += 8;
                }
                if (MASK & 6) ptx::umma_commit(&bar[1 + e]);
            }
        }
        ptx::umma_commit(&bar[3]);
        ptx::mbar_wait(&bar[3], 0);
        long long t1 = clock64();
        out[blockIdx.x * 2] = t1 - t0;
        out[blockIdx.x * 2 + 1] = n;
        ptx::mbar_arrive(&bar[4]);  // release the spinners
    } else if ((MASK & 32) && threadIdx.x >= 128 && (threadIdx.x & 31) == 0) {
        ptx::mbar_wait(&bar[4], 0);  // 20 warps spinning on try_wait meanwhile (lane 0 only)
    } else if ((MASK & 64) && threadIdx.x >= 128) {
        ptx::mbar_wait(&bar[4], 0);  // 20 warps, every lane polling the barrier
    } else if ((MASK & 256) && threadIdx.x >= 128 && threadIdx.x < 640) {
        // 16 warps streaming SMEM stores + loads (the elementwise / flush warps' traffic)
        // into the upper 64 KB until the MMA thread finishes
        uint4* region = reinterpret_cast<uint4*>(smem + 8 * kTile);  // 4096 x 16 B
        uint32_t acc = 0;
        for (int it = 0; !ptx::mbar_test(&bar[4], 0); ++it) {
            const int idx = (threadIdx.x + it * 256) & 4095;
            region[idx] = make_uint4(acc, acc + 1, acc + 2, acc + 3);
            acc += region[idx ^ 128].x;
        }
        if (acc == 0xffffffffu) out[0] = acc;
    } else if ((MASK & 512) && threadIdx.x >= 128 && threadIdx.x < 640) {
        // 16 warps streaming tcgen05.ld of TMEM columns 0-255 (the S / dP reads)
        const int w = threadIdx.x / 32;
        uint32_t acc = 0;
        for (int it = 0; !ptx::mbar_test(&bar[4], 0); ++it) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>((w & 3) * 32) << 16) + ((it * 32) & 255), v);
            ptx::tmem_ld_wait();
            acc += v[0] ^ v[31];
        }
        if (acc == 0x12345678u) out[0] = acc;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

template <int MASK>
void run(long long* d, const char* name) {
    auto k = k_mix<MASK>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * kTile + 1024);
    k<<<148, 768, 12 * kTile + 1024>>>(d, 200);
    cudaDeviceSynchronize();
    k<<<148, 768, 12 * kTile + 1024>>>(d, 200);
    cudaError_t e = cudaDeviceSynchronize();
    long long c[2];
    cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
    printf("%-28s %s: %.1f clk per MMA, %.0f clk per tile\n", name, cudaGetErrorString(e), (double)c[0] / c[1],
           (double)c[0] / 200);
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * 16);
    run<7>(d, "all (S/dP, dV/dK, dQ)");
    run<1>(d, "S/dP only (SS N64 K-major)");
    run<2>(d, "dV/dK only (TS + SS, B MN)");
    run<4>(d, "dQ only (SS, A+B MN-major)");
    run<15>(d, "all + fence per group");
    run<31>(d, "all + wait + fence per group");
    run<39>(d, "all + 20 warps spinning");
    run<63>(d, "all + wait/fence + 20 spinning");
    run<7 | 64>(d, "all + 20 warps x 32 lanes polling");
    run<7 | 128>(d, "all, random operands");
    run<7 | 256>(d, "all + 16 warps of SMEM ld/st");
    run<7 | 512>(d, "all + 16 warps of TMEM loads");
    return 0;
}
