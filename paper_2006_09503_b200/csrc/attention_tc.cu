// Softmax attention forward on tcgen05 tensor cores (head dim 64,
// seq % 128 == 0): key blocks of 64 with a lazy online softmax, P kept in TMEM as the
// A operand of O += P V, 128 TMEM columns and ~50 KB SMEM per CTA so that four CTAs
// share each SM (one's softmax overlaps the others' MMAs and loads).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "launch.h"
#include "profiler.h"
#include "ptx.cuh"
#include "tkernels.h"
#include "util.h"

namespace p2bw {

CUtensorMap make_tmap_bf16_2d(const bf16* ptr, uint64_t inner, uint64_t outer, int64_t ld_elems,
                              uint32_t box_inner, uint32_t box_outer);  // gemm.cu

namespace {

constexpr int kBQ = 128;   // query rows per CTA
constexpr int kBK = 64;    // keys per block
constexpr int kD = 64;
constexpr int kThreads = 256;  // 4 role warps + 4 softmax warps (one per TMEM lane quarter)
constexpr int kRowBytes = 128;                 // one 64-element bf16 row
constexpr int kQBytes = kBQ * kRowBytes;       // 16 KB
constexpr int kKVBytes = kBK * kRowBytes;      // 8 KB
constexpr int kSmemQ = 0;
constexpr int kSmemK = kSmemQ + kQBytes;       // [2] key blocks
constexpr int kSmemV = kSmemK + 2 * kKVBytes;  // [2]
constexpr int kSmemBar = kSmemV + 2 * kKVBytes;
constexpr int kSmemTotal = kSmemBar + 128 + 1024;  // + barriers + alignment slack (~50 KB: 4 CTAs per SM)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescale = 8.0f;  // lazy rescale threshold (log2 units): P <= 2^8 between rescales
// TMEM (128 columns per CTA, so four CTAs share an SM): S block [0, 64) -- P overwrites
// its first 32 columns in place as packed bf16 -- and the O accumulator [64, 128).
constexpr uint32_t tS = 0, tO = 64;

// Phase timestamps of every CTA (debug; null in production): p2bw_debug_attention_timing.
// Per CTA 16 u64: [4 j + 0] softmax warp 4 saw S_j, [4 j + 1] its max done, [4 j + 2]
// its P_j stored, [4 j + 3] MMA thread issued PV_j (j < 4).
__device__ unsigned long long* g_attn_dbg = nullptr;

__device__ __forceinline__ void fmark(bool on, int j, int k) {
    if (on && j < 4) g_attn_dbg[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + 4 * j + k] = clock64();
}

// One CTA per (sequence, head, 128-query tile); four CTAs per SM hide each other's
// MMA / softmax latencies.  Keys stream in blocks of 64 (K/V double-buffered by TMA):
//   UMMA  S = Q K_j^T                 128 x 64 fp32 -> TMEM
//   SIMT  one thread per query row owns the whole block row: lazy online softmax
//         (the running max m only moves when a row's block max exceeds it by > 2^8,
//         and then O and l are rescaled, O in TMEM by the same thread);
//         P = exp2(S*scale - m) -> bf16 -> TMEM over S
//   UMMA  O += P V_j                  A = P from TMEM, B = V_j (MN-major) from SMEM
// The epilogue divides by l = sum P and writes O (bf16) and lse = (m + log2 l) / log2 e.
template <bool kCausal>
__global__ void __launch_bounds__(kThreads, 4)
    k_attn_fwd_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                  bf16* __restrict__ out, float* __restrict__ lse, int seq, int heads) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* bar_q = bar + 0;
    uint64_t* kv_full = bar + 1;   // [2]
    uint64_t* kv_empty = bar + 3;  // [2]
    uint64_t* s_full = bar + 5;
    uint64_t* p_full = bar + 6;    // 4 arrivals
    uint64_t* o_done = bar + 7;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int bh = blockIdx.x, b = bh / heads, hd = bh % heads;
    // causal: the longest query tiles (most key blocks) are scheduled first
    const int qt = kCausal ? static_cast<int>(gridDim.y) - 1 - static_cast<int>(blockIdx.y) : blockIdx.y;
    const int q0 = qt * kBQ;
    const int nb = kCausal ? (q0 + kBQ) / kBK : seq / kBK;  // key blocks this tile sees
    const int h = heads * kD;
    const int row0 = b * seq;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tm_q);
        ptx::tma_prefetch_desc(&tm_kv);
        ptx::mbar_init(bar_q, 1);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&kv_full[i], 1);
            ptx::mbar_init(&kv_empty[i], 1);
        }
        ptx::mbar_init(s_full, 1);
        ptx::mbar_init(p_full, 4);
        ptx::mbar_init(o_done, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<128>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::pdl_trigger();
    ptx::pdl_wait();

    if (warp == 0) {
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(bar_q, kQBytes);
            ptx::tma_load_2d(smem + kSmemQ, &tm_q, bar_q, hd * kD, row0 + q0);
            for (int j = 0; j < nb; ++j) {
                const int buf = j & 1;
                ptx::mbar_wait(&kv_empty[buf], ((j >> 1) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&kv_full[buf], 2 * kKVBytes);
                ptx::tma_load_2d(smem + kSmemK + buf * kKVBytes, &tm_kv, &kv_full[buf], h + hd * kD, row0 + j * kBK);
                ptx::tma_load_2d(smem + kSmemV + buf * kKVBytes, &tm_kv, &kv_full[buf], 2 * h + hd * kD,
                                 row0 + j * kBK);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t q_addr = ptx::smem_u32(smem + kSmemQ);
            constexpr uint32_t id_s = ptx::idesc_bf16(128, kBK, false, false);
            constexpr uint32_t id_pv = ptx::idesc_bf16(128, kD, false, true);
            ptx::mbar_wait(bar_q, 0);
            for (int j = 0; j < nb; ++j) {
                const int buf = j & 1;
                const uint32_t k_addr = ptx::smem_u32(smem + kSmemK + buf * kKVBytes);
                const uint32_t v_addr = ptx::smem_u32(smem + kSmemV + buf * kKVBytes);
                ptx::mbar_wait(&kv_full[buf], (j >> 1) & 1);
                ptx::tc_fence_after();
                // S_j overwrites P_{j-1}: in issue order after PV_{j-1}, which reads it
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk)
                    ptx::umma_bf16(tmem + tS, ptx::sdesc_sw128(q_addr + kk * 32, 16, 1024),
                                   ptx::sdesc_sw128(k_addr + kk * 32, 16, 1024), id_s, kk > 0 ? 1u : 0u);
                ptx::umma_commit(s_full);
                ptx::mbar_wait(p_full, j & 1);
                ptx::tc_fence_after();
                fmark(g_attn_dbg != nullptr, j, 3);
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk)
                    ptx::umma_bf16_ts(tmem + tO, tmem + tS + kk * 8, ptx::sdesc_sw128(v_addr + kk * 2048, 8192, 1024),
                                      id_pv, (j | kk) != 0 ? 1u : 0u);
                ptx::umma_commit(&kv_empty[buf]);
            }
            ptx::umma_commit(o_done);
        }
    } else if (warp >= 4) {
        const int qw = warp & 3;           // TMEM lane quarter
        const int r = qw * 32 + lane;      // query row within the tile
        const int i = q0 + r;
        const uint32_t trow = tmem + (static_cast<uint32_t>(qw * 32) << 16);
        const float sc = 0.125f * kLog2e;
        const bool dbg = g_attn_dbg != nullptr && warp == 4 && lane == 0;
        float m = -INFINITY;  // running max (log2 domain)
        float l = 0.0f;       // row sum at max m
        for (int j = 0; j < nb; ++j) {
            ptx::mbar_wait(s_full, j & 1);
            fmark(dbg, j, 0);
            ptx::tc_fence_after();
            const int kbase = j * kBK;
            const bool diag = kCausal && kbase + kBK > q0;  // block crosses the diagonal
            // block max of the row
            float bm = -INFINITY;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(trow + tS + c * 32, v);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    if (!diag || kbase + c * 32 + e <= i) bm = fmaxf(bm, __uint_as_float(v[e]));
            }
            bm *= sc;
            const float m_new = bm > m + kRescale ? bm : m;  // lazy: only large increases move m
            const bool moved = m_new != m;
            const float f = moved ? (m == -INFINITY ? 0.0f : ptx::ex2(m - m_new)) : 1.0f;
            l *= f;
            m = m_new;
            fmark(dbg, j, 1);
            if (j > 0 && __any_sync(0xffffffffu, moved)) {
                // rescale the O row (rows that did not move scale by 1); PV_{j-1} has
                // completed: S_j's commit covers every earlier MMA
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t o[32];
                    ptx::tmem_ld_32x32b_x32(trow + tO + c * 32, o);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
                    ptx::tmem_st_32x32b_x32(trow + tO + c * 32, o);
                }
            }
            // P = exp2(S * sc - m) -> bf16 -> TMEM over S (keys 0-31 -> columns 0-15,
            // 32-63 -> 16-31, each written after its S columns were read)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(trow + tS + c * 32, v);
                ptx::tmem_ld_wait();
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 32; e += 2) {
                    float p0 = ptx::ex2(fmaf(__uint_as_float(v[e]), sc, -m));
                    float p1 = ptx::ex2(fmaf(__uint_as_float(v[e + 1]), sc, -m));
                    if (diag && kbase + c * 32 + e > i) p0 = 0.0f;
                    if (diag && kbase + c * 32 + e + 1 > i) p1 = 0.0f;
                    l += p0 + p1;
                    pk[e / 2] = ptx::pack_bf16x2(p0, p1);
                }
                ptx::tmem_st_32x32b_x16(trow + tS + c * 16, pk);
            }
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(p_full);
            fmark(dbg, j, 2);
        }
        // epilogue: O / l, lse
        ptx::mbar_wait(o_done, 0);
        ptx::tc_fence_after();
        const float inv = 1.0f / l;
        bf16* orow = out + static_cast<size_t>(row0 + i) * h + hd * kD;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            uint32_t o[32];
            ptx::tmem_ld_32x32b_x32(trow + tO + c * 32, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 w = make_uint4(
                    ptx::pack_bf16x2(__uint_as_float(o[8 * q]) * inv, __uint_as_float(o[8 * q + 1]) * inv),
                    ptx::pack_bf16x2(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv),
                    ptx::pack_bf16x2(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv),
                    ptx::pack_bf16x2(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv));
                *reinterpret_cast<uint4*>(orow + c * 32 + 8 * q) = w;
            }
        }
        lse[static_cast<size_t>(bh) * seq + i] = (m + log2f(l)) / kLog2e;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<128>(tmem);
    }
}

// One attribute call per (instantiation, device).
template <bool kCausal>
void set_smem_once() {
    static std::atomic<uint32_t> done{0};
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    const uint32_t bit = 1u << (dev & 31);
    if (done.load() & bit) return;
    check_cuda(cudaFuncSetAttribute(k_attn_fwd_tc<kCausal>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal),
               "cudaFuncSetAttribute(k_attn_fwd_tc)");
    done.fetch_or(bit);
}

}  // namespace

void attention_debug_timing(unsigned long long* dev_buf) {
    check_cuda(cudaMemcpyToSymbol(g_attn_dbg, &dev_buf, sizeof(dev_buf)), "cudaMemcpyToSymbol(g_attn_dbg)");
}

void attention_fwd_tc(const bf16* qkv, bf16* o, float* lse, int batch, int seq, int heads, bool causal,
                      cudaStream_t s) {
    const int h = heads * kD;
    const uint64_t rows = static_cast<uint64_t>(batch) * seq;
    const CUtensorMap tq = make_tmap_bf16_2d(qkv, 3ull * h, rows, 3ll * h, 64, kBQ);
    const CUtensorMap tkv = make_tmap_bf16_2d(qkv, 3ull * h, rows, 3ll * h, 64, kBK);
    dim3 grid(batch * heads, seq / kBQ);
    if (causal) {
        set_smem_once<true>();
        launch_pdl(k_attn_fwd_tc<true>, grid, dim3(kThreads), kSmemTotal, s, "k_attn_fwd_tc", tq, tkv, o, lse, seq,
                   heads);
    } else {
        set_smem_once<false>();
        launch_pdl(k_attn_fwd_tc<false>, grid, dim3(kThreads), kSmemTotal, s, "k_attn_fwd_tc", tq, tkv, o, lse, seq,
                   heads);
    }
    check_cuda(cudaGetLastError(), "attention_fwd_tc");
}

}  // namespace p2bw
