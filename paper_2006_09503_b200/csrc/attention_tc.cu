// Softmax attention forward on tcgen05 tensor cores (head dim 64, seq <= 512,
// seq % 128 == 0).  One CTA per (sequence, head, 128-query tile):
//
//   TMA     Q tile [128 x 64], K and V rows [kv x 64] of the head (one 2-D map over
//           qkv [T x 3h], box 64 x 128, 128-byte swizzle) -> SMEM
//   UMMA    S = Q K^T for every key at once: 128 x kv fp32 in TMEM (<= 512 columns)
//   softmax two threads per query row (8 warps; thread half `sel` takes the
//           interleaved 32-key chunks 2j+sel): pass 1 row max, pass 2 exp2 and
//           sum -- exact, no online rescaling, because the whole row is resident.
//           Row max / sum are exchanged through SMEM (fixed order: deterministic).
//           P is written as bf16 straight into SMEM in the UMMA K-major SW128 layout
//   UMMA    O = P V (V read as an MN-major operand), TMEM columns 0..63, issued per
//           256-key half so the second half's exp overlaps the first half's MMA
//   epilogue O / l -> bf16 -> global (each row thread stores 32 of the 64 columns);
//           lse = m + ln l (fp32) for the backward
//
// SMEM: Q 16 KB + K 64 KB + V 64 KB + P 64 KB (the second P half reuses K's
// buffer once S is complete) = 208 KB; TMEM: 512 columns.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "profiler.h"
#include "ptx.cuh"
#include "tkernels.h"
#include "util.h"

namespace p2bw {

CUtensorMap make_tmap_bf16_2d(const bf16* ptr, uint64_t inner, uint64_t outer, int64_t ld_elems,
                              uint32_t box_inner, uint32_t box_outer);  // gemm.cu

namespace {

constexpr int kBQ = 128;
constexpr int kD = 64;
constexpr int kGroups = 4;                     // softmax threads per query row
constexpr int kThreads = 128 + 128 * kGroups;  // 4 role warps + 4*kGroups softmax warps
constexpr int kRowBytes = 128;                 // one 64-element bf16 row
constexpr int kTileBytes = kBQ * kRowBytes;    // 16 KB: 128 rows
constexpr int kSmemQ = 0;
constexpr int kSmemK = kSmemQ + kTileBytes;            // 4 tiles
constexpr int kSmemV = kSmemK + 4 * kTileBytes;        // 4 tiles
constexpr int kSmemP = kSmemV + 4 * kTileBytes;        // 4 blocks of 64 keys
constexpr int kSmemX = kSmemP + 4 * kTileBytes;        // row max / sum exchange [2][kGroups][128] f32
constexpr int kSmemBar = kSmemX + 2 * kGroups * kBQ * 4;
constexpr int kSmemTotal = kSmemBar + 128 + 1024;      // + barriers + alignment slack
constexpr float kLog2e = 1.4426950408889634f;

// Writes 32 consecutive keys' bf16 probabilities of row r into a K-major SW128
// block set (64 keys per 16 KB block).
__device__ __forceinline__ void store_p32(uint8_t* pbase, int r, int key0, const float (&p)[32]) {
    uint8_t* blk = pbase + (key0 / 64) * kTileBytes + r * kRowBytes;
    const int chunk0 = (key0 % 64) / 8;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint4 v = make_uint4(ptx::pack_bf16x2(p[8 * q], p[8 * q + 1]), ptx::pack_bf16x2(p[8 * q + 2], p[8 * q + 3]),
                                   ptx::pack_bf16x2(p[8 * q + 4], p[8 * q + 5]),
                                   ptx::pack_bf16x2(p[8 * q + 6], p[8 * q + 7]));
        const int c = (chunk0 + q) ^ (r & 7);
        *reinterpret_cast<uint4*>(blk + c * 16) = v;
    }
}

// Phase timestamps of every CTA (debug; null in production): p2bw_debug_attention_timing.
__device__ unsigned long long* g_attn_dbg = nullptr;

__device__ __forceinline__ void dbg_mark(unsigned long long* d, int slot) {
    if (d != nullptr) d[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + slot] = clock64();
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void softmax_bar(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(128 * kGroups) : "memory");
}

template <bool kCausal>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_fwd_tc(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ out, float* __restrict__ lse,
                  int seq, int heads) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* bar_qk = bar + 0;
    uint64_t* bar_v = bar + 1;
    uint64_t* bar_s = bar + 2;
    uint64_t* bar_p = bar + 3;  // [2], 8 arrivals (one per softmax warp)
    uint64_t* bar_o = bar + 5;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 6);
    float* xmax = reinterpret_cast<float*>(smem + kSmemX);  // [2][128]
    float* xsum = xmax + kGroups * kBQ;                      // [kGroups][128]

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int bh = blockIdx.x, b = bh / heads, hd = bh % heads;
    const int q0 = blockIdx.y * kBQ;
    const int kv = kCausal ? q0 + kBQ : seq;  // keys this tile can see (multiple of 128)
    const int halves = (kv + 255) / 256;
    const int h = heads * kD;
    const int row0 = b * seq;  // first token row of this sequence

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tm);
        for (int i = 0; i < 6; ++i) ptx::mbar_init(&bar[i], i == 3 || i == 4 ? 4 * kGroups : 1);
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(bar_qk, kTileBytes + kv * kRowBytes);
            ptx::tma_load_2d(smem + kSmemQ, &tm, bar_qk, hd * kD, row0 + q0);
            for (int t = 0; t < kv / kBQ; ++t)
                ptx::tma_load_2d(smem + kSmemK + t * kTileBytes, &tm, bar_qk, h + hd * kD, row0 + t * kBQ);
            ptx::mbar_arrive_expect_tx(bar_v, kv * kRowBytes);
            for (int t = 0; t < kv / kBQ; ++t)
                ptx::tma_load_2d(smem + kSmemV + t * kTileBytes, &tm, bar_v, 2 * h + hd * kD, row0 + t * kBQ);
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t q_addr = ptx::smem_u32(smem + kSmemQ);
            const uint32_t k_addr = ptx::smem_u32(smem + kSmemK);
            const uint32_t v_addr = ptx::smem_u32(smem + kSmemV);
            ptx::mbar_wait(bar_qk, 0);
            ptx::tc_fence_after();
            for (int c = 0; c * 256 < kv; ++c) {
                const int n = kv - c * 256 < 256 ? kv - c * 256 : 256;
                const uint32_t idesc = ptx::idesc_bf16(128, n, false, false);
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) {
                    const uint64_t ad = ptx::sdesc_sw128(q_addr + kk * 32, 16, 1024);
                    const uint64_t bd = ptx::sdesc_sw128(k_addr + c * 2 * kTileBytes + kk * 32, 16, 1024);
                    ptx::umma_bf16(tmem + c * 256, ad, bd, idesc, kk > 0 ? 1u : 0u);
                }
            }
            ptx::umma_commit(bar_s);
            ptx::mbar_wait(bar_v, 0);
            const uint32_t idesc_pv = ptx::idesc_bf16(128, kD, false, true);
            for (int hf = 0; hf < halves; ++hf) {
                ptx::mbar_wait(&bar_p[hf], 0);
                ptx::tc_fence_after();
                const uint32_t p_addr = ptx::smem_u32(smem + (hf == 0 ? kSmemP : kSmemK));
                const int steps = (kv - hf * 256 < 256 ? kv - hf * 256 : 256) / 16;
                for (int kk = 0; kk < steps; ++kk) {
                    const uint64_t ad = ptx::sdesc_sw128(p_addr + (kk / 4) * kTileBytes + (kk % 4) * 32, 16, 1024);
                    const uint64_t bd = ptx::sdesc_sw128(v_addr + (hf * 16 + kk) * 2048, 8192, 1024);
                    ptx::umma_bf16(tmem, ad, bd, idesc_pv, (hf | kk) != 0 ? 1u : 0u);
                }
            }
            ptx::umma_commit(bar_o);
        }
    } else if (warp >= 4) {
        const int qw = warp & 3;          // TMEM lane quarter
        const int sel = (warp - 4) >> 2;  // which interleaved 32-key chunks (of kGroups)
        const int r = qw * 32 + lane;     // query row within the tile
        const int i = q0 + r;
        const int n_valid = kCausal ? i + 1 : kv;
        const uint32_t trow = tmem + (static_cast<uint32_t>(qw * 32) << 16);
        unsigned long long* dbg = (warp == 4 && lane == 0) ? g_attn_dbg : nullptr;
        dbg_mark(dbg, 0);
        if (dbg) dbg[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + 8] = gtimer();
        ptx::mbar_wait(bar_s, 0);
        ptx::tc_fence_after();
        dbg_mark(dbg, 1);
        float m0 = -INFINITY, m1 = -INFINITY;
        for (int c = sel * 32; c < kv; c += 32 * kGroups) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(trow + c, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
                if (c + j < n_valid) m0 = fmaxf(m0, __uint_as_float(v[j]));
                if (c + j + 1 < n_valid) m1 = fmaxf(m1, __uint_as_float(v[j + 1]));
            }
        }
        xmax[sel * kBQ + r] = fmaxf(m0, m1);
        dbg_mark(dbg, 2);
        softmax_bar(1);
        dbg_mark(dbg, 3);
        float m = xmax[r];
#pragma unroll
        for (int g = 1; g < kGroups; ++g) m = fmaxf(m, xmax[g * kBQ + r]);
        const float sc = 0.125f * kLog2e;
        const float mc = m * sc;
        float l[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (int hf = 0; hf < halves; ++hf) {
            uint8_t* pbuf = smem + (hf == 0 ? kSmemP : kSmemK);
            const int end = kv < (hf + 1) * 256 ? kv : (hf + 1) * 256;
            for (int c = hf * 256 + sel * 32; c < end; c += 32 * kGroups) {
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(trow + c, v);
                ptx::tmem_ld_wait();
                float p[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    p[j] = c + j < n_valid ? ptx::ex2(fmaf(__uint_as_float(v[j]), sc, -mc)) : 0.0f;
                    l[j & 3] += p[j];
                }
                store_p32(pbuf, r, c - hf * 256, p);
            }
            ptx::fence_proxy_async();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&bar_p[hf]);
        }
        xsum[sel * kBQ + r] = (l[0] + l[1]) + (l[2] + l[3]);
        dbg_mark(dbg, 4);
        softmax_bar(2);
        float ltot = xsum[r];
#pragma unroll
        for (int g = 1; g < kGroups; ++g) ltot += xsum[g * kBQ + r];
        const float inv = 1.0f / ltot;
        dbg_mark(dbg, 5);
        ptx::mbar_wait(bar_o, 0);
        ptx::tc_fence_after();
        dbg_mark(dbg, 6);
        bf16* orow = out + static_cast<size_t>(row0 + i) * h + hd * kD + sel * (kD / kGroups);
        {
            uint32_t v[16];
            ptx::tmem_ld_32x32b_x16(trow + sel * (kD / kGroups), v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint4 w = make_uint4(
                    ptx::pack_bf16x2(__uint_as_float(v[8 * q]) * inv, __uint_as_float(v[8 * q + 1]) * inv),
                    ptx::pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv),
                    ptx::pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv),
                    ptx::pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv));
                *reinterpret_cast<uint4*>(orow + 8 * q) = w;
            }
        }
        if (sel == 0) lse[static_cast<size_t>(bh) * seq + i] = (mc + log2f(ltot)) / kLog2e;
        dbg_mark(dbg, 7);
        if (dbg) dbg[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + 9] = gtimer();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
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

bool attention_tc_supported(int seq) { return seq >= 128 && seq <= 512 && seq % 128 == 0; }

void attention_debug_timing(unsigned long long* dev_buf) {
    check_cuda(cudaMemcpyToSymbol(g_attn_dbg, &dev_buf, sizeof(dev_buf)), "cudaMemcpyToSymbol(g_attn_dbg)");
}

void attention_fwd_tc(const bf16* qkv, bf16* o, float* lse, int batch, int seq, int heads, bool causal,
                      cudaStream_t s) {
    const int h = heads * kD;
    const CUtensorMap tm = make_tmap_bf16_2d(qkv, 3ull * h, static_cast<uint64_t>(batch) * seq, 3ll * h, 64, 128);
    dim3 grid(batch * heads, seq / kBQ);
    if (causal) {
        set_smem_once<true>();
        k_attn_fwd_tc<true><<<grid, kThreads, kSmemTotal, s>>>(tm, o, lse, seq, heads);
    } else {
        set_smem_once<false>();
        k_attn_fwd_tc<false><<<grid, kThreads, kSmemTotal, s>>>(tm, o, lse, seq, heads);
    }
    check_cuda(cudaGetLastError(), "attention_fwd_tc");
}

}  // namespace p2bw
