// Softmax attention backward on tcgen05 tensor cores (head dim 64, seq % 128 == 0,
// seq <= 512).  Key-outer: one CTA per (sequence, head, 128-key tile j) walks the
// query tiles i that can see it (all of them, or i >= j when causal):
//
//   UMMA  S^T  = K_j Q_i^T          128 x 128 fp32, TMEM [0, 128)
//   UMMA  dP^T = V_j dO_i^T         TMEM [128, 256)
//   SIMT  P^T  = exp(S^T/8 - lse_i), dS^T = P^T (dP^T - delta_i)  (thread = key row)
//         written as bf16 into SMEM in the UMMA K-major SW128 layout
//   UMMA  dV_j += P^T dO_i          TMEM [256, 320)   (dO_i read MN-major)
//   UMMA  dK_j += dS^T Q_i          TMEM [320, 384)   (Q_i read MN-major)
//   UMMA  dQ_i|j = dS K_j           TMEM [384, 448)   (dS^T read MN-major, K_j MN-major)
//
// The same SMEM bytes serve as K-major and MN-major operands (a 128-byte swizzled
// row of 64 elements is both "64 k-values of one row" and "64 mn-values of one
// k"), so no transposes are materialised.  dQ partials are written per key tile
// (fp32, no atomics) and summed in fixed order by a small kernel: deterministic.
// Q_i / dO_i / lse_i / delta_i are double-buffered so TMA overlaps compute.
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

constexpr int kT = 128;   // tile rows (keys or queries)
constexpr int kD = 64;
constexpr int kTile = kT * 128;  // 16 KB
constexpr int oK = 0, oV = oK + kTile;
constexpr int oQ = oV + kTile;          // [2] tiles
constexpr int oDO = oQ + 2 * kTile;     // [2]
constexpr int oPt = oDO + 2 * kTile;    // 2 blocks (q 0-63, 64-127)
constexpr int oDSt = oPt + 2 * kTile;   // 2 blocks
constexpr int oLse = oDSt + 2 * kTile;  // [2][128] f32
constexpr int oDel = oLse + 2 * kT * 4; // [2][128] f32
constexpr int oBar = oDel + 2 * kT * 4;
constexpr int kSmem = oBar + 256 + 1024;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ptx::smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
                 : "memory");
}

// 32 consecutive q-values of key row r into a K-major SW128 pair of 64-column blocks.
__device__ __forceinline__ void store_row32(uint8_t* base, int r, int col0, const float (&v)[32]) {
    uint8_t* blk = base + (col0 / 64) * kTile + r * 128;
    const int chunk0 = (col0 % 64) / 8;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint4 w = make_uint4(ptx::pack_bf16x2(v[8 * q], v[8 * q + 1]), ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                                   ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]),
                                   ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
        *reinterpret_cast<uint4*>(blk + (((chunk0 + q) ^ (r & 7)) << 4)) = w;
    }
}

__device__ __forceinline__ void elem_bar(int id) {
    asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory");
}

template <bool kCausal>
__global__ void __launch_bounds__(640, 1)
    k_attn_bwd_tc(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                  const float* __restrict__ lse, const float* __restrict__ delta, bf16* __restrict__ dqkv,
                  float* __restrict__ dq_part, int seq, int heads) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + oBar);
    uint64_t* b_kv = bar + 0;
    uint64_t* b_qfull = bar + 1;   // [2]
    uint64_t* b_qempty = bar + 3;  // [2]
    uint64_t* b_sdp = bar + 5;     // S^T / dP^T of an iteration are in TMEM
    uint64_t* b_pds = bar + 6;     // 16 arrivals: P^T / dS^T written to SMEM
    uint64_t* b_mm2 = bar + 7;     // dV / dK / dQ MMAs of an iteration done
    uint64_t* b_dqfree = bar + 8;  // 16 arrivals: dQ TMEM read out
    uint64_t* b_sdfree = bar + 9;  // 16 arrivals: S^T / dP^T TMEM read into registers
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int bh = blockIdx.x, b = bh / heads, hd = bh % heads;
    const int j = blockIdx.y;                 // key tile
    const int nq = seq / kT;
    const int i0 = kCausal ? j : 0;
    const int iters = nq - i0;
    const int h = heads * kD;
    const int row0 = b * seq;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tm_qkv);
        ptx::tma_prefetch_desc(&tm_do);
        for (int q = 0; q < 10; ++q) ptx::mbar_init(&bar[q], (q == 6 || q == 8 || q == 9) ? 16 : 1);
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t tS = 0, tDP = 128, tDV = 256, tDK = 320, tDQ = 384;

    if (warp == 0) {
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(b_kv, 2 * kTile);
            ptx::tma_load_2d(smem + oK, &tm_qkv, b_kv, h + hd * kD, row0 + j * kT);
            ptx::tma_load_2d(smem + oV, &tm_qkv, b_kv, 2 * h + hd * kD, row0 + j * kT);
            for (int it = 0; it < iters; ++it) {
                const int buf = it & 1, i = i0 + it;
                if (it >= 2) ptx::mbar_wait(&b_qempty[buf], ((it - 2) >> 1) & 1);
                ptx::mbar_arrive_expect_tx(&b_qfull[buf], 2 * kTile + 2 * kT * 4);
                ptx::tma_load_2d(smem + oQ + buf * kTile, &tm_qkv, &b_qfull[buf], hd * kD, row0 + i * kT);
                ptx::tma_load_2d(smem + oDO + buf * kTile, &tm_do, &b_qfull[buf], hd * kD, row0 + i * kT);
                bulk_load(smem + oLse + buf * kT * 4, lse + static_cast<size_t>(bh) * seq + i * kT, kT * 4, &b_qfull[buf]);
                bulk_load(smem + oDel + buf * kT * 4, delta + static_cast<size_t>(bh) * seq + i * kT, kT * 4,
                          &b_qfull[buf]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t aK = ptx::smem_u32(smem + oK), aV = ptx::smem_u32(smem + oV);
            const uint32_t aPt = ptx::smem_u32(smem + oPt), aDSt = ptx::smem_u32(smem + oDSt);
            const uint32_t id_sq = ptx::idesc_bf16(128, 128, false, false);  // S^T, dP^T
            const uint32_t id_kv = ptx::idesc_bf16(128, 64, false, true);    // dV, dK: B MN-major
            const uint32_t id_q = ptx::idesc_bf16(128, 64, true, true);      // dQ: A and B MN-major
            auto issue_sdp = [&](int it) {
                const int buf = it & 1;
                const uint32_t aQ = ptx::smem_u32(smem + oQ + buf * kTile);
                const uint32_t aDO = ptx::smem_u32(smem + oDO + buf * kTile);
                ptx::mbar_wait(&b_qfull[buf], (it >> 1) & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) {
                    ptx::umma_bf16(tmem + tS, ptx::sdesc_sw128(aK + kk * 32, 16, 1024),
                                   ptx::sdesc_sw128(aQ + kk * 32, 16, 1024), id_sq, kk > 0);
                    ptx::umma_bf16(tmem + tDP, ptx::sdesc_sw128(aV + kk * 32, 16, 1024),
                                   ptx::sdesc_sw128(aDO + kk * 32, 16, 1024), id_sq, kk > 0);
                }
                ptx::umma_commit(b_sdp);
            };
            ptx::mbar_wait(b_kv, 0);
            issue_sdp(0);
            for (int it = 0; it < iters; ++it) {
                const int buf = it & 1;
                if (it + 1 < iters) {
                    // S^T / dP^T of the next query tile overlap this tile's P / dS math
                    ptx::mbar_wait(b_sdfree, it & 1);
                    ptx::tc_fence_after();
                    issue_sdp(it + 1);
                }
                const uint32_t aQ = ptx::smem_u32(smem + oQ + buf * kTile);
                const uint32_t aDO = ptx::smem_u32(smem + oDO + buf * kTile);
                ptx::mbar_wait(b_pds, it & 1);
                if (it > 0) ptx::mbar_wait(b_dqfree, (it - 1) & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < kT / 16; ++kk) {
                    const uint32_t a_off = (kk / 4) * kTile + (kk % 4) * 32;  // K-major, 16 q per step
                    const uint32_t b_off = kk * 2048;                         // MN-major, 16 rows per step
                    const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
                    ptx::umma_bf16(tmem + tDV, ptx::sdesc_sw128(aPt + a_off, 16, 1024),
                                   ptx::sdesc_sw128(aDO + b_off, 8192, 1024), id_kv, acc);
                    ptx::umma_bf16(tmem + tDK, ptx::sdesc_sw128(aDSt + a_off, 16, 1024),
                                   ptx::sdesc_sw128(aQ + b_off, 8192, 1024), id_kv, acc);
                    ptx::umma_bf16(tmem + tDQ, ptx::sdesc_sw128(aDSt + kk * 2048, kTile, 1024),
                                   ptx::sdesc_sw128(aK + kk * 2048, 8192, 1024), id_q, kk > 0);
                }
                ptx::umma_commit(b_mm2);
                ptx::umma_commit(&b_qempty[buf]);
            }
        }
    } else if (warp >= 4) {
        // 16 elementwise warps: 4 threads per key row, thread `sel` owns query columns
        // [32 sel, 32 sel + 32) of every 128-query tile and 16 of the 64 head dims.
        const int qw = warp & 3;
        const int sel = (warp - 4) >> 2;
        const int r = qw * 32 + lane;     // key row (S^T / dP^T / dV / dK) or query row (dQ)
        const int key = j * kT + r;
        const uint32_t trow = tmem + (static_cast<uint32_t>(qw * 32) << 16);
        const float sc = 0.125f * kLog2e;
        auto flush_dq = [&](int it) {  // dQ partial of query tile i0 + it: row r, dims 16 sel..+15
            const int i = i0 + it;
            float* dst = dq_part + (static_cast<size_t>(j) * (static_cast<size_t>(gridDim.x / heads) * seq) +
                                    static_cast<size_t>(row0 + i * kT + r)) * h + hd * kD + sel * 16;
            uint32_t v[16];
            ptx::tmem_ld_32x32b_x16(trow + tDQ + sel * 16, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 16; q += 4)
                *reinterpret_cast<float4*>(dst + q) = make_float4(__uint_as_float(v[q]), __uint_as_float(v[q + 1]),
                                                                  __uint_as_float(v[q + 2]), __uint_as_float(v[q + 3]));
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(b_dqfree);
        };
        for (int it = 0; it < iters; ++it) {
            const int buf = it & 1, i = i0 + it;
            ptx::mbar_wait(b_sdp, it & 1);
            ptx::tc_fence_after();
            uint32_t s[32], dp[32];
            ptx::tmem_ld_32x32b_x32(trow + tS + sel * 32, s);
            ptx::tmem_ld_32x32b_x32(trow + tDP + sel * 32, dp);
            ptx::tmem_ld_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(b_sdfree);  // the MMA may overwrite S^T / dP^T now
            ptx::mbar_wait(&b_qfull[buf], (it >> 1) & 1);
            if (it > 0) {
                ptx::mbar_wait(b_mm2, (it - 1) & 1);  // P^T / dS^T free, dQ of it-1 ready
                ptx::tc_fence_after();
                flush_dq(it - 1);
            }
            const float* sl = reinterpret_cast<const float*>(smem + oLse + buf * kT * 4);
            const float* sd = reinterpret_cast<const float*>(smem + oDel + buf * kT * 4);
            const int c = sel * 32;
            float p[32], ds[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const int qi = i * kT + c + q;  // absolute query index
                const bool vis = !kCausal || qi >= key;
                p[q] = vis ? ptx::ex2(fmaf(__uint_as_float(s[q]), sc, -sl[c + q] * kLog2e)) : 0.0f;
                ds[q] = p[q] * (__uint_as_float(dp[q]) - sd[c + q]);
            }
            store_row32(smem + oPt, r, c, p);
            store_row32(smem + oDSt, r, c, ds);
            ptx::fence_proxy_async();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(b_pds);
        }
        ptx::mbar_wait(b_mm2, (iters - 1) & 1);
        ptx::tc_fence_after();
        flush_dq(iters - 1);
        // dK (x 1/8) and dV for key row r, dims 16 sel..+15
        bf16* dk = dqkv + static_cast<size_t>(row0 + key) * 3 * h + h + hd * kD + sel * 16;
        bf16* dv = dk + h;
        {
            uint32_t vk[16], vv[16];
            ptx::tmem_ld_32x32b_x16(trow + tDK + sel * 16, vk);
            ptx::tmem_ld_32x32b_x16(trow + tDV + sel * 16, vv);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 16; q += 8) {
                uint32_t wk[4], wv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    wk[e] = ptx::pack_bf16x2(__uint_as_float(vk[q + 2 * e]) * 0.125f,
                                             __uint_as_float(vk[q + 2 * e + 1]) * 0.125f);
                    wv[e] = ptx::pack_bf16x2(__uint_as_float(vv[q + 2 * e]), __uint_as_float(vv[q + 2 * e + 1]));
                }
                *reinterpret_cast<uint4*>(dk + q) = make_uint4(wk[0], wk[1], wk[2], wk[3]);
                *reinterpret_cast<uint4*>(dv + q) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

// delta[bh, i] = sum_d dO[t, hd*64+d] * O[t, hd*64+d]; one thread per (token, head).
__global__ void k_attn_delta(const bf16* __restrict__ o, const bf16* __restrict__ dout, float* __restrict__ delta,
                             int tokens, int seq, int heads) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= tokens * heads) return;
    const int t = idx / heads, hd = idx % heads;
    const int h = heads * kD;
    const bf16* po = o + static_cast<size_t>(t) * h + hd * kD;
    const bf16* pd = dout + static_cast<size_t>(t) * h + hd * kD;
    float acc = 0.0f;
#pragma unroll
    for (int c = 0; c < kD; c += 8) {
        const uint4 a = *reinterpret_cast<const uint4*>(po + c);
        const uint4 d = *reinterpret_cast<const uint4*>(pd + c);
        const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, dw[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 fa = ptx::unpack_bf16x2(aw[e]), fd = ptx::unpack_bf16x2(dw[e]);
            acc = fmaf(fa.x, fd.x, fmaf(fa.y, fd.y, acc));
        }
    }
    const int b = t / seq, i = t % seq;
    delta[(static_cast<size_t>(b) * heads + hd) * seq + i] = acc;
}

// dq (bf16, x 1/8) = sum over key tiles j (<= query tile when causal) of dq_part[j].
__global__ void k_attn_dq_sum(const float* __restrict__ part, bf16* __restrict__ dqkv, int tokens, int seq, int heads,
                              int causal) {
    const int h = heads * kD;
    const size_t total = static_cast<size_t>(tokens) * h / 4;
    for (size_t v = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; v < total;
         v += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t e = v * 4;
        const int t = static_cast<int>(e / h), c = static_cast<int>(e % h);
        const int qt = (t % seq) / kT;
        const int nj = causal ? qt + 1 : seq / kT;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = 0; j < nj; ++j) {
            const float4 x = *reinterpret_cast<const float4*>(part + static_cast<size_t>(j) * tokens * h + e);
            acc.x += x.x;
            acc.y += x.y;
            acc.z += x.z;
            acc.w += x.w;
        }
        *reinterpret_cast<uint2*>(dqkv + static_cast<size_t>(t) * 3 * h + c) =
            make_uint2(ptx::pack_bf16x2(acc.x * 0.125f, acc.y * 0.125f), ptx::pack_bf16x2(acc.z * 0.125f, acc.w * 0.125f));
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
    check_cuda(cudaFuncSetAttribute(k_attn_bwd_tc<kCausal>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem),
               "cudaFuncSetAttribute(k_attn_bwd_tc)");
    done.fetch_or(bit);
}

}  // namespace

size_t attention_bwd_tc_scratch_floats(int batch, int seq, int heads) {
    return static_cast<size_t>(seq / kT) * batch * seq * heads * kD;
}

void attention_bwd_tc(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, bf16* dqkv, float* delta,
                      float* dq_part, int batch, int seq, int heads, bool causal, cudaStream_t s) {
    const int h = heads * kD;
    const int tokens = batch * seq;
    k_attn_delta<<<(tokens * heads + 255) / 256, 256, 0, s>>>(o, dout, delta, tokens, seq, heads);
    const CUtensorMap tq = make_tmap_bf16_2d(qkv, 3ull * h, static_cast<uint64_t>(tokens), 3ll * h, 64, kT);
    const CUtensorMap tdo = make_tmap_bf16_2d(dout, static_cast<uint64_t>(h), static_cast<uint64_t>(tokens), h, 64, kT);
    dim3 grid(batch * heads, seq / kT);
    if (causal) {
        set_smem_once<true>();
        k_attn_bwd_tc<true><<<grid, 640, kSmem, s>>>(tq, tdo, lse, delta, dqkv, dq_part, seq, heads);
    } else {
        set_smem_once<false>();
        k_attn_bwd_tc<false><<<grid, 640, kSmem, s>>>(tq, tdo, lse, delta, dqkv, dq_part, seq, heads);
    }
    const size_t vecs = static_cast<size_t>(tokens) * h / 4;
    k_attn_dq_sum<<<static_cast<int>(std::min<size_t>((vecs + 255) / 256, 148u * 32u)), 256, 0, s>>>(
        dq_part, dqkv, tokens, seq, heads, causal ? 1 : 0);
    check_cuda(cudaGetLastError(), "attention_bwd_tc");
}

}  // namespace p2bw
