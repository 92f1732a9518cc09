// Softmax attention backward on tcgen05 tensor cores (head dim 64 or 128, seq % 128 == 0).
// Persistent and key-outer: one CTA per SM walks work items
// (128-key tile j, sequence, head) -- (sequence, head)-major, see item_of -- and for each
// item the query tiles i that can see it:
//
//   UMMA  S^T  = K_j Q_i^T          128 x 128 fp32, TMEM [0, 128)
//   UMMA  dP^T = V_j dO_i^T         TMEM [128, 256)
//   SIMT  P^T  = exp(S^T/8 - lse_i), dS^T = P^T (dP^T - delta_i)   (16 warps, thread =
//         key row, warp = 32 query columns); P^T goes back into TMEM as packed
//         bf16 [448, 512), dS^T into SMEM in the UMMA K-major SW128 layout
//   UMMA  dV_j += P^T dO_i          TMEM [256, 320)   (A = P^T from TMEM, dO_i MN-major)
//   UMMA  dK_j += dS^T Q_i          TMEM [320, 384)   (Q_i read MN-major)
//   UMMA  dQ_i|j = dS K_j           TMEM [384, 448)   (dS^T and K_j read MN-major)
//   flush dQ_i|j: TMEM -> SMEM (SW128) -> TMA reduce-add into an fp32 dQ accumulator
//         (L2-resident, zeroed by the delta kernel; k_attn_dq_convert casts it)
//
// Warp roles (24 warps): 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4-19
// elementwise (four per TMEM lane quarter, 32 query columns each), 20-23 dQ flush +
// dK/dV epilogue of an item's last query tile.
// K/V (per item) are double-buffered and Q/dO/lse/delta (per query tile) triple-
// buffered, so TMA runs ahead across items; the S/dP MMAs of tile g+1 are issued before the dV/dK/dQ MMAs
// of tile g, so the exp work of g+1 overlaps them.  The same SMEM bytes serve as
// K-major and MN-major operands, so no transposes are materialised.
//
// The fp32 dQ reduce-add makes dQ's summation order over key tiles (<= 4 terms)
// run-dependent; everything else is deterministic.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "kernels.h"
#include "launch.h"
#include "profiler.h"
#include "ptx.cuh"
#include "tkernels.h"
#include "util.h"

namespace p2bw {

CUtensorMap make_tmap_bf16_2d(const bf16* ptr, uint64_t inner, uint64_t outer, int64_t ld_elems,
                              uint32_t box_inner, uint32_t box_outer);  // gemm.cu
CUtensorMap make_tmap_f32_2d(const float* ptr, uint64_t inner, uint64_t outer, int64_t ld_elems,
                             uint32_t box_inner, uint32_t box_outer);  // gemm.cu

namespace {

constexpr int kT = 128;  // tile rows (keys or queries)
constexpr int kD = 64;
constexpr int kTile = kT * 128;  // 16 KB: 128 rows of 64 bf16
constexpr int kQS = 3;                  // query-tile ring depth (covers the TMA latency)
constexpr int oK = 0;                   // [2] per item
constexpr int oV = oK + 2 * kTile;      // [2]
constexpr int oQ = oV + 2 * kTile;      // [kQS] per query tile
constexpr int oDO = oQ + kQS * kTile;   // [kQS]
constexpr int oDSt = oDO + kQS * kTile; // 2 blocks of 64 queries
constexpr int oDQ = oDSt + 2 * kTile;   // 4 flush warps x 32 rows x 128 B
constexpr int oLse = oDQ + 4 * 4096;    // [kQS][128] f32
constexpr int oDel = oLse + kQS * kT * 4; // [kQS][128] f32
constexpr int oBar = oDel + kQS * kT * 4;
constexpr int kSmem = oBar + 256 + 1024;
constexpr int kElemWarps = 16;  // four per TMEM lane quarter, 32 query columns each
constexpr int kThreads = 128 + 32 * kElemWarps + 128;  // roles + elementwise + dQ flush
constexpr float kLog2e = 1.4426950408889634f;
// dQ leaves TMEM by red.global.add.v4.f32 from registers (true) or through SMEM and a
// TMA reduce-add (false).  Measured: the per-row 16-byte L2 reductions made the flush
// 70% slower (93 -> 108 us per call), so the bulk reduce-add stays.
constexpr bool kDqRed = false;

// barrier indices
// S^T and dP^T are released separately (bSFree / bDpFree) as soon as the elementwise
// warps have them in registers, so the next tile's S^T / dP^T MMAs overlap the exp work.
constexpr int bKvFull = 0, bKvEmpty = 2, bQFull = 4, bQEmpty = 4 + kQS, bSdpFull = 4 + 2 * kQS,
              bSFree = bSdpFull + 1, bPdsFull = bSdpFull + 2, bMm2 = bSdpFull + 3, bDqFree = bSdpFull + 4,
              bKvAccFree = bSdpFull + 5, bDpFree = bSdpFull + 6, kNumBars = bSdpFull + 7;
// P^T lives in TMEM as bf16 (two per 32-bit column) and feeds dV = P^T dO as the
// tcgen05 A operand straight from TMEM.
constexpr uint32_t tS = 0, tDP = 128, tDV = 256, tDK = 320, tDQ = 384, tPT = 448;

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
                 : "memory");
}

// Phase timestamps (debug; null in production): p2bw_debug_attention_timing.  Per CTA
// 64 u64 slots: [0..7] elem warp 4 "S/dP seen" for g = 0..7, [8..15] its "computed",
// [16..23] its "mm2(g-1) seen", [24..31] its "pds arrived", [32..39] MMA "S/dP issued",
// [40..47] MMA "mm2 issued", [48..55] flush "mm2 seen", [56..63] flush "dq free".
__device__ unsigned long long* g_attn_bwd_dbg = nullptr;

__device__ __forceinline__ void bmark(bool on, int slot, int g) {
    if (on && g < 8) g_attn_bwd_dbg[blockIdx.x * 64 + slot * 8 + g] = clock64();
}

struct Item {
    int bh, j, i0, iters;
};

// Item order: (sequence, head)-major -- the nq key tiles of one (sequence, head) are
// consecutive items, so the CTAs running them at the same time share its Q / dO / lse /
// delta tiles and its dQ accumulator rows in L2 (the former key-tile-major order re-read
// them from DRAM for every key tile; in the GPT-2.2B step +0.4%, paired runs).  Causal
// items differ in length (nq - j query tiles); j is rotated by the (sequence, head) index
// so that the static round-robin hands every CTA a mix of lengths (with nq | #CTAs an
// unrotated order would give CTA b only j = b % nq).
__device__ __forceinline__ Item item_of(int n, int bhn, int nq, bool causal) {
    (void)bhn;
    Item it;
    it.bh = n / nq;
    const int r = n % nq;
    it.j = causal ? (r + it.bh) % nq : r;
    it.i0 = causal ? it.j : 0;
    it.iters = nq - it.i0;
    return it;
}

template <bool kCausal>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_bwd_tc(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                  const __grid_constant__ CUtensorMap tm_dq, const float* __restrict__ nl2,
                  const float* __restrict__ delta, bf16* __restrict__ dqkv, float* __restrict__ dq_acc, int seq,
                  int heads, int bhn, float4* __restrict__ zero_next, long long zero_n4) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = ptx::smem_u32(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + oBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + kNumBars);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nq = seq / kT;
    const int items = bhn * nq;
    const int h = heads * kD;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tm_qkv);
        ptx::tma_prefetch_desc(&tm_do);
        ptx::tma_prefetch_desc(&tm_dq);
        for (int q = 0; q < kNumBars; ++q) {
            const uint32_t cnt =
                (q == bSFree || q == bDpFree || q == bPdsFull) ? kElemWarps : (q == bDqFree || q == bKvAccFree) ? 4 : 1;
            ptx::mbar_init(&bar[q], cnt);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::pdl_trigger();
    ptx::pdl_wait();

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            int ln = 0, g = 0;
            for (int n = blockIdx.x; n < items; n += gridDim.x, ++ln) {
                const Item it = item_of(n, bhn, nq, kCausal);
                const int b = it.bh / heads, hd = it.bh % heads, row0 = b * seq;
                const int kb = ln & 1;
                ptx::mbar_wait(&bar[bKvEmpty + kb], ((ln >> 1) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&bar[bKvFull + kb], 2 * kTile);
                ptx::tma_load_2d(smem + oK + kb * kTile, &tm_qkv, &bar[bKvFull + kb], h + hd * kD, row0 + it.j * kT);
                ptx::tma_load_2d(smem + oV + kb * kTile, &tm_qkv, &bar[bKvFull + kb], 2 * h + hd * kD,
                                 row0 + it.j * kT);
                for (int t = 0; t < it.iters; ++t, ++g) {
                    const int i = it.i0 + t, qb = g % kQS;
                    ptx::mbar_wait(&bar[bQEmpty + qb], ((g / kQS) & 1) ^ 1);
                    uint64_t* full = &bar[bQFull + qb];
                    ptx::mbar_arrive_expect_tx(full, 2 * kTile + 2 * kT * 4);
                    ptx::tma_load_2d(smem + oQ + qb * kTile, &tm_qkv, full, hd * kD, row0 + i * kT);
                    ptx::tma_load_2d(smem + oDO + qb * kTile, &tm_do, full, hd * kD, row0 + i * kT);
                    const size_t so = static_cast<size_t>(it.bh) * seq + i * kT;
                    bulk_load(sbase + oLse + qb * kT * 4, nl2 + so, kT * 4, full);
                    bulk_load(sbase + oDel + qb * kT * 4, delta + so, kT * 4, full);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            const uint32_t aDSt = sbase + oDSt;
            constexpr uint32_t id_sq = ptx::idesc_bf16(128, 128, false, false);  // S^T, dP^T
            constexpr uint32_t id_kv = ptx::idesc_bf16(128, 64, false, true);    // dV, dK: B MN-major
            constexpr uint32_t id_q = ptx::idesc_bf16(128, 64, true, true);      // dQ: A and B MN-major
            struct Pend {
                int g, ln, kb;
                bool first, last;
            };
            auto issue_mm2 = [&](const Pend& p) {
                const int qb = p.g % kQS;
                const uint32_t aQ = sbase + oQ + qb * kTile, aDO = sbase + oDO + qb * kTile;
                const uint32_t aK = sbase + oK + p.kb * kTile;
                ptx::mbar_wait(&bar[bPdsFull], p.g & 1);
                if (p.g > 0) ptx::mbar_wait(&bar[bDqFree], (p.g - 1) & 1);
                if (p.first && p.ln > 0) ptx::mbar_wait(&bar[bKvAccFree], (p.ln - 1) & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < kT / 16; ++kk) {
                    const uint32_t a_off = (kk / 4) * kTile + (kk % 4) * 32;  // K-major, 16 q per step
                    const uint32_t b_off = kk * 2048;                         // MN-major, 16 rows per step
                    const uint32_t acc = (!p.first || kk > 0) ? 1u : 0u;
                    ptx::umma_bf16_ts(tmem + tDV, tmem + tPT + kk * 8, ptx::sdesc_sw128(aDO + b_off, 8192, 1024),
                                      id_kv, acc);
                    ptx::umma_bf16(tmem + tDK, ptx::sdesc_sw128(aDSt + a_off, 16, 1024),
                                   ptx::sdesc_sw128(aQ + b_off, 8192, 1024), id_kv, acc);
                    ptx::umma_bf16(tmem + tDQ, ptx::sdesc_sw128(aDSt + kk * 2048, kTile, 1024),
                                   ptx::sdesc_sw128(aK + kk * 2048, 8192, 1024), id_q, kk > 0 ? 1u : 0u);
                }
                ptx::umma_commit(&bar[bMm2]);
                bmark(g_attn_bwd_dbg != nullptr, 5, p.g);
                ptx::umma_commit(&bar[bQEmpty + qb]);
                if (p.last) ptx::umma_commit(&bar[bKvEmpty + p.kb]);
            };
            Pend prev{};
            bool have = false;
            int ln = 0, g = 0;
            for (int n = blockIdx.x; n < items; n += gridDim.x, ++ln) {
                const Item it = item_of(n, bhn, nq, kCausal);
                const int kb = ln & 1;
                const uint32_t aK = sbase + oK + kb * kTile, aV = sbase + oV + kb * kTile;
                ptx::mbar_wait(&bar[bKvFull + kb], (ln >> 1) & 1);
                for (int t = 0; t < it.iters; ++t, ++g) {
                    const int qb = g % kQS;
                    const uint32_t aQ = sbase + oQ + qb * kTile, aDO = sbase + oDO + qb * kTile;
                    ptx::mbar_wait(&bar[bQFull + qb], (g / kQS) & 1);
                    if (g > 0) ptx::mbar_wait(&bar[bSFree], (g - 1) & 1);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < kD / 16; ++kk)
                        ptx::umma_bf16(tmem + tS, ptx::sdesc_sw128(aK + kk * 32, 16, 1024),
                                       ptx::sdesc_sw128(aQ + kk * 32, 16, 1024), id_sq, kk > 0);
                    if (g > 0) ptx::mbar_wait(&bar[bDpFree], (g - 1) & 1);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < kD / 16; ++kk)
                        ptx::umma_bf16(tmem + tDP, ptx::sdesc_sw128(aV + kk * 32, 16, 1024),
                                       ptx::sdesc_sw128(aDO + kk * 32, 16, 1024), id_sq, kk > 0);
                    ptx::umma_commit(&bar[bSdpFull]);
                    bmark(g_attn_bwd_dbg != nullptr, 4, g);
                    if (have) issue_mm2(prev);
                    prev = Pend{g, ln, kb, t == 0, t == it.iters - 1};
                    have = true;
                }
            }
            if (have) issue_mm2(prev);
        }
    } else if (warp == 3) {
        // idle role warp: zero the NEXT call's dQ accumulator (double-buffered per stage,
        // attention_bwd_tc), which takes the zero-fill off the delta kernel on the stage
        // stream's critical path; plain 512 B-per-instruction stores, drained at exit
        if (zero_next != nullptr) {
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            for (long long i = static_cast<long long>(blockIdx.x) * 32 + lane; i < zero_n4;
                 i += static_cast<long long>(gridDim.x) * 32)
                zero_next[i] = z;
        }
    } else if (warp >= 4 && warp < 4 + kElemWarps) {
        // ---------------- elementwise: P^T, dS^T ----------------
        const int qw = warp & 3;
        const int sel = (warp - 4) >> 2;  // query columns [32 sel, 32 sel + 32): UMMA block sel / 2
        const int r = qw * 32 + lane;     // key row within the tile
        const uint32_t trow = tmem + (static_cast<uint32_t>(qw * 32) << 16);
        const float sc = 0.125f * kLog2e;
        const uint32_t drow = sbase + oDSt + (sel >> 1) * kTile + r * 128;  // + 64 B for odd sel
        const bool dbg = g_attn_bwd_dbg != nullptr && warp == 4 && lane == 0;
        int g = 0;
        for (int n = blockIdx.x; n < items; n += gridDim.x) {
            const Item it = item_of(n, bhn, nq, kCausal);
            const int key = it.j * kT + r;
            for (int t = 0; t < it.iters; ++t, ++g) {
                const int i = it.i0 + t, qb = g % kQS;
                ptx::mbar_wait(&bar[bSdpFull], g & 1);
                bmark(dbg, 0, g);
                ptx::mbar_wait(&bar[bQFull + qb], (g / kQS) & 1);  // lse / delta visible
                ptx::tc_fence_after();
                uint32_t pp[16], dd[16];  // bf16x2: 32 P^T and 32 dS^T values of row r
#pragma unroll
                for (int c = 0; c < 2; ++c) {  // 16 query columns per TMEM load (register budget)
                    const int col0 = sel * 32 + c * 16;
                    uint32_t sv[16], dv[16];
                    ptx::tmem_ld_32x32b_x16(trow + tS + col0, sv);
                    ptx::tmem_ld_32x32b_x16(trow + tDP + col0, dv);
                    ptx::tmem_ld_wait();
                    const uint32_t la = sbase + oLse + qb * kT * 4 + col0 * 4;  // -lse log2(e)
                    const uint32_t da = sbase + oDel + qb * kT * 4 + col0 * 4;
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 l4 = ptx::lds_f4(la + q4 * 16);
                        const float4 d4 = ptx::lds_f4(da + q4 * 16);
                        const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dl[4] = {d4.x, d4.y, d4.z, d4.w};
                        float p[4], ds[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int q = q4 * 4 + e;
                            float x = ptx::ex2(fmaf(__uint_as_float(sv[q]), sc, lv[e]));
                            if (kCausal && i * kT + col0 + q < key) x = 0.0f;
                            p[e] = x;
                            ds[e] = x * (__uint_as_float(dv[q]) - dl[e]);
                        }
                        pp[c * 8 + q4 * 2] = ptx::pack_bf16x2(p[0], p[1]);
                        pp[c * 8 + q4 * 2 + 1] = ptx::pack_bf16x2(p[2], p[3]);
                        dd[c * 8 + q4 * 2] = ptx::pack_bf16x2(ds[0], ds[1]);
                        dd[c * 8 + q4 * 2 + 1] = ptx::pack_bf16x2(ds[2], ds[3]);
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {  // S^T / dP^T may be overwritten by the next tile's MMAs
                    ptx::mbar_arrive(&bar[bSFree]);
                    ptx::mbar_arrive(&bar[bDpFree]);
                }
                bmark(dbg, 1, g);
                if (g > 0) ptx::mbar_wait(&bar[bMm2], (g - 1) & 1);  // P^T / dS^T buffers free
                bmark(dbg, 2, g);
                ptx::tc_fence_after();
                ptx::tmem_st_32x32b_x16(trow + tPT + sel * 16, pp);  // queries 32 sel .. +31 of key row r
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    const int cc = (sel & 1) * 4 + ch;  // 16-byte chunk of the 128-byte row
                    const uint32_t off = static_cast<uint32_t>((cc ^ (r & 7)) << 4);
                    ptx::sts_u4(drow + off, dd[4 * ch], dd[4 * ch + 1], dd[4 * ch + 2], dd[4 * ch + 3]);
                }
                ptx::tmem_st_wait();
                ptx::fence_proxy_async();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&bar[bPdsFull]);
                bmark(dbg, 3, g);
            }
        }
    } else if (warp >= 4 + kElemWarps) {
        // ---------------- dQ flush (TMA reduce-add) + dK / dV epilogue ----------------
        const int qw = warp & 3;
        const uint32_t trow = tmem + (static_cast<uint32_t>(qw * 32) << 16);
        uint8_t* stage = smem + oDQ + qw * 4096;
        const uint32_t sstage = ptx::smem_u32(stage);
        const bool fdbg = g_attn_bwd_dbg != nullptr && warp == 4 + kElemWarps && lane == 0;
        int g = 0;
        for (int n = blockIdx.x; n < items; n += gridDim.x) {
            const Item it = item_of(n, bhn, nq, kCausal);
            const int b = it.bh / heads, hd = it.bh % heads, row0 = b * seq;
            for (int t = 0; t < it.iters; ++t, ++g) {
                const int i = it.i0 + t;
                ptx::mbar_wait(&bar[bMm2], g & 1);
                bmark(fdbg, 6, g);
                ptx::tc_fence_after();
#pragma unroll 1
                for (int half = 0; half < 2; ++half) {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(trow + tDQ + half * 32, v);
                    ptx::tmem_ld_wait();
                    if (half == 1) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(&bar[bDqFree]);
                        bmark(fdbg, 7, g);
                    }
                    if constexpr (kDqRed) {
                        // straight from registers: 16-byte fp32 reductions into L2 (no SMEM traffic)
                        float* dst = dq_acc + static_cast<size_t>(row0 + i * kT + qw * 32 + lane) * h + hd * kD +
                                     half * 32;
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * c),
                                         "f"(__uint_as_float(v[4 * c])), "f"(__uint_as_float(v[4 * c + 1])),
                                         "f"(__uint_as_float(v[4 * c + 2])), "f"(__uint_as_float(v[4 * c + 3]))
                                         : "memory");
                    } else {
                        if (lane == 0) ptx::bulk_wait_read<0>();  // staging buffer read out by the last reduce
                        __syncwarp();
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            ptx::sts_f4(sstage + ptx::swz128(lane, c), __uint_as_float(v[4 * c]),
                                        __uint_as_float(v[4 * c + 1]), __uint_as_float(v[4 * c + 2]),
                                        __uint_as_float(v[4 * c + 3]));
                        ptx::fence_proxy_async();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_reduce_add_2d(&tm_dq, stage, hd * kD + half * 32, row0 + i * kT + qw * 32);
                            ptx::bulk_commit();
                        }
                    }
                }
                if (t == it.iters - 1) {
                    // dK (x 1/8) and dV of key row qw*32 + lane of tile j
                    const int key = it.j * kT + qw * 32 + lane;
                    bf16* dk = dqkv + static_cast<size_t>(row0 + key) * 3 * h + h + hd * kD;
                    bf16* dv = dk + h;
#pragma unroll 1
                    for (int half = 0; half < 2; ++half) {
                        uint32_t vk[32], vv[32];
                        ptx::tmem_ld_32x32b_x32(trow + tDK + half * 32, vk);
                        ptx::tmem_ld_32x32b_x32(trow + tDV + half * 32, vv);
                        ptx::tmem_ld_wait();
                        if (half == 1) {
                            ptx::tc_fence_before();
                            __syncwarp();
                            if (lane == 0) ptx::mbar_arrive(&bar[bKvAccFree]);
                        }
#pragma unroll
                        for (int q = 0; q < 32; q += 8) {
                            uint32_t wk[4], wv[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                wk[e] = ptx::pack_bf16x2(__uint_as_float(vk[q + 2 * e]) * 0.125f,
                                                         __uint_as_float(vk[q + 2 * e + 1]) * 0.125f);
                                wv[e] = ptx::pack_bf16x2(__uint_as_float(vv[q + 2 * e]),
                                                         __uint_as_float(vv[q + 2 * e + 1]));
                            }
                            *reinterpret_cast<uint4*>(dk + half * 32 + q) = make_uint4(wk[0], wk[1], wk[2], wk[3]);
                            *reinterpret_cast<uint4*>(dv + half * 32 + q) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                        }
                    }
                }
            }
        }
        if (lane == 0) ptx::bulk_wait<0>();
        __syncwarp();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

// ---- head dim 128 -----------------------------------------------------------------
//
// The same key-outer item walk and operand tricks at D = 128, where the accumulators
// alone fill TMEM: S^T [0, 128), dP^T [128, 256), dV [256, 384), dK [384, 512).  So
//   * P^T goes to SMEM (K-major SW128, like dS^T) instead of TMEM, and
//   * dQ_i|j = dS K_j reuses the S^T columns once the elementwise warps have read S^T:
//     the next tile's S^T / dP^T wait for the dQ flush (no S/dP-ahead-of-mm2 overlap);
//   * instead the tile is split in two phases: S^T is committed alone, so the exponentials
//     (P^T -> SMEM) run while dP^T computes, and dV = P^T dO runs while dS^T is formed
//     (GPT-2.2B shape 184 -> 167 us).  The same split measured neutral at D = 64, whose
//     next-tile S / dP already overlap the dV / dK / dQ MMAs.
// SMEM: K, V (one item) and Q, dO (one query tile) of 32 KB each, P^T and dS^T 32 KB,
// dQ staging 16 KB: ~209 KB.  Numerics as at D = 64 (scale 1 / sqrt(128)).
namespace d128 {
constexpr int kD = 128;
constexpr int kTileD = 2 * kTile;  // 128 rows x 128 bf16: two 64-column boxes kTile apart
constexpr int oK = 0, oV = oK + kTileD, oQ = oV + kTileD, oDO = oQ + kTileD, oPT = oDO + kTileD,
              oDSt = oPT + kTileD, oDQ = oDSt + kTileD, oLse = oDQ + 4 * 4096, oDel = oLse + kT * 4,
              oBar = oDel + kT * 4;
constexpr int bKvFull = 0, bKvEmpty = 1, bQFull = 2, bQEmpty = 3, bSFull = 4, bPFull = 5, bMm2 = 6,
              bDqFree = 7, bKvAccFree = 8, bDpFull = 9, bDsFull = 10, kNumBars = 11;
constexpr int kSmem = oBar + 256 + 1024;
static_assert(kSmem <= 227 * 1024, "D = 128 backward SMEM");
constexpr uint32_t tS = 0, tDP = 128, tDV = 256, tDK = 384, tDQ = 0;
constexpr float kScale = 0.08838834764831845f;  // 1 / sqrt(128)
}  // namespace d128

template <bool kCausal>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_bwd_tc128(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                     const __grid_constant__ CUtensorMap tm_dq, const float* __restrict__ nl2,
                     const float* __restrict__ delta, bf16* __restrict__ dqkv, int seq, int heads, int bhn,
                     float4* __restrict__ zero_next, long long zero_n4) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = ptx::smem_u32(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + d128::oBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + d128::kNumBars);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nq = seq / kT;
    const int items = bhn * nq;
    const int h = heads * d128::kD;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tm_qkv);
        ptx::tma_prefetch_desc(&tm_do);
        ptx::tma_prefetch_desc(&tm_dq);
        for (int q = 0; q < d128::kNumBars; ++q)
            ptx::mbar_init(&bar[q], (q == d128::bPFull || q == d128::bDsFull) ? kElemWarps
                                    : (q == d128::bDqFree || q == d128::bKvAccFree) ? 4 : 1);
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::pdl_trigger();
    ptx::pdl_wait();

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            int ln = 0, g = 0;
            for (int n = blockIdx.x; n < items; n += gridDim.x, ++ln) {
                const Item it = item_of(n, bhn, nq, kCausal);
                const int b = it.bh / heads, hd = it.bh % heads, row0 = b * seq;
                ptx::mbar_wait(&bar[d128::bKvEmpty], (ln & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&bar[d128::bKvFull], 2 * d128::kTileD);
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    ptx::tma_load_2d(smem + d128::oK + x * kTile, &tm_qkv, &bar[d128::bKvFull], h + hd * d128::kD + 64 * x,
                                     row0 + it.j * kT);
                    ptx::tma_load_2d(smem + d128::oV + x * kTile, &tm_qkv, &bar[d128::bKvFull], 2 * h + hd * d128::kD + 64 * x,
                                     row0 + it.j * kT);
                }
                for (int t = 0; t < it.iters; ++t, ++g) {
                    const int i = it.i0 + t;
                    ptx::mbar_wait(&bar[d128::bQEmpty], (g & 1) ^ 1);
                    uint64_t* full = &bar[d128::bQFull];
                    ptx::mbar_arrive_expect_tx(full, 2 * d128::kTileD + 2 * kT * 4);
#pragma unroll
                    for (int x = 0; x < 2; ++x) {
                        ptx::tma_load_2d(smem + d128::oQ + x * kTile, &tm_qkv, full, hd * d128::kD + 64 * x, row0 + i * kT);
                        ptx::tma_load_2d(smem + d128::oDO + x * kTile, &tm_do, full, hd * d128::kD + 64 * x, row0 + i * kT);
                    }
                    const size_t so = static_cast<size_t>(it.bh) * seq + i * kT;
                    bulk_load(sbase + d128::oLse, nl2 + so, kT * 4, full);
                    bulk_load(sbase + d128::oDel, delta + so, kT * 4, full);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t id_sq = ptx::idesc_bf16(128, 128, false, false);  // S^T, dP^T (K = d)
            constexpr uint32_t id_kv = ptx::idesc_bf16(128, 128, false, true);   // dV, dK: B MN-major
            constexpr uint32_t id_q = ptx::idesc_bf16(128, 128, true, true);     // dQ: A and B MN-major
            const uint32_t aK = sbase + d128::oK, aV = sbase + d128::oV, aQ = sbase + d128::oQ, aDO = sbase + d128::oDO;
            const uint32_t aPT = sbase + d128::oPT, aDSt = sbase + d128::oDSt;
            int ln = 0, g = 0;
            for (int n = blockIdx.x; n < items; n += gridDim.x, ++ln) {
                const Item it = item_of(n, bhn, nq, kCausal);
                ptx::mbar_wait(&bar[d128::bKvFull], ln & 1);
                for (int t = 0; t < it.iters; ++t, ++g) {
                    ptx::mbar_wait(&bar[d128::bQFull], g & 1);
                    if (g > 0) ptx::mbar_wait(&bar[d128::bDqFree], (g - 1) & 1);  // S^T columns (dQ) flushed
                    ptx::tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < d128::kD / 16; ++kk) {
                        const uint32_t off = (kk / 4) * kTile + (kk % 4) * 32;  // K-major over d
                        ptx::umma_bf16(tmem + d128::tS, ptx::sdesc_sw128(aK + off, 16, 1024),
                                       ptx::sdesc_sw128(aQ + off, 16, 1024), id_sq, kk > 0);
                    }
                    ptx::umma_commit(&bar[d128::bSFull]);  // the exponentials start while dP^T runs
#pragma unroll
                    for (int kk = 0; kk < d128::kD / 16; ++kk) {
                        const uint32_t off = (kk / 4) * kTile + (kk % 4) * 32;
                        ptx::umma_bf16(tmem + d128::tDP, ptx::sdesc_sw128(aV + off, 16, 1024),
                                       ptx::sdesc_sw128(aDO + off, 16, 1024), id_sq, kk > 0);
                    }
                    ptx::umma_commit(&bar[d128::bDpFull]);
                    const bool first = t == 0;
                    ptx::mbar_wait(&bar[d128::bPFull], g & 1);
                    if (first && ln > 0) ptx::mbar_wait(&bar[d128::bKvAccFree], (ln - 1) & 1);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < kT / 16; ++kk)  // dV = P^T dO runs while dS^T is computed
                        ptx::umma_bf16(tmem + d128::tDV, ptx::sdesc_sw128(aPT + (kk / 4) * kTile + (kk % 4) * 32, 16, 1024),
                                       ptx::sdesc_sw128(aDO + kk * 2048, kTile, 1024), id_kv,
                                       (!first || kk > 0) ? 1u : 0u);
                    ptx::mbar_wait(&bar[d128::bDsFull], g & 1);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < kT / 16; ++kk) {
                        const uint32_t a_off = (kk / 4) * kTile + (kk % 4) * 32;  // K-major, 16 queries per step
                        const uint32_t b_off = kk * 2048;                         // MN-major, 16 rows per step
                        ptx::umma_bf16(tmem + d128::tDK, ptx::sdesc_sw128(aDSt + a_off, 16, 1024),
                                       ptx::sdesc_sw128(aQ + b_off, kTile, 1024), id_kv, (!first || kk > 0) ? 1u : 0u);
                        ptx::umma_bf16(tmem + d128::tDQ, ptx::sdesc_sw128(aDSt + b_off, kTile, 1024),
                                       ptx::sdesc_sw128(aK + b_off, kTile, 1024), id_q, kk > 0 ? 1u : 0u);
                    }
                    ptx::umma_commit(&bar[d128::bMm2]);
                    ptx::umma_commit(&bar[d128::bQEmpty]);
                    if (t == it.iters - 1) ptx::umma_commit(&bar[d128::bKvEmpty]);
                }
            }
        }
    } else if (warp == 3) {
        // idle role warp: zero the NEXT call's dQ accumulator (double-buffered per stage,
        // attention_bwd_tc), which takes the zero-fill off the delta kernel on the stage
        // stream's critical path; plain 512 B-per-instruction stores, drained at exit
        if (zero_next != nullptr) {
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            for (long long i = static_cast<long long>(blockIdx.x) * 32 + lane; i < zero_n4;
                 i += static_cast<long long>(gridDim.x) * 32)
                zero_next[i] = z;
        }
    } else if (warp >= 4 && warp < 4 + kElemWarps) {
        // ---------------- elementwise: P^T, dS^T -> SMEM ----------------
        const int qw = warp & 3;
        const int sel = (warp - 4) >> 2;  // query columns [32 sel, 32 sel + 32)
        const int r = qw * 32 + lane;     // key row within the tile
        const uint32_t trow = tmem + (static_cast<uint32_t>(qw * 32) << 16);
        const float sc = d128::kScale * kLog2e;
        const uint32_t prow = sbase + d128::oPT + (sel >> 1) * kTile + r * 128;
        const uint32_t drow = sbase + d128::oDSt + (sel >> 1) * kTile + r * 128;
        int g = 0;
        for (int n = blockIdx.x; n < items; n += gridDim.x) {
            const Item it = item_of(n, bhn, nq, kCausal);
            const int key = it.j * kT + r;
            for (int t = 0; t < it.iters; ++t, ++g) {
                const int i = it.i0 + t;
                ptx::mbar_wait(&bar[d128::bSFull], g & 1);
                ptx::mbar_wait(&bar[d128::bQFull], g & 1);  // lse / delta visible
                ptx::tc_fence_after();
                // phase 1 (S^T only): P^T -> SMEM, so dV starts while dP^T is still computing
                float pf[32];
                uint32_t pk[16];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int col0 = sel * 32 + c * 16;
                    uint32_t sv[16];
                    ptx::tmem_ld_32x32b_x16(trow + d128::tS + col0, sv);
                    ptx::tmem_ld_wait();
                    const uint32_t la = sbase + d128::oLse + col0 * 4;
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 l4 = ptx::lds_f4(la + q4 * 16);
                        const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int q = q4 * 4 + e;
                            float x = ptx::ex2(fmaf(__uint_as_float(sv[q]), sc, lv[e]));
                            if (kCausal && i * kT + col0 + q < key) x = 0.0f;
                            pf[c * 16 + q] = x;
                        }
                        pk[c * 8 + q4 * 2] = ptx::pack_bf16x2(pf[c * 16 + q4 * 4], pf[c * 16 + q4 * 4 + 1]);
                        pk[c * 8 + q4 * 2 + 1] = ptx::pack_bf16x2(pf[c * 16 + q4 * 4 + 2], pf[c * 16 + q4 * 4 + 3]);
                    }
                }
                if (g > 0) ptx::mbar_wait(&bar[d128::bMm2], (g - 1) & 1);  // P^T / dS^T buffers free
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    const int cc = (sel & 1) * 4 + ch;  // 16-byte chunk of the 128-byte row
                    const uint32_t off = static_cast<uint32_t>((cc ^ (r & 7)) << 4);
                    ptx::sts_u4(prow + off, pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
                }
                ptx::fence_proxy_async();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&bar[d128::bPFull]);
                // phase 2: dS^T = P^T (dP^T - delta) -> SMEM
                ptx::mbar_wait(&bar[d128::bDpFull], g & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int col0 = sel * 32 + c * 16;
                    uint32_t dv[16];
                    ptx::tmem_ld_32x32b_x16(trow + d128::tDP + col0, dv);
                    ptx::tmem_ld_wait();
                    const uint32_t da = sbase + d128::oDel + col0 * 4;
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 d4 = ptx::lds_f4(da + q4 * 16);
                        const float dl[4] = {d4.x, d4.y, d4.z, d4.w};
                        float ds[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            ds[e] = pf[c * 16 + q4 * 4 + e] * (__uint_as_float(dv[q4 * 4 + e]) - dl[e]);
                        pk[c * 8 + q4 * 2] = ptx::pack_bf16x2(ds[0], ds[1]);
                        pk[c * 8 + q4 * 2 + 1] = ptx::pack_bf16x2(ds[2], ds[3]);
                    }
                }
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    const int cc = (sel & 1) * 4 + ch;
                    const uint32_t off = static_cast<uint32_t>((cc ^ (r & 7)) << 4);
                    ptx::sts_u4(drow + off, pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
                }
                ptx::fence_proxy_async();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&bar[d128::bDsFull]);
            }
        }
    } else if (warp >= 4 + kElemWarps) {
        // ---------------- dQ flush (TMA reduce-add) + dK / dV epilogue ----------------
        const int qw = warp & 3;
        const uint32_t trow = tmem + (static_cast<uint32_t>(qw * 32) << 16);
        uint8_t* stage = smem + d128::oDQ + qw * 4096;
        const uint32_t sstage = ptx::smem_u32(stage);
        int g = 0;
        for (int n = blockIdx.x; n < items; n += gridDim.x) {
            const Item it = item_of(n, bhn, nq, kCausal);
            const int b = it.bh / heads, hd = it.bh % heads, row0 = b * seq;
            for (int t = 0; t < it.iters; ++t, ++g) {
                const int i = it.i0 + t;
                ptx::mbar_wait(&bar[d128::bMm2], g & 1);
                ptx::tc_fence_after();
#pragma unroll 1
                for (int q = 0; q < 4; ++q) {  // 32 columns at a time (768 threads: ~80 registers each)
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(trow + d128::tDQ + q * 32, v);
                    ptx::tmem_ld_wait();
                    if (q == 3) {  // the S^T columns may take the next tile's S^T
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(&bar[d128::bDqFree]);
                    }
                    if (lane == 0) ptx::bulk_wait_read<0>();  // staging buffer read out by the last reduce
                    __syncwarp();
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        ptx::sts_f4(sstage + ptx::swz128(lane, c), __uint_as_float(v[4 * c]),
                                    __uint_as_float(v[4 * c + 1]), __uint_as_float(v[4 * c + 2]),
                                    __uint_as_float(v[4 * c + 3]));
                    ptx::fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_reduce_add_2d(&tm_dq, stage, hd * d128::kD + q * 32, row0 + i * kT + qw * 32);
                        ptx::bulk_commit();
                    }
                }
                if (t == it.iters - 1) {
                    // dK (x 1/sqrt(128)) and dV of key row qw*32 + lane of tile j
                    const int key = it.j * kT + qw * 32 + lane;
                    bf16* dk = dqkv + static_cast<size_t>(row0 + key) * 3 * h + h + hd * d128::kD;
                    bf16* dv = dk + h;
#pragma unroll 1
                    for (int q = 0; q < 4; ++q) {
                        uint32_t vk[32], vv[32];
                        ptx::tmem_ld_32x32b_x32(trow + d128::tDK + q * 32, vk);
                        ptx::tmem_ld_32x32b_x32(trow + d128::tDV + q * 32, vv);
                        ptx::tmem_ld_wait();
                        if (q == 3) {
                            ptx::tc_fence_before();
                            __syncwarp();
                            if (lane == 0) ptx::mbar_arrive(&bar[d128::bKvAccFree]);
                        }
#pragma unroll
                        for (int c = 0; c < 32; c += 8) {
                            uint32_t wk[4], wv[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                wk[e] = ptx::pack_bf16x2(__uint_as_float(vk[c + 2 * e]) * d128::kScale,
                                                         __uint_as_float(vk[c + 2 * e + 1]) * d128::kScale);
                                wv[e] = ptx::pack_bf16x2(__uint_as_float(vv[c + 2 * e]),
                                                         __uint_as_float(vv[c + 2 * e + 1]));
                            }
                            *reinterpret_cast<uint4*>(dk + q * 32 + c) = make_uint4(wk[0], wk[1], wk[2], wk[3]);
                            *reinterpret_cast<uint4*>(dv + q * 32 + c) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                        }
                    }
                }
            }
        }
        if (lane == 0) ptx::bulk_wait<0>();
        __syncwarp();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

// delta[bh, i] = sum_d dO[t, hd*64+d] * O[t, hd*64+d] and nl2 = -lse log2(e); also
// zeroes the fp32 dQ accumulator slice of (t, hd).  Eight threads per (token, head).
template <int D>
__global__ void k_attn_delta(const bf16* __restrict__ o, const bf16* __restrict__ dout, const float* __restrict__ lse,
                             float* __restrict__ delta, float* __restrict__ nl2, float* __restrict__ dq_acc, int tokens,
                             int seq, int heads, int zero) {
    constexpr int kD = D, kSub = D / 8;  // threads per (token, head), 8 elements each
    ptx::pdl_trigger();
    ptx::pdl_wait();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int pair = idx / kSub, sub = idx % kSub;
    const bool ok = pair < tokens * heads;  // no early return: the shuffles below need every lane
    const int t = ok ? pair / heads : 0, hd = ok ? pair % heads : 0;
    const int h = heads * kD;
    const size_t off = static_cast<size_t>(t) * h + hd * kD + sub * 8;
    const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
    const uint4 a = ok ? *reinterpret_cast<const uint4*>(o + off) : z4;
    const uint4 d = ok ? *reinterpret_cast<const uint4*>(dout + off) : z4;
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, dw[4] = {d.x, d.y, d.z, d.w};
    float acc = 0.0f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 fa = ptx::unpack_bf16x2(aw[e]), fd = ptx::unpack_bf16x2(dw[e]);
        acc = fmaf(fa.x, fd.x, fmaf(fa.y, fd.y, acc));
    }
#pragma unroll
    for (int w = 1; w < kSub; w *= 2) acc += __shfl_xor_sync(0xffffffffu, acc, w);
    if (!ok) return;
    if (zero) {  // else the previous call's backward kernel zeroed this accumulator
        float4* z = reinterpret_cast<float4*>(dq_acc + off);
        z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (sub == 0) {
        const int b = t / seq, i = t % seq;
        const size_t si = (static_cast<size_t>(b) * heads + hd) * seq + i;
        delta[si] = acc;
        nl2[si] = -lse[si] * kLog2e;  // exp(s/8 - lse) = exp2(s log2(e)/8 + nl2)
    }
}

// dq (bf16, x 1/sqrt(D)) = the fp32 accumulator.
template <int D>
__global__ void k_attn_dq_convert(const float* __restrict__ acc, bf16* __restrict__ dqkv, int tokens, int h) {
    constexpr float kSc = D == 64 ? 0.125f : d128::kScale;
    ptx::pdl_trigger();
    ptx::pdl_wait();
    const size_t total = static_cast<size_t>(tokens) * h / 8;
    for (size_t v = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; v < total;
         v += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t e = v * 8;
        const int t = static_cast<int>(e / h), c = static_cast<int>(e % h);
        const float4 x = *reinterpret_cast<const float4*>(acc + e);
        const float4 y = *reinterpret_cast<const float4*>(acc + e + 4);
        *reinterpret_cast<uint4*>(dqkv + static_cast<size_t>(t) * 3 * h + c) =
            make_uint4(ptx::pack_bf16x2(x.x * kSc, x.y * kSc), ptx::pack_bf16x2(x.z * kSc, x.w * kSc),
                       ptx::pack_bf16x2(y.x * kSc, y.y * kSc), ptx::pack_bf16x2(y.z * kSc, y.w * kSc));
    }
}

// One attribute call per (kernel, device); Tag tells apart kernels of the same type.
template <int Tag, typename K>
void set_smem_once(K kern, int bytes) {
    static std::atomic<uint32_t> done{0};
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    const uint32_t bit = 1u << (dev & 31);
    if (done.load() & bit) return;
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
               "cudaFuncSetAttribute(k_attn_bwd_tc)");
    done.fetch_or(bit);
}

}  // namespace

void attention_bwd_debug_timing(unsigned long long* dev_buf) {
    check_cuda(cudaMemcpyToSymbol(g_attn_bwd_dbg, &dev_buf, sizeof(dev_buf)), "cudaMemcpyToSymbol(g_attn_bwd_dbg)");
}

size_t attention_bwd_tc_scratch_floats(int batch, int seq, int heads, int head_dim) {
    // the fp32 dQ accumulator, then -lse log2(e) per (sequence, head, query)
    return static_cast<size_t>(batch) * seq * heads * head_dim + static_cast<size_t>(batch) * heads * seq;
}

void attention_bwd_tc(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, bf16* dqkv, float* delta,
                      float* scratch, int batch, int seq, int heads, bool causal, cudaStream_t s, int head_dim,
                      float* dq_alt, int phase, bool last) {
    const bool d128 = head_dim == 128;
    const int h = heads * head_dim;
    const int tokens = batch * seq;
    const int pairs = tokens * heads;
    float* nl2 = scratch + static_cast<size_t>(tokens) * h;
    // dQ accumulator of this call: with dq_alt (the model's consecutive calls, phase = 0, 1,
    // ...) the two buffers alternate; the delta kernel zeroes only the first call's, and
    // each call's backward kernel zeroes the next call's (read by its dq convert already).
    const bool dbuf = dq_alt != nullptr;
    float* dq_acc = dbuf && (phase & 1) ? dq_alt : scratch;
    float4* zero_next = dbuf && !last ? reinterpret_cast<float4*>((phase & 1) ? scratch : dq_alt) : nullptr;
    const long long zero_n4 = static_cast<long long>(tokens) * h / 4;
    const int zero_own = !dbuf || phase == 0;
    const int sub = head_dim / 8;
    if (d128)
        launch_pdl(k_attn_delta<128>, dim3((pairs * sub + 255) / 256), dim3(256), 0, s, "k_attn_delta", o, dout, lse,
                   delta, nl2, dq_acc, tokens, seq, heads, zero_own);
    else
        launch_pdl(k_attn_delta<64>, dim3((pairs * sub + 255) / 256), dim3(256), 0, s, "k_attn_delta", o, dout, lse,
                   delta, nl2, dq_acc, tokens, seq, heads, zero_own);
    const CUtensorMap tq = make_tmap_bf16_2d(qkv, 3ull * h, static_cast<uint64_t>(tokens), 3ll * h, 64, kT);
    const CUtensorMap tdo = make_tmap_bf16_2d(dout, static_cast<uint64_t>(h), static_cast<uint64_t>(tokens), h, 64, kT);
    const CUtensorMap tdq = make_tmap_f32_2d(dq_acc, static_cast<uint64_t>(h), static_cast<uint64_t>(tokens), h, 32, 32);
    const int bhn = batch * heads;
    const int items = bhn * (seq / kT);
    const int grid = std::min(items, num_sms());
    const float* cnl2 = nl2;
    const float* cdelta = delta;
    if (d128) {
        if (causal) {
            set_smem_once<0>(k_attn_bwd_tc128<true>, d128::kSmem);
            launch_pdl(k_attn_bwd_tc128<true>, dim3(grid), dim3(kThreads), d128::kSmem, s, "k_attn_bwd_tc", tq, tdo,
                       tdq, cnl2, cdelta, dqkv, seq, heads, bhn, zero_next, zero_n4);
        } else {
            set_smem_once<1>(k_attn_bwd_tc128<false>, d128::kSmem);
            launch_pdl(k_attn_bwd_tc128<false>, dim3(grid), dim3(kThreads), d128::kSmem, s, "k_attn_bwd_tc", tq, tdo,
                       tdq, cnl2, cdelta, dqkv, seq, heads, bhn, zero_next, zero_n4);
        }
    } else if (causal) {
        set_smem_once<2>(k_attn_bwd_tc<true>, kSmem);
        launch_pdl(k_attn_bwd_tc<true>, dim3(grid), dim3(kThreads), kSmem, s, "k_attn_bwd_tc", tq, tdo, tdq, cnl2,
                   cdelta, dqkv, dq_acc, seq, heads, bhn, zero_next, zero_n4);
    } else {
        set_smem_once<3>(k_attn_bwd_tc<false>, kSmem);
        launch_pdl(k_attn_bwd_tc<false>, dim3(grid), dim3(kThreads), kSmem, s, "k_attn_bwd_tc", tq, tdo, tdq, cnl2,
                   cdelta, dqkv, dq_acc, seq, heads, bhn, zero_next, zero_n4);
    }
    const size_t vecs = static_cast<size_t>(tokens) * h / 8;
    const dim3 cgrid(static_cast<int>(std::min<size_t>((vecs + 255) / 256, 148u * 16u)));
    const float* cacc = dq_acc;
    if (d128)
        launch_pdl(k_attn_dq_convert<128>, cgrid, dim3(256), 0, s, "k_attn_dq_convert", cacc, dqkv, tokens, h);
    else
        launch_pdl(k_attn_dq_convert<64>, cgrid, dim3(256), 0, s, "k_attn_dq_convert", cacc, dqkv, tokens, h);
    check_cuda(cudaGetLastError(), "attention_bwd_tc");
}

}  // namespace p2bw
