// Persistent, warp-specialised tcgen05 GEMM for the stage executor.
//
//   D[M x N] = A[M x K] . B[N x K]^T     (bf16 operands, fp32 accumulation in TMEM)
//
// One kernel serves the three dense contractions of every stage layer
// (reference: semantics.cpp:9-19 matmul -> forward, :21-32 matmul_tn -> dgrad,
// :34-44 matmul_nt -> wgrad accumulated like axpy at :329):
//   forward  Y  = X  . W^T    A = X  (K-major),  B = W (K-major)
//   dgrad    dX = dY . W      A = dY (K-major),  B = W (MN-major)
//   wgrad    dW += dY^T . X   A = dY (MN-major), B = X (MN-major), fp32 += epilogue
//
// Roles (384 threads, 1 CTA per SM, grid = min(tiles, #SMs), static round-robin tiles):
//   warp 0  : TMA producer  (one lane)   global -> SMEM ring of kStages stages
//   warp 1  : MMA issuer    (one lane)   tcgen05.mma 128 x BN x 16, commit -> mbarriers
//   warp 2  : TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4-11: epilogue    tcgen05.ld -> registers -> fused bias/GELU/residual -> global
//                           (two warps per TMEM lane quarter on alternate 64-column
//                           chunks: the GELU / dGELU epilogues outran the mainloop)
// The epilogue of tile i overlaps the main loop of tile i+1 through the two TMEM buffers.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "kernels.h"
#include "launch.h"
#include "tkernels.h"
#include "profiler.h"
#include "ptx.cuh"
#include "util.h"

namespace p2bw {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 bytes = one swizzle row
// Epilogue warps per CTA (kEW): 4 (one per TMEM lane quarter) for the plain bf16 and
// fp32 (wgrad) stores, 8 (two per quarter on alternate 64-column chunks) for the GELU /
// dGELU / residual epilogues, which outran the mainloop with 4 (fc1 forward 670 vs
// 1145 TF/s plain).  More epilogue SMEM costs stages, hence the split.
__host__ __device__ constexpr int gemm_threads(int kEW) { return 128 + 32 * kEW; }
constexpr int kEpiBuf = 32 * 128;  // one staging buffer: 32 rows x 128 B (TMA box, SW128)

// kCl == 2 is the CTA-pair (cta_group::2) mode: each CTA holds its own 128 rows of A
// and HALF of the B tile, so the same SMEM carries a deeper stage ring.  kCl == 4 is
// two such pairs side by side along N sharing their A rows: each CTA TMA-multicasts
// half of its A tile into itself and the matching CTA of the other pair, which
// halves the L2 -> SMEM bytes of A (the GEMMs are L2-feed bound at 256 x 256 tiles).
template <int BN, int kCl, int kEW>
struct GemmCfg {
    static constexpr int kABytes = kBM * kBK * 2;
    static constexpr int kBBytes = (BN / (kCl >= 2 ? 2 : 1)) * kBK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = BN == 128 ? 256 : 512;  // 2 x BN accumulator columns, a power of two
    static constexpr int kEpiBytes = kEW * 2 * kEpiBuf;  // epilogue warps x 2 buffers
    static constexpr int kFixed = kEpiBytes + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int kStages0 = (227 * 1024 - kFixed) / kStageBytes;
    static constexpr int kStages = kStages0 > 8 ? 8 : kStages0;
    static constexpr int kSmemBytes = kStages * kStageBytes + kFixed;
};

// tanh-GELU and its derivative in the fewest FP ops (the epilogue is issue-bound):
//   u = x (k0 + k0 k1 x^2), t = tanh(u), gelu = 0.5 x (1 + t)
//   gelu' = 0.5 (1 + t) + 0.5 x (1 - t^2) (k0 + 3 k0 k1 x^2)
__device__ __forceinline__ float gelu_fwd(float x) {
    constexpr float k0 = 0.7978845608028654f, k01 = 0.7978845608028654f * 0.044715f;
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(x * fmaf(x * x, k01, k0)));
    const float hx = 0.5f * x;
    return fmaf(hx, t, hx);
}

__device__ __forceinline__ float gelu_bwd(float x) {
    constexpr float k0 = 0.7978845608028654f, k01 = 0.7978845608028654f * 0.044715f;
    const float x2 = x * x;
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(x * fmaf(x2, k01, k0)));
    const float a = 0.5f * x * fmaf(x2, 3.0f * k01, k0);
    return fmaf(a, fmaf(-t, t, 1.0f), fmaf(0.5f, t, 0.5f));
}

struct KParams {
    int m, n, k;
    int splits;  // split-K factor (fp32 reduce-add epilogue only)
    GemmEpilogue epi;
    float* rsum;  // row sums of A (bias gradient partials [splits][m]) or nullptr
    // Tail split (bf16 epilogues, splits == 1): the last tail_tiles output tiles -- the
    // ragged last wave -- are cut into tail_f K parts run by otherwise idle CTAs.  Parts
    // 0 .. f-2 ("contributors") write fp32 partial accumulators to tail_ws and count
    // themselves in tail_flags (per tile, CTA of the pair and epilogue warp); part f-1
    // (the "finisher") waits for them, adds the partials and runs the fused epilogue.
    int tail_tiles, tail_f;
    float* tail_ws;
    unsigned* tail_flags;
    // Grouped raster: tiles walk N inside groups of `group_m` M tiles (0: M-fastest over
    // the whole output), so the operand L2 can hold is the one re-read.
    int group_m;
    // Ragged last N tile with <= BN / 2 valid columns (e.g. N = 1920 on 256-wide tiles):
    // issue its MMAs at N = BN / 2 (pair: BN / 4 columns of B per CTA) instead of spending
    // half the tensor work on zero-filled columns.  The accumulator's upper half then
    // holds stale values, which only ever reach columns >= n (clipped by the TMA stores).
    int half_n;
};

// Output tile (M-group index, N-group index) of tile number t.
__device__ __forceinline__ int2 tile_mn(int t, int tiles_mg, int tiles_ng, int gm) {
    if (gm <= 0) return make_int2(t % tiles_mg, t / tiles_mg);
    const int per = gm * tiles_ng;
    const int first = (t / per) * gm;
    const int gsz = min(tiles_mg - first, gm);
    const int r = t % per;
    return make_int2(first + r % gsz, r / gsz);
}

// One work unit: an output tile (group) over the K blocks [kb0, kb1).  role 0: a whole
// tile or split-K slice; 1: tail contributor part; 2: tail finisher.  Units are numbered
// full tiles first, then all contributors, then the finishers, and unit w runs on CTA
// slot w % slots: every finisher sits on a higher slot than its contributors, so with
// in-order CTA dispatch a spinning finisher never holds an SM its contributors need.
struct Unit {
    int tile, kb0, kb1, role, t, part;
};

__device__ __forceinline__ Unit unit_of(int w, int num_tiles, int kblocks, int kb_per, const KParams& p) {
    Unit u;
    const int full = num_tiles - p.tail_tiles;
    if (p.tail_tiles == 0 || w < full) {
        u.tile = w % num_tiles;
        u.kb0 = (w / num_tiles) * kb_per;
        u.kb1 = min(kblocks, u.kb0 + kb_per);
        u.role = 0;
        u.t = 0;
        u.part = 0;
        return u;
    }
    const int f = p.tail_f, j = w - full, nc = p.tail_tiles * (f - 1);
    if (j < nc) {
        u.t = j / (f - 1);
        u.part = j % (f - 1);
        u.role = 1;
    } else {
        u.t = j - nc;
        u.part = f - 1;
        u.role = 2;
    }
    u.tile = full + u.t;
    const int kbp = (kblocks + f - 1) / f;
    u.kb0 = u.part * kbp;
    u.kb1 = min(kblocks, u.kb0 + kbp);
    return u;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Output / side-input tensor maps of the epilogue (32-row boxes, 128 B rows, SW128).
struct EpiMaps {
    CUtensorMap d;    // D: bf16 box 64x32, or fp32 box 32x32
    CUtensorMap pre;  // GELU pre-activation copy (bf16)
    CUtensorMap aux;  // residual (StoreBF16) or u (DGeluBF16), bf16
};

// Byte offset of 16-byte chunk j of row r in a 128 B-row SW128 staging buffer.


// Phase timestamps (debug; null in production): p2bw_debug_gemm_timing.  Per CTA 8
// u64 of %globaltimer (ns, comparable across SMs): [0] entry, [1] setup done (barriers,
// TMEM, PDL wait), [2] producer issued its last load, [3] MMA saw its first full stage,
// [4] MMA issued its last commit, [5] epilogue warp 4 saw its first accumulator,
// [6] epilogue warp 4 done (stores read out), [7] teardown done.
__device__ unsigned long long* g_gemm_dbg = nullptr;

__device__ __forceinline__ void gmark(int k) {
    unsigned long long* p = g_gemm_dbg;
    if (p != nullptr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p[blockIdx.x * 8 + k] = t;
    }
}

// kCl == 2: a CTA pair (cluster of 2) computes one 256 x BN tile with cta_group::2
// MMAs issued by the even CTA: each CTA TMA-loads its own 128 A rows and half of the
// B tile into its SMEM (completing on the leader's full barrier), the accumulator
// rows land in each CTA's own TMEM, and both epilogues release the leader's TMEM
// buffer through remote mbarrier arrivals.
template <int BN, bool kAMN, bool kBMN, EpiKind kKind, int kCl, int kEW>
__global__ void __launch_bounds__(gemm_threads(kEW), 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                   const __grid_constant__ EpiMaps em, const KParams p) {
    using Cfg = GemmCfg<BN, kCl, kEW>;
    constexpr int S = Cfg::kStages;
    static_assert(!(kBMN && kCl >= 2 && (BN / 2) % 64 != 0), "MN-major B halves must be whole 64-column atoms");
    constexpr bool kPair = kCl >= 2;        // cta_group::2 MMAs over a CTA pair
    constexpr int kNP = kCl == 4 ? 2 : 1;   // pairs side by side along N
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* s_a = smem;
    uint8_t* s_b = smem + S * Cfg::kABytes;
    uint8_t* s_epi = smem + S * Cfg::kStageBytes;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(s_epi + Cfg::kEpiBytes);
    uint64_t* empty_bar = full_bar + S;
    uint64_t* tfull_bar = empty_bar + S;   // [2]
    uint64_t* tempty_bar = tfull_bar + 2;  // [2]
    uint64_t* aux_bar = tempty_bar + 2;    // [kEW] per epilogue warp
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aux_bar + kEW);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int tiles_m = (p.m + kBM - 1) / kBM;
    const int tiles_n = p.n / BN + (p.n % BN != 0);
    const int kblocks = (p.k + kBK - 1) / kBK;
    // work item w: tile group (w % num_tiles) -- kCl vertically adjacent M tiles of one
    // N tile, this CTA taking M tile kCl*g + rank -- and K slice (w / num_tiles)
    const int rank = kPair ? static_cast<int>(ptx::cluster_ctarank()) : 0;
    const int prank = rank & 1, pair = rank >> 1;  // rank inside the pair, pair index along N
    const int tiles_mg = kPair ? (tiles_m + 1) / 2 : tiles_m;
    const int tiles_ng = (tiles_n + kNP - 1) / kNP;
    const int num_tiles = tiles_mg * tiles_ng;
    const int num_work = p.tail_tiles > 0 ? num_tiles + p.tail_tiles * (p.tail_f - 1) : num_tiles * p.splits;
    const int kb_per = (kblocks + p.splits - 1) / p.splits;
    const int w0 = blockIdx.x / kCl, wstep = gridDim.x / kCl;
    const uint16_t pair_mask = static_cast<uint16_t>(kPair ? (0x3 << (2 * pair)) : 0x1);  // my pair's CTAs
    constexpr uint16_t kAllMask = kCl == 4 ? 0xF : (kCl == 2 ? 0x3 : 0x1);
    // half-width last tile: MN-major B halves must stay whole 64-column atoms
    constexpr bool kHalfOk = kCl <= 2 && (!kBMN || (BN / (kPair ? 4 : 2)) % 64 == 0);
    if (threadIdx.x == 0) gmark(0);

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmap_a);
        ptx::tma_prefetch_desc(&tmap_b);
        ptx::tma_prefetch_desc(&em.d);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full_bar[s], 1);
            // every pair leader's MMA commit frees a stage (+ the two row-sum warps)
            ptx::mbar_init(&empty_bar[s], kNP + (p.rsum != nullptr ? 2 : 0));
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull_bar[i], 1);
            ptx::mbar_init(&tempty_bar[i], kPair ? 2 * kEW : kEW);  // pair: both CTAs' epilogues
        }
        for (int i = 0; i < kEW; ++i) ptx::mbar_init(&aux_bar[i], 1);
        ptx::fence_mbar_init();
    }
    if (warp == 2) {
        if constexpr (kPair) ptx::tmem_alloc_2sm<Cfg::kTmemCols>(tmem_slot);
        else ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    }
    ptx::tc_fence_before();
    if constexpr (kPair) ptx::cluster_sync();  // peer barriers initialised before any multicast
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_trigger();  // launch.h: the next kernel's prologue may overlap our tail
    ptx::pdl_wait();     // the previous kernel's outputs (our operands) are complete
    if (threadIdx.x == 0) gmark(1);

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int w = w0; w < num_work; w += wstep) {
                const Unit u = unit_of(w, num_tiles, kblocks, kb_per, p);
                const int2 mn = tile_mn(u.tile, tiles_mg, tiles_ng, p.group_m);
                const int m0 = (mn.x * (kPair ? 2 : 1) + prank) * kBM;
                const int n0 = (mn.y * kNP + pair) * BN;
                for (int kb = u.kb0; kb < u.kb1; ++kb) {
                    ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
                    uint8_t* da = s_a + stage * Cfg::kABytes;
                    uint8_t* db = s_b + stage * Cfg::kBBytes;
                    const int k0 = kb * kBK;
                    if constexpr (kCl == 4) {
                        // A: my half of the shared A tile, multicast into me and my
                        // counterpart in the other pair; B: my half of my pair's B tile.
                        // Everything completes on each destination pair leader's barrier.
                        if (prank == 0) ptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::kStageBytes);
                        const uint16_t amask = static_cast<uint16_t>((1u << rank) | (1u << (rank ^ 2)));
                        if constexpr (kAMN)
                            ptx::tma_load_2d_2sm_mc(da + pair * 64 * kBK * 2, &tmap_a, &full_bar[stage], m0 + pair * 64,
                                                    k0, amask);
                        else
                            ptx::tma_load_2d_2sm_mc(da + pair * 64 * 128, &tmap_a, &full_bar[stage], k0, m0 + pair * 64,
                                                    amask);
                        const int nb = n0 + prank * (BN / 2);
                        if constexpr (kBMN) {
#pragma unroll
                            for (int j = 0; j < BN / 128; ++j)
                                ptx::tma_load_2d_2sm(db + j * 64 * kBK * 2, &tmap_b, &full_bar[stage], nb + j * 64,
                                                     k0);
                        } else {
                            ptx::tma_load_2d_2sm(db, &tmap_b, &full_bar[stage], k0, nb);
                        }
                    } else if constexpr (kCl == 2) {
                        // both CTAs' bytes complete on the leader's full barrier
                        if (rank == 0) ptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::kStageBytes);
                        if constexpr (kAMN) {
#pragma unroll
                            for (int j = 0; j < kBM / 64; ++j)
                                ptx::tma_load_2d_2sm(da + j * 64 * kBK * 2, &tmap_a, &full_bar[stage], m0 + j * 64,
                                                     k0);
                        } else {
                            ptx::tma_load_2d_2sm(da, &tmap_a, &full_bar[stage], k0, m0);
                        }
                        const bool half = kHalfOk && p.half_n && p.n - n0 <= BN / 2;
                        const int nb = n0 + rank * (half ? BN / 4 : BN / 2);  // my half of the B tile
                        if constexpr (kBMN) {
#pragma unroll
                            for (int j = 0; j < BN / 128; ++j)
                                ptx::tma_load_2d_2sm(db + j * 64 * kBK * 2, &tmap_b, &full_bar[stage], nb + j * 64,
                                                     k0);
                        } else {
                            ptx::tma_load_2d_2sm(db, &tmap_b, &full_bar[stage], k0, nb);
                        }
                    } else {
                    ptx::mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
                    if constexpr (kAMN) {
#pragma unroll
                        for (int j = 0; j < kBM / 64; ++j)
                            ptx::tma_load_2d(da + j * 64 * kBK * 2, &tmap_a, &full_bar[stage], m0 + j * 64, k0);
                    } else {
                        ptx::tma_load_2d(da, &tmap_a, &full_bar[stage], k0, m0);
                    }
                    if constexpr (kBMN) {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j)
                            ptx::tma_load_2d(db + j * 64 * kBK * 2, &tmap_b, &full_bar[stage], n0 + j * 64, k0);
                    } else {
                        ptx::tma_load_2d(db, &tmap_b, &full_bar[stage], k0, n0);
                    }
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            gmark(2);
        }
    } else if (warp == 1) {
        if (lane == 0 && prank == 0) {  // pair mode: the even CTA issues for both
            constexpr uint32_t idesc_full = ptx::idesc_bf16(kBM * (kPair ? 2 : 1), BN, kAMN, kBMN);
            constexpr uint32_t idesc_half = ptx::idesc_bf16(kBM * (kPair ? 2 : 1), BN / 2, kAMN, kBMN);
            // K-major SW128: rows of 128 B, 8-row groups 1024 B apart; a K step of 16
            // elements is +32 B inside the swizzle atom.  MN-major SW128: 64-element MN
            // groups one TMA box (kBK rows x 128 B) apart, 8-row K groups 1024 B apart;
            // a K step of 16 rows is +2048 B.
            constexpr uint32_t a_lbo = kAMN ? kBK * 128 : 16, a_sbo = 1024;
            constexpr uint32_t b_lbo = kBMN ? kBK * 128 : 16, b_sbo = 1024;
            constexpr uint32_t a_kstep = kAMN ? 16 * 128 : 32;
            constexpr uint32_t b_kstep = kBMN ? 16 * 128 : 32;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int w = w0; w < num_work; w += wstep) {
                const Unit u = unit_of(w, num_tiles, kblocks, kb_per, p);
                const int kb0 = u.kb0, kb1 = u.kb1;
                const int n0 = tile_mn(u.tile, tiles_mg, tiles_ng, p.group_m).y * kNP * BN;
                const uint32_t idesc = kHalfOk && p.half_n && p.n - n0 <= BN / 2 ? idesc_half : idesc_full;
                ptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&full_bar[stage], phase);
                    ptx::tc_fence_after();
                    if (w == w0 && kb == kb0) gmark(3);
                    const uint32_t a_addr = ptx::smem_u32(s_a + stage * Cfg::kABytes);
                    const uint32_t b_addr = ptx::smem_u32(s_b + stage * Cfg::kBBytes);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint64_t ad = ptx::sdesc_sw128(a_addr + kk * a_kstep, a_lbo, a_sbo);
                        const uint64_t bd = ptx::sdesc_sw128(b_addr + kk * b_kstep, b_lbo, b_sbo);
                        const uint32_t accum = (kb != kb0 || kk != 0) ? 1u : 0u;
                        if constexpr (kPair) ptx::umma_bf16_2sm(d_tmem, ad, bd, idesc, accum);
                        else ptx::umma_bf16(d_tmem, ad, bd, idesc, accum);
                    }
                    // the stage is free once every pair that reads it (kCl == 4: both,
                    // through the shared A halves) has consumed it
                    if constexpr (kPair) ptx::umma_commit_2sm_mc(&empty_bar[stage], kAllMask);
                    else ptx::umma_commit(&empty_bar[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if constexpr (kPair) ptx::umma_commit_2sm_mc(&tfull_bar[acc], pair_mask);
                else ptx::umma_commit(&tfull_bar[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
            gmark(4);
        }
    } else if ((warp == 2 || warp == 3) && p.rsum != nullptr) {
        // Row sums of A while it sits in SMEM (the bias gradient rides on the wgrad):
        // warp 2 + j sums A box j (64 rows of the tile) over this unit's K blocks.  Only
        // units in the first N tile sum (each A element counts once); every unit still
        // releases its stages.  Box layout (MN-major SW128): K row k is 128 B of 64 row
        // values, 16-byte chunk c at position c ^ (k & 7).  Lane: the 8 rows of chunk
        // lane & 7, K rows k = lane >> 3 (mod 4).
        if constexpr (kAMN && kKind == EpiKind::StoreF32 && !kPair) {
            const int j = warp - 2;
            const int c = lane & 7;  // 16-byte chunk: rows 8c .. 8c+7 of the box; K rows of lane >> 3 (mod 4)
            int stage = 0;
            uint32_t phase = 0;
            for (int w = w0; w < num_work; w += wstep) {  // (no tail split with row sums)
                const int tile = w % num_tiles;
                const int2 mn = tile_mn(tile, tiles_mg, tiles_ng, p.group_m);
                const int m0 = mn.x * kBM;
                const bool active = mn.y == 0;  // n0 == 0
                const int kb0 = (w / num_tiles) * kb_per;
                const int kb1 = min(kblocks, kb0 + kb_per);
                float acc[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&full_bar[stage], phase);
                    if (active) {
                        const uint32_t box = ptx::smem_u32(s_a + stage * Cfg::kABytes + j * 64 * kBK * 2);
#pragma unroll 4
                        for (int k = lane >> 3; k < kBK; k += 4) {
                            uint32_t v[4];
                            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                                         : "r"(box + k * 128 + ((c ^ (k & 7)) << 4)));
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                const float2 f = ptx::unpack_bf16x2(v[t]);
                                acc[2 * t] += f.x;
                                acc[2 * t + 1] += f.y;
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&empty_bar[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (active) {  // combine the four K-row phases (lanes c, c+8, c+16, c+24)
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        acc[q] += __shfl_down_sync(0xffffffffu, acc[q], 16);
                        acc[q] += __shfl_down_sync(0xffffffffu, acc[q], 8);
                    }
                    const int r = m0 + j * 64 + 8 * lane;
                    if (lane < 8 && r < p.m) {
                        float* dst = p.rsum + static_cast<size_t>(w / num_tiles) * p.m + r;
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (r + q < p.m) dst[q] = acc[q];
                    }
                }
            }
        } else if constexpr (!kAMN && !kPair) {
            // Column sums of a K-major A over the tile's rows (the bias gradient rides on
            // the dgrad, whose A is the layer's output gradient): per stage, the 64
            // columns of the A box summed over its 128 rows, one partial row per warp
            // and M tile.  Box layout (K-major SW128): row r is 128 B of 64 K values,
            // 16-byte chunk c at position c ^ (r & 7).  Lane L of the 64: chunk L & 7 of
            // rows (L >> 3) + 8 t, so its swizzled chunk position is fixed.
            const int L = (warp - 2) * 32 + lane;
            const int c = L & 7, rg = L >> 3;
            const uint32_t sw = static_cast<uint32_t>((c ^ rg) << 4);
            int stage = 0;
            uint32_t phase = 0;
            for (int w = w0; w < num_work; w += wstep) {
                const Unit u = unit_of(w, num_tiles, kblocks, kb_per, p);  // tail parts: disjoint K blocks
                const int2 mn = tile_mn(u.tile, tiles_mg, tiles_ng, p.group_m);
                const int mt = mn.x;
                const bool active = mn.y == 0;  // n0 == 0: each A element counts once
                const int kb0 = u.kb0, kb1 = u.kb1;
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&full_bar[stage], phase);
                    if (active) {
                        const uint32_t box = ptx::smem_u32(s_a + stage * Cfg::kABytes) + sw;
                        float acc[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 4
                        for (int t = 0; t < kBM / 8; ++t) {
                            uint32_t v[4];
                            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                                         : "r"(box + (rg + 8 * t) * 128));
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float2 f = ptx::unpack_bf16x2(v[q]);
                                acc[2 * q] += f.x;
                                acc[2 * q + 1] += f.y;
                            }
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q) {  // the warp's four row groups of chunk c
                            acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 8);
                            acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 16);
                        }
                        const int kc = kb * kBK + 8 * lane;
                        if (lane < 8 && kc < p.k) {
                            float* dst = p.rsum + static_cast<size_t>(mt * 2 + (warp - 2)) * p.k + kc;
                            reinterpret_cast<float4*>(dst)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                            reinterpret_cast<float4*>(dst)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&empty_bar[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp >= 4) {
        // Epilogue: warp q owns tile rows [32q, 32q+32) (its TMEM lane quarter).  Each
        // chunk of 128 B per row (64 bf16 / 32 fp32 columns) goes TMEM -> registers ->
        // fused math -> swizzled SMEM -> one TMA bulk-tensor store (or reduce-add).
        const int q = warp & 3;           // TMEM lane quarter (warp % 4, as tcgen05.ld requires)
        const int ew = warp - 4;          // epilogue warp index
        const int ch = ew >> 2;           // which alternate chunks of the tile's columns
        const GemmEpilogue& e = p.epi;
        uint8_t* ebuf = s_epi + ew * 2 * kEpiBuf;
        constexpr bool kF32 = kKind == EpiKind::StoreF32;
        constexpr int W = kF32 ? 32 : 64;  // columns per chunk
        const bool need_aux = kKind == EpiKind::DGeluBF16 || (kKind == EpiKind::StoreBF16 && e.residual != nullptr);
        const bool two_out = kKind == EpiKind::StoreBF16 && e.gelu && e.preact != nullptr;
        const bool reduce = kF32 && (e.beta != 0.0f || p.splits > 1);  // split-K: host pre-zeroed D
        uint32_t aux_phase = 0;
        int slot = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        constexpr bool kTail = !kF32 && kCl <= 2;
        constexpr int kP = kPair ? 2 : 1;
        for (int w = w0; w < num_work; w += wstep) {
            const Unit u = unit_of(w, num_tiles, kblocks, kb_per, p);
            const int tile = u.tile;
            const int2 mn = tile_mn(tile, tiles_mg, tiles_ng, p.group_m);
            const int m0 = (mn.x * (kPair ? 2 : 1) + prank) * kBM;
            const int n0 = (mn.y * kNP + pair) * BN;
            const int r0 = m0 + q * 32;
            const int role = kTail ? u.role : 0;
            // Side inputs (residual / GELU pre-activation) do not depend on the
            // accumulator: the warp's (<= 2) chunks of them are TMA-prefetched into its
            // two staging buffers before waiting for the MMA, hiding their latency.
            bool aux_pending = false;
            if (need_aux && role != 1) {
                if (lane == 0) ptx::bulk_wait_read<0>();  // both buffers read out by earlier stores
                __syncwarp();
                int bytes = 0;
                for (int c = ch, j = 0; c < BN / W && j < 2; c += kEW / 4, ++j)
                    if (n0 + c * W < p.n && r0 < p.m) bytes += kEpiBuf;
                aux_pending = bytes > 0;
                if (lane == 0 && bytes > 0) {
                    ptx::mbar_arrive_expect_tx(&aux_bar[ew], bytes);
                    for (int c = ch, j = 0; c < BN / W && j < 2; c += kEW / 4, ++j)
                        if (n0 + c * W < p.n && r0 < p.m)
                            ptx::tma_load_2d(ebuf + j * kEpiBuf, &em.aux, &aux_bar[ew], n0 + c * W, r0);
                }
            }
            ptx::mbar_wait(&tfull_bar[acc], acc_phase);
            ptx::tc_fence_after();
            if (ew == 0 && lane == 0 && w == w0) gmark(5);
            const uint32_t tbase =
                tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN);
            // tail split: this warp's partial block (fp32, [BN / 4 column quads][128 rows]
            // float4, so a warp's accesses are 512 contiguous bytes) and its arrival counter
            unsigned* tflag = nullptr;
            if constexpr (kTail) {
                if (role != 0) tflag = p.tail_flags + (u.t * kP + prank) * kEW + ew;
                if (role == 2) {  // finisher: wait for the f - 1 contributors of this tile
                    if (lane == 0) {
                        const unsigned want = static_cast<unsigned>(p.tail_f - 1);
                        while (ld_acquire_u32(tflag) != want) __nanosleep(64);
                        *tflag = 0u;  // re-armed for the next launch (all contributors are done)
                    }
                    __syncwarp();
                }
            }
            int jj = 0;  // index of this warp's chunk within the tile
#pragma unroll 1
            for (int c = ch; c < BN / W; c += kEW / 4, ++jj) {
                const int col0 = n0 + c * W;
                if (col0 >= p.n || r0 >= p.m) continue;  // warp-uniform: whole chunk out of range
                uint8_t* buf = ebuf + (need_aux ? jj : slot) * kEpiBuf;
                float x[W];
                {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(tbase + c * W, v);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(v[j]);
                    if constexpr (W == 64) {
                        ptx::tmem_ld_32x32b_x32(tbase + c * W + 32, v);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) x[32 + j] = __uint_as_float(v[j]);
                    }
                }
                if constexpr (kTail) {
                    if (role != 0) {
                        const int row = q * 32 + lane;
                        if (role == 1) {
                            float4* dst = reinterpret_cast<float4*>(
                                p.tail_ws +
                                (static_cast<size_t>((u.t * (p.tail_f - 1) + u.part) * kP + prank) * kBM * BN));
#pragma unroll
                            for (int j = 0; j < W / 4; ++j)
                                __stcg(dst + (c * (W / 4) + j) * kBM + row,
                                       make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]));
                            continue;
                        }
                        for (int part = 0; part < p.tail_f - 1; ++part) {  // fixed order: deterministic
                            const float4* src = reinterpret_cast<const float4*>(
                                p.tail_ws +
                                (static_cast<size_t>((u.t * (p.tail_f - 1) + part) * kP + prank) * kBM * BN));
#pragma unroll
                            for (int j = 0; j < W / 4; ++j) {
                                const float4 y = __ldcg(src + (c * (W / 4) + j) * kBM + row);
                                x[4 * j] += y.x;
                                x[4 * j + 1] += y.y;
                                x[4 * j + 2] += y.z;
                                x[4 * j + 3] += y.w;
                            }
                        }
                    }
                }
                if (e.alpha != 1.0f) {  // warp-uniform; the stage GEMMs all use alpha 1
#pragma unroll
                    for (int j = 0; j < W; ++j) x[j] *= e.alpha;
                }
                if (!need_aux) {
                    // the buffer's previous bulk store must have finished reading it
                    if (lane == 0) {
                        if (two_out) ptx::bulk_wait_read<0>();
                        else ptx::bulk_wait_read<1>();
                    }
                    __syncwarp();
                }
                if constexpr (kF32) {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        *reinterpret_cast<float4*>(buf + ptx::swz128(lane, j)) =
                            make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
                } else {
                    if (need_aux && aux_pending) {  // once per tile: both prefetched chunks
                        ptx::mbar_wait(&aux_bar[ew], aux_phase);
                        aux_phase ^= 1;
                        aux_pending = false;
                    }
                    if (kKind == EpiKind::StoreBF16 && e.bias != nullptr) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const uint4 bb = *reinterpret_cast<const uint4*>(e.bias + col0 + 8 * j);
                            const uint32_t bw[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                const float2 bf = ptx::unpack_bf16x2(bw[t]);
                                x[8 * j + 2 * t] += bf.x;
                                x[8 * j + 2 * t + 1] += bf.y;
                            }
                        }
                    }
                    if constexpr (kKind == EpiKind::DGeluBF16) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const uint4 uu = *reinterpret_cast<const uint4*>(buf + ptx::swz128(lane, j));
                            const uint32_t uw[4] = {uu.x, uu.y, uu.z, uu.w};
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                const float2 uf = ptx::unpack_bf16x2(uw[t]);
                                x[8 * j + 2 * t] *= gelu_bwd(uf.x);
                                x[8 * j + 2 * t + 1] *= gelu_bwd(uf.y);
                            }
                        }
                    } else {
                        if (two_out) {
                            // pre-activation copy into the other buffer; GELU of the
                            // bf16-rounded value so the backward sees the same function
                            uint8_t* pbuf = ebuf + (slot ^ 1) * kEpiBuf;
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                uint32_t w4[4];
#pragma unroll
                                for (int t = 0; t < 4; ++t) {
                                    w4[t] = ptx::pack_bf16x2(x[8 * j + 2 * t], x[8 * j + 2 * t + 1]);
                                    const float2 r = ptx::unpack_bf16x2(w4[t]);
                                    x[8 * j + 2 * t] = r.x;
                                    x[8 * j + 2 * t + 1] = r.y;
                                }
                                *reinterpret_cast<uint4*>(pbuf + ptx::swz128(lane, j)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                            }
                        }
                        if (e.gelu) {
#pragma unroll
                            for (int j = 0; j < W; ++j) x[j] = gelu_fwd(x[j]);
                        }
                        if (need_aux) {
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const uint4 rr = *reinterpret_cast<const uint4*>(buf + ptx::swz128(lane, j));
                                const uint32_t rw[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
                                for (int t = 0; t < 4; ++t) {
                                    const float2 rf = ptx::unpack_bf16x2(rw[t]);
                                    x[8 * j + 2 * t] += rf.x;
                                    x[8 * j + 2 * t + 1] += rf.y;
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        *reinterpret_cast<uint4*>(buf + ptx::swz128(lane, j)) =
                            make_uint4(ptx::pack_bf16x2(x[8 * j], x[8 * j + 1]),
                                       ptx::pack_bf16x2(x[8 * j + 2], x[8 * j + 3]),
                                       ptx::pack_bf16x2(x[8 * j + 4], x[8 * j + 5]),
                                       ptx::pack_bf16x2(x[8 * j + 6], x[8 * j + 7]));
                }
                ptx::fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    if (reduce) ptx::tma_reduce_add_2d(&em.d, buf, col0, r0);
                    else ptx::tma_store_2d(&em.d, buf, col0, r0);
                    if (two_out) ptx::tma_store_2d(&em.pre, ebuf + (slot ^ 1) * kEpiBuf, col0, r0);
                    ptx::bulk_commit();
                }
                if (!two_out) slot ^= 1;
            }
            if constexpr (kTail) {
                if (role == 1) {  // publish this warp's partial block
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) atomicAdd(tflag, 1u);
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (kPair) ptx::mbar_arrive_cluster(&tempty_bar[acc], 2 * pair);  // my pair leader
                else ptx::mbar_arrive(&tempty_bar[acc]);
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) ptx::bulk_wait_read<0>();
        __syncwarp();
        if (ew == 0 && lane == 0) gmark(6);
    }
    ptx::tc_fence_before();
    if constexpr (kPair) ptx::cluster_sync();  // no CTA exits while its peer may still signal it
    else __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        if constexpr (kPair) ptx::tmem_dealloc_2sm<Cfg::kTmemCols>(tmem_base);
        else ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    }
    if (threadIdx.x == 0) gmark(7);
}

}  // namespace

void gemm_debug_timing(unsigned long long* dev_buf) {
    check_cuda(cudaMemcpyToSymbol(g_gemm_dbg, &dev_buf, sizeof(dev_buf)), "cudaMemcpyToSymbol(g_gemm_dbg)");
}

namespace {

// d[r, c] = bf16(ws[r * n + c]) for an fp32 split-K workspace.
__global__ void k_cast_f32_bf16_2d(const float* __restrict__ ws, int m, int n, bf16* __restrict__ d, int64_t ldd) {
    const int nv = n / 4;
    for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < static_cast<int64_t>(m) * nv;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(v / nv), c = static_cast<int>(v % nv) * 4;
        const float4 x = *reinterpret_cast<const float4*>(ws + static_cast<int64_t>(r) * n + c);
        *reinterpret_cast<uint2*>(d + r * ldd + c) = make_uint2(ptx::pack_bf16x2(x.x, x.y), ptx::pack_bf16x2(x.z, x.w));
    }
}

void cast_f32_bf16_2d(const float* ws, int m, int n, bf16* d, int64_t ldd, cudaStream_t s) {
    const int64_t vec = static_cast<int64_t>(m) * (n / 4);
    k_cast_f32_bf16_2d<<<static_cast<int>(std::min<int64_t>((vec + 255) / 256, 148 * 16)), 256, 0, s>>>(ws, m, n, d,
                                                                                                         ldd);
    check_cuda(cudaGetLastError(), "cast_f32_bf16_2d");
}

// ---- host side -------------------------------------------------------------

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        check_cuda(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (p == nullptr || q != cudaDriverEntryPointSuccess)
            throw Error("cuTensorMapEncodeTiled is unavailable in this driver");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D tensor map with 128 B swizzle; box = {box_inner, box_outer} elements.
CUtensorMap make_map_t(const void* ptr, CUtensorMapDataType dt, int esize, uint64_t inner, uint64_t outer,
                       int64_t ld_elems, uint32_t box_inner, uint32_t box_outer) {
    CUtensorMap map;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems) * esize};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return map;
}

// bf16 map with a 64-element (128 B) inner box.
CUtensorMap make_map(const bf16* ptr, uint64_t inner, uint64_t outer, int64_t ld_elems, uint32_t box_outer) {
    return make_map_t(ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, inner, outer, ld_elems, 64, box_outer);
}

int wgrad_sms();

template <int BN, bool kAMN, bool kBMN, EpiKind kKind, int kCl, int kEW>
void launch(const CUtensorMap& ta, const CUtensorMap& tb, const EpiMaps& em, const KParams& p, cudaStream_t s) {
    using Cfg = GemmCfg<BN, kCl, kEW>;
    auto kern = gemm_tc_kernel<BN, kAMN, kBMN, kKind, kCl, kEW>;
    static std::atomic<uint32_t> configured{0};  // one attribute call per device
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    const uint32_t bit = 1u << (dev & 31);
    if ((configured.load() & bit) == 0) {
        check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes),
                   "cudaFuncSetAttribute(gemm smem)");
        configured.fetch_or(bit);
    }
    const int tiles_m = (p.m + kBM - 1) / kBM, tiles_n = (p.n + BN - 1) / BN;
    const int tiles_mg = kCl >= 2 ? (tiles_m + 1) / 2 : tiles_m;
    const int tiles_ng = kCl == 4 ? (tiles_n + 1) / 2 : tiles_n;
    const int work = p.tail_tiles > 0 ? tiles_mg * tiles_ng + p.tail_tiles * (p.tail_f - 1)
                                      : tiles_mg * tiles_ng * p.splits;
    // fp32 (weight-gradient) GEMMs may be held to fewer SMs (P2BW_GEMM_WGRAD_SMS, diagnostic:
    // the side stream's share of the GPU while the stage stream's chain runs beside it)
    const int slots = (kKind == EpiKind::StoreF32 && p.splits == 1 ? wgrad_sms() : num_sms()) / kCl;
    const int grid = kCl * (work < slots ? work : slots);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(gemm_threads(kEW));
    cfg.dynamicSmemBytes = Cfg::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // launch.h
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    check_cuda(cudaLaunchKernelEx(&cfg, kern, ta, tb, em, p), "gemm_tc_kernel launch");
}

template <int BN, bool kAMN, bool kBMN, int kCl>
void dispatch_epi(const CUtensorMap& ta, const CUtensorMap& tb, const EpiMaps& em, const KParams& p,
                  cudaStream_t s) {
    switch (p.epi.kind) {
        case EpiKind::StoreBF16:
            if (p.epi.gelu || p.epi.residual) launch<BN, kAMN, kBMN, EpiKind::StoreBF16, kCl, 8>(ta, tb, em, p, s);
            else launch<BN, kAMN, kBMN, EpiKind::StoreBF16, kCl, 4>(ta, tb, em, p, s);
            break;
        case EpiKind::StoreF32: launch<BN, kAMN, kBMN, EpiKind::StoreF32, kCl, 4>(ta, tb, em, p, s); break;
        case EpiKind::DGeluBF16: launch<BN, kAMN, kBMN, EpiKind::DGeluBF16, kCl, 8>(ta, tb, em, p, s); break;
    }
}

template <int BN, int kCl>
void dispatch_major(bool amn, bool bmn, const CUtensorMap& ta, const CUtensorMap& tb, const EpiMaps& em,
                    const KParams& p, cudaStream_t s) {
    if (!amn && !bmn) {
        dispatch_epi<BN, false, false, kCl>(ta, tb, em, p, s);
    } else if (amn && !bmn) {
        dispatch_epi<BN, true, false, kCl>(ta, tb, em, p, s);
    } else if constexpr (kCl >= 2 && (BN / 2) % 64 != 0) {
        throw Error("gemm: no CTA-pair tile with MN-major B for this BN");
    } else if (!amn) {
        dispatch_epi<BN, false, true, kCl>(ta, tb, em, p, s);
    } else {
        dispatch_epi<BN, true, true, kCl>(ta, tb, em, p, s);
    }
}

struct TileChoice {
    int bn;
    int cl;
    int splits;
    double t;  // modelled time, in 256 x 256 pair k-block units
    int tail_f = 1;  // tail split: K parts of each last-wave tile (1 = off)
};

// Tail-split workspace of one stream: the fp32 partials of at most one CTA per SM
// (tail tiles x (f - 1) contributor parts x CTAs per tile <= SMs) of 128 x 256 floats,
// and one arrival counter per (tail tile, CTA, epilogue warp) -- kept zero between
// launches by the finishers.  Allocated on a stream's first tail-split GEMM, outside
// graph capture (a capture without one runs the GEMM without the tail split).
struct TailPool {
    float* ws = nullptr;
    unsigned* flags = nullptr;
};

TailPool tail_pool(cudaStream_t s) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, TailPool>* pools = new std::map<std::pair<int, cudaStream_t>, TailPool>();
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    auto it = pools->find({dev, s});
    if (it != pools->end()) return it->second;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    check_cuda(cudaStreamIsCapturing(s, &cs), "cudaStreamIsCapturing");
    if (cs != cudaStreamCaptureStatusNone) return TailPool{};
    TailPool tp;
    const size_t n_ws = static_cast<size_t>(num_sms()) * kBM * 256;
    const size_t n_flags = static_cast<size_t>(num_sms()) * 8;
    check_cuda(cudaMalloc(&tp.ws, n_ws * sizeof(float)), "cudaMalloc(gemm tail workspace)");
    check_cuda(cudaMalloc(&tp.flags, n_flags * sizeof(unsigned)), "cudaMalloc(gemm tail flags)");
    check_cuda(cudaMemset(tp.flags, 0, n_flags * sizeof(unsigned)), "cudaMemset(gemm tail flags)");
    (*pools)[{dev, s}] = tp;
    return tp;
}

bool raster_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("P2BW_GEMM_RASTER");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return on;
}

bool tail_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("P2BW_GEMM_TAIL");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return on;
}

int wgrad_sms() {
    static const int n = [] {
        const char* e = std::getenv("P2BW_GEMM_WGRAD_SMS");
        const int v = e ? std::atoi(e) : 0;
        return v >= 2 && v < num_sms() ? v : num_sms();
    }();
    return n;
}
// Half-width ragged last N tile (KParams::half_n); P2BW_GEMM_HALF_N=0 turns it off.
bool half_n_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("P2BW_GEMM_HALF_N");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return on;
}

// Upper bound on split-K slices of the fp32 (weight-gradient) GEMMs; P2BW_GEMM_MAX_SPLIT
// overrides it (diagnostic A/B knob).
int max_split_cap() {
    static const int cap = [] {
        const char* e = std::getenv("P2BW_GEMM_MAX_SPLIT");
        return e ? std::max(1, std::atoi(e)) : 1 << 20;
    }();
    return cap;
}

bool tile_ok(int bn, int cl, bool bmn) { return !(bmn && cl >= 2 && (bn / 2) % 64 != 0); }

// Steady-state speed of a tile shape relative to the 256 x 256 CTA-pair tile, from the
// B200 sweeps (scripts/gemm_sweep.py, profiles/r1_gemm_sweep_*.json, corrected for
// each shape's wave efficiency): 128 x 256 0.95, 128 x 192 0.86, 128 x 128 0.67,
// pair 256 x 192 0.89, pair 256 x 128 0.64.  (4-CTA clusters sharing A by TMA
// multicast measured slower on every stage shape and are only reachable by the knob.)
double tile_speed(int bn, int cl) {
    if (cl == 2) return bn == 256 ? 1.0 : (bn == 192 ? 0.89 : 0.64);
    return bn == 256 ? 0.95 : (bn == 192 ? 0.86 : 0.67);
}

// Tile shape, cluster and split-K minimising a wave-quantised time model:
//   time = waves * (k-blocks per unit * tile time per k-block + per-unit overhead)
// where a unit is one output tile (or K slice of it) of one CTA (pair), waves =
// ceil(units / (SMs / cluster)), the per-unit overhead (pipeline fill + the epilogue
// of the last unit) is ~3 k-blocks, and split-K slices pay one more for their fp32
// reduce-add.  The ragged last wave is what this decides: 96 pair tiles of a
// [8192 x 768] output on 74 SM pairs run as two waves at 65% occupancy, 256 128 x 192
// tiles as two waves at 86%.  fp32 (wgrad) outputs keep 256-wide tiles, which the
// sweeps favour for MN-major operands, and choose only their split count.
//
// Tail split (bf16 outputs): the r tiles of a ragged last wave may instead run as f K
// parts each on the idle slots (r f <= slots), the last wave then costing
// ceil(kb / f) k-blocks plus the fp32 partial traffic through L2 (~128 KB written and
// read per contributor CTA, ~7.5 k-block times per part at a 256-wide tile, measured).
TileChoice choose_tile(int m, int n, int k, bool f32_out, bool bmn, bool allow_split, bool single_cta = false,
                       bool allow_tail = false) {
    const int kblocks = (k + kBK - 1) / kBK;
    if (const char* env = std::getenv("P2BW_GEMM_TILE")) {  // tuning knob: "bn,cl[,splits]"
        int bn = 0, cl = 0, sp = 0;
        const int got = std::sscanf(env, "%d,%d,%d", &bn, &cl, &sp);
        if (got >= 2 && (bn == 128 || bn == 192 || bn == 256) && (cl == 1 || cl == 2 || cl == 4))
            return {bn, cl, allow_split && got == 3 && sp >= 1 ? std::min(sp, kblocks) : 1, 0.0};
    }
    const int sms = num_sms();
    TileChoice best{256, 1, 1, 1e300};
    double best_t = 1e300;
    for (int bn : {256, 192, 128}) {
        if (f32_out && bn != 256) continue;
        for (int cl : {2, 1}) {
            if (!tile_ok(bn, cl, bmn) || (cl == 2 && m <= kBM) || (cl == 2 && single_cta)) continue;
            const int tiles_m = (m + kBM - 1) / kBM;
            const int tiles = (cl == 2 ? (tiles_m + 1) / 2 : tiles_m) * ((n + bn - 1) / bn);
            const int max_split = allow_split ? std::min(max_split_cap(), std::max(1, kblocks / 8)) : 1;  // >= 8 k-blocks (512) per slice
            const double per_kb = (bn / 256.0) / tile_speed(bn, cl);
            for (int sp = 1; sp <= max_split; ++sp) {
                const int kb_per = (kblocks + sp - 1) / sp;
                const int s_eff = (kblocks + kb_per - 1) / kb_per;
                if (s_eff != sp) continue;  // no empty slices
                const long units = static_cast<long>(tiles) * s_eff;
                const long slots = sms / cl;
                const long waves = (units + slots - 1) / slots;
                const double t = waves * (kb_per * per_kb + 3.0 + (s_eff > 1 ? 1.0 : 0.0));
                if (t < best_t - 1e-9) {
                    best_t = t;
                    best = {bn, cl, s_eff, t};
                }
                if (allow_tail && sp == 1 && units % slots != 0) {
                    const long full_waves = units / slots, r = units % slots;
                    const int f = static_cast<int>(std::min<long>({4, slots / r, kblocks / 8}));
                    if (f >= 2) {
                        const double tt = full_waves * (kblocks * per_kb + 3.0) +
                                          ((kblocks + f - 1) / f) * per_kb + 3.0 + 7.5 * f * (bn / 256.0);
                        if (tt < best_t - 1e-9) {
                            best_t = tt;
                            best = {bn, cl, 1, tt, f};
                        }
                    }
                }
            }
        }
    }
    return best;
}

// The launch plan of the main path: tile, cluster, split-K and tail split.
TileChoice plan_tile(int m, int n, int k, bool bmn, bool f32, bool want_rsum, bool want_csum) {
    const bool tail_ok = !f32 && !want_rsum && tail_enabled();
    TileChoice tc = choose_tile(m, n, k, f32, bmn, f32, want_rsum || want_csum, tail_ok);
    if (!tile_ok(tc.bn, tc.cl, bmn)) tc.cl = 1;
    if (want_rsum || want_csum) tc.cl = 1;  // the sum warps read a local full barrier (no CTA pairs)
    if (!f32) tc.splits = 1;
    if (!tail_ok || tc.cl > 2) tc.tail_f = 1;
    return tc;
}

}  // namespace

void gemm_plan(int m, int n, int k, bool amn, bool bmn, bool f32, bool bias_grad, int out[4]) {
    const TileChoice tc = plan_tile(m, n, k, bmn, f32, bias_grad && amn, bias_grad && !amn);
    out[0] = tc.bn;
    out[1] = tc.cl;
    out[2] = tc.splits;
    out[3] = tc.tail_f;
}

CUtensorMap make_tmap_bf16_2d(const bf16* ptr, uint64_t inner, uint64_t outer, int64_t ld_elems,
                              uint32_t box_inner, uint32_t box_outer) {
    if (box_inner != 64) throw Error("tensor maps here use a 64-element (128 B) swizzled inner box");
    return make_map(ptr, inner, outer, ld_elems, box_outer);
}

CUtensorMap make_tmap_f32_2d(const float* ptr, uint64_t inner, uint64_t outer, int64_t ld_elems, uint32_t box_inner,
                             uint32_t box_outer) {
    if (box_inner != 32) throw Error("fp32 tensor maps here use a 32-element (128 B) swizzled inner box");
    return make_map_t(ptr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, inner, outer, ld_elems, box_inner, box_outer);
}

void gemm_bf16(const GemmOperand& a, const GemmOperand& b, int m, int n, int k,
               const GemmEpilogue& epi, cudaStream_t stream) {
    if (m <= 0 || n <= 0 || k <= 0) throw Error("gemm: empty problem");
    if (n % 32 != 0) throw Error("gemm: N must be a multiple of 32");
    if ((a.ld % 8) != 0 || (b.ld % 8) != 0) throw Error("gemm: leading dims must be multiples of 8");
    if (epi.kind == EpiKind::StoreF32 && epi.beta != 0.0f && epi.beta != 1.0f)
        throw Error("gemm: fp32 epilogue supports beta 0 (store) or 1 (TMA reduce-add) only");
    if ((epi.ldd % 8) != 0 || (epi.residual && epi.ldr % 8 != 0))
        throw Error("gemm: output leading dims must be multiples of 8");
    const bool amn = a.major == Major::MN, bmn = b.major == Major::MN;
    const bool f32 = epi.kind == EpiKind::StoreF32;
    const bool want_rsum = epi.bias_grad != nullptr && amn;   // wgrad: row sums of A over K
    const bool want_csum = epi.bias_grad != nullptr && !amn;  // dgrad: column sums of A over M
    if (want_rsum && !f32) throw Error("gemm: bias_grad with an MN-major A needs an fp32 store (wgrad)");
    if (want_csum && k % 8 != 0) throw Error("gemm: bias_grad with a K-major A needs K % 8 == 0");
    TileChoice tc = plan_tile(m, n, k, bmn, f32, want_rsum, want_csum);
    // Plain bf16 stores with few output tiles and a long K (the LM-head dgrad: 1232 x 768
    // over K = 30592 fills 60 SMs with 128 x 128 tiles) run split-K into the caller's
    // fp32 workspace and are cast afterwards, when the model says that wins.
    const bool plain = epi.kind == EpiKind::StoreBF16 && !epi.bias && !epi.residual && !epi.gelu && !epi.preact;
    if (plain && !want_csum && epi.workspace != nullptr && epi.workspace_floats >= static_cast<int64_t>(m) * n &&
        std::getenv("P2BW_GEMM_TILE") == nullptr) {
        TileChoice ts = choose_tile(m, n, k, true, bmn, true);
        // memset + cast: ~10 B per output at HBM speed, in k-block units (~0.26 us each)
        ts.t += 10.0 * m * n / 6.5e12 / 0.26e-6;
        if (ts.splits > 1 && ts.t < tc.t) {
            GemmEpilogue f;
            f.kind = EpiKind::StoreF32;
            f.d = epi.workspace;
            f.ldd = n;
            f.alpha = epi.alpha;
            f.beta = 0.0f;
            gemm_bf16(a, b, m, n, k, f, stream);
            cast_f32_bf16_2d(epi.workspace, m, n, static_cast<bf16*>(epi.d), epi.ldd, stream);
            return;
        }
    }
    const int bn = tc.bn, cl = tc.cl;
    int tail_tiles = 0, tail_f = 1;
    TailPool tp{};
    if (tc.tail_f >= 2) {
        const int tiles_m = (m + kBM - 1) / kBM;
        const int units = (cl == 2 ? (tiles_m + 1) / 2 : tiles_m) * ((n + bn - 1) / bn);
        const int slots = num_sms() / cl;
        tp = tail_pool(stream);
        if (tp.ws != nullptr && units % slots != 0 && (units % slots) * tc.tail_f <= slots) {
            tail_tiles = units % slots;
            tail_f = tc.tail_f;
        }
    }
    // A: rows = m (tile kBM), B: rows = n (tile bn; each CTA of a pair loads bn / 2).
    // K-major maps put k innermost.
    // kCl == 4: each CTA multicasts half (64 rows) of the A tile
    const CUtensorMap ta = amn ? make_map(a.ptr, m, k, a.ld, kBK) : make_map(a.ptr, k, m, a.ld, cl == 4 ? kBM / 2 : kBM);
    const CUtensorMap tb = bmn ? make_map(b.ptr, n, k, b.ld, kBK) : make_map(b.ptr, k, n, b.ld, bn / (cl >= 2 ? 2 : 1));
    EpiMaps em{};
    if (epi.kind == EpiKind::StoreF32) {
        em.d = make_map_t(epi.d, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, n, m, epi.ldd, 32, 32);
    } else {
        em.d = make_map(static_cast<const bf16*>(epi.d), n, m, epi.ldd, 32);
        if (epi.kind == EpiKind::StoreBF16 && epi.gelu && epi.preact)
            em.pre = make_map(epi.preact, n, m, epi.ldd, 32);
        if (epi.kind == EpiKind::StoreBF16 && epi.residual)
            em.aux = make_map(epi.residual, n, m, epi.ldr, 32);
        if (epi.kind == EpiKind::DGeluBF16) {
            if (!epi.aux) throw Error("gemm: DGelu epilogue needs the pre-activation");
            em.aux = make_map(epi.aux, n, m, epi.ldd, 32);
        }
    }
    // Split-K for fp32 (wgrad) GEMMs whose output has too few tiles to fill the
    // SMs: every K slice reduce-adds into D (pre-zeroed when beta == 0).
    const int splits = f32 ? tc.splits : 1;
    if (epi.kind == EpiKind::StoreF32) {
        if (splits > 1 && epi.beta == 0.0f) {
            if (epi.ldd == n) {
                check_cuda(cudaMemsetAsync(epi.d, 0, static_cast<size_t>(m) * n * sizeof(float), stream), "memset");
            } else {
                check_cuda(cudaMemset2DAsync(epi.d, static_cast<size_t>(epi.ldd) * sizeof(float), 0,
                                             static_cast<size_t>(n) * sizeof(float), static_cast<size_t>(m), stream),
                           "memset2D");
            }
        }
    }
    float* rsum = nullptr;
    const int csum_parts = 2 * ((m + kBM - 1) / kBM);  // two warps' partial rows per M tile
    if (want_rsum) {
        if (epi.bias_scratch == nullptr || epi.bias_scratch_floats < static_cast<int64_t>(splits) * m)
            throw Error("gemm: bias_scratch must hold splits * M floats");
        rsum = epi.bias_scratch;
    }
    if (want_csum) {
        if (epi.bias_scratch == nullptr || epi.bias_scratch_floats < static_cast<int64_t>(csum_parts) * k)
            throw Error("gemm: bias_scratch must hold 2 * ceil(M / 128) * K floats");
        rsum = epi.bias_scratch;
    }
    // Raster order by which operand L2 (126 MB) can keep: A resident -> M fastest (B is
    // streamed once); else B resident -> N fastest within each M tile (A streamed once);
    // else groups of ~sqrt(concurrent units) M tiles.  (M-fastest everywhere re-streamed a
    // 126 MB wgrad A once per N column.)
    int group_m = 0;
    if (raster_enabled()) {
        const double a_bytes = 2.0 * m * k, b_bytes = 2.0 * n * k, resident = 48e6;
        if (a_bytes > resident) group_m = b_bytes <= resident ? 1 : 8;
    }
    KParams p{m, n, k, splits, epi, rsum, tail_tiles, tail_f, tp.ws, tp.flags, group_m, half_n_enabled() ? 1 : 0};
    const double out_bytes = epi.kind == EpiKind::StoreF32 ? (epi.beta != 0.0f ? 8.0 : 4.0) : 2.0;
    // profiler class by pass: forward (K-major x K-major), dgrad (B MN-major), wgrad (both MN-major)
    const char* cls = amn ? "gemm_wgrad" : (bmn ? "gemm_dgrad" : "gemm_fwd");
    prof::Scope scope(cls, 2.0 * m * n * k,
                      2.0 * (static_cast<double>(m) * k + static_cast<double>(n) * k) + out_bytes * m * n, 1,
                      stream);
    if (bn == 256 && cl == 4) dispatch_major<256, 4>(amn, bmn, ta, tb, em, p, stream);
    else if (bn == 192 && cl == 4) dispatch_major<192, 4>(amn, bmn, ta, tb, em, p, stream);
    else if (bn == 128 && cl == 4) dispatch_major<128, 4>(amn, bmn, ta, tb, em, p, stream);
    else if (bn == 256 && cl == 2) dispatch_major<256, 2>(amn, bmn, ta, tb, em, p, stream);
    else if (bn == 256) dispatch_major<256, 1>(amn, bmn, ta, tb, em, p, stream);
    else if (bn == 192 && cl == 2) dispatch_major<192, 2>(amn, bmn, ta, tb, em, p, stream);
    else if (bn == 192) dispatch_major<192, 1>(amn, bmn, ta, tb, em, p, stream);
    else if (cl == 2) dispatch_major<128, 2>(amn, bmn, ta, tb, em, p, stream);
    else dispatch_major<128, 1>(amn, bmn, ta, tb, em, p, stream);
    if (want_rsum) reduce_partials(rsum, splits, m, epi.bias_grad, !epi.bias_grad_accumulate, stream);
    if (want_csum) reduce_partials(rsum, csum_parts, k, epi.bias_grad, !epi.bias_grad_accumulate, stream);
}

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
        check_cuda(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev),
                   "cudaDeviceGetAttribute(SM count)");
    }
    return n;
}

}  // namespace p2bw
