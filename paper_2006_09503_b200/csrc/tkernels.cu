// Transformer-stage kernels other than the tcgen05 GEMM: embedding, LayerNorm,
// deterministic column reductions (bias / LN-parameter gradients), fused
// softmax cross-entropy, the fused momentum optimizer and synthetic init.
// All are HBM-bound: 16-byte vector accesses, one warp (LN) or one CTA (CE)
// per row, grids sized to the SM count where a reduction follows.
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "profiler.h"
#include "ptx.cuh"
#include "launch.h"
#include "tkernels.h"
#include "util.h"

namespace p2bw {
namespace {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void load8(const bf16* p, float (&v)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = ptx::unpack_bf16x2(w[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}

__device__ __forceinline__ void store8(bf16* p, const float (&v)[8]) {
    *reinterpret_cast<uint4*>(p) = make_uint4(ptx::pack_bf16x2(v[0], v[1]), ptx::pack_bf16x2(v[2], v[3]),
                                              ptx::pack_bf16x2(v[4], v[5]), ptx::pack_bf16x2(v[6], v[7]));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

int grid_for(size_t n, int threads) {
    return static_cast<int>(std::min<size_t>((n + threads - 1) / threads, 148u * 64u));
}

// ---- embedding ----------------------------------------------------------------------

__global__ void k_embed_fwd(const int* __restrict__ ids, const bf16* __restrict__ tok,
                            const bf16* __restrict__ pos, bf16* __restrict__ x0, int tokens, int seq,
                            int h) {
    const int hv = h / 8;
    const size_t total = static_cast<size_t>(tokens) * hv;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int t = static_cast<int>(i / hv), c = static_cast<int>(i % hv) * 8;
        float a[8], b[8];
        load8(tok + static_cast<size_t>(ids[t]) * h + c, a);
        load8(pos + static_cast<size_t>(t % seq) * h + c, b);
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] += b[q];
        store8(x0 + static_cast<size_t>(t) * h + c, a);
    }
}

__global__ void k_embed_bwd_tok(const int* __restrict__ ids, const bf16* __restrict__ dx0,
                                float* __restrict__ dtok, int tokens, int h) {
    const int hv = h / 8;
    const size_t total = static_cast<size_t>(tokens) * hv;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int t = static_cast<int>(i / hv), c = static_cast<int>(i % hv) * 8;
        float g[8];
        load8(dx0 + static_cast<size_t>(t) * h + c, g);
        float* dst = dtok + static_cast<size_t>(ids[t]) * h + c;  // 32-byte aligned (h % 8 == 0)
        // two 16-byte vector reductions instead of eight scalar atomics
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(g[0]), "f"(g[1]), "f"(g[2]),
                     "f"(g[3])
                     : "memory");
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4), "f"(g[4]), "f"(g[5]), "f"(g[6]),
                     "f"(g[7])
                     : "memory");
    }
}

__global__ void k_embed_bwd_pos(const bf16* __restrict__ dx0, float* __restrict__ dpos, int batch,
                                int seq, int h, int overwrite) {
    const int hv = h / 8;
    const size_t total = static_cast<size_t>(seq) * hv;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int p = static_cast<int>(i / hv), c = static_cast<int>(i % hv) * 8;
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 8
        for (int b = 0; b < batch; ++b) {  // unrolled: eight sequences' loads in flight
            float g[8];
            load8(dx0 + (static_cast<size_t>(b) * seq + p) * h + c, g);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] += g[q];
        }
        float* dst = dpos + static_cast<size_t>(p) * h + c;
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[q] = overwrite ? acc[q] : dst[q] + acc[q];
    }
}

// ---- deterministic reductions ------------------------------------------------------

// Second phase of the deterministic column reductions, for up to 3 statistics at
// once (blockIdx.y): out_y[c] (=|+=) sum_{p < parts} part[(y * parts + p) * n + c] in a
// fixed order.  8 columns x 32 part lanes per CTA, so even a 768-wide statistic
// spreads over 96 CTAs; each thread keeps its (parts / 32) loads in flight at once
// (the phase is latency-, not byte-bound: it was 7 us at 24 CTAs x 8 part lanes).
struct ReduceOut {
    float* out[3];
};

__global__ void __launch_bounds__(256) k_reduce_parts(const float* __restrict__ part, int parts, int n,
                                                      ReduceOut outs, int overwrite) {
    ptx::pdl_trigger();
    ptx::pdl_wait();
    __shared__ float red[32][9];
    const int cl = threadIdx.x & 7, plane = threadIdx.x >> 3;
    const int col = blockIdx.x * 8 + cl;
    const float* base = part + static_cast<size_t>(blockIdx.y) * parts * n;
    float acc = 0.0f;
    if (col < n) {
        int p = plane;
        for (; p + 96 < parts; p += 128) {
            const float v0 = base[static_cast<size_t>(p) * n + col], v1 = base[static_cast<size_t>(p + 32) * n + col];
            const float v2 = base[static_cast<size_t>(p + 64) * n + col], v3 = base[static_cast<size_t>(p + 96) * n + col];
            acc += v0;
            acc += v1;
            acc += v2;
            acc += v3;
        }
        for (; p < parts; p += 32) acc += base[static_cast<size_t>(p) * n + col];
    }
    red[plane][cl] = acc;
    __syncthreads();
    if (plane == 0 && col < n) {
        float s = 0.0f;
#pragma unroll
        for (int i = 0; i < 32; ++i) s += red[i][cl];
        float* out = outs.out[blockIdx.y];
        out[col] = overwrite ? s : out[col] + s;
    }
}

void reduce_parts(const float* part, int parts, int n, float* out, bool overwrite, cudaStream_t s) {
    ReduceOut o{{out, nullptr, nullptr}};
    launch_pdl(k_reduce_parts, dim3((n + 7) / 8, 1), dim3(256), 0, s, "k_reduce_parts", part, parts, n, o,
               overwrite ? 1 : 0);
}

// Column statistics of a bf16 matrix, per row-block partials (block = 32 column
// vectors of 8 = 256 columns x 8 row lanes):
//   kLn = false: part0[c] = sum_r x[r, c]                       (bias gradient)
//   kLn = true : part0[c] = sum_r dy[r, c] * (x[r, c] - mean_r) * rstd_r   (LN gamma)
//                part1[c] = sum_r dy[r, c]                                (LN beta)
template <bool kLn>
__global__ void __launch_bounds__(256) k_colstats(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                                  const float* __restrict__ mean, const float* __restrict__ rstd,
                                                  int rows, int n, int ld, int rows_per_block,
                                                  float* __restrict__ part0, float* __restrict__ part1) {
    ptx::pdl_trigger();
    ptx::pdl_wait();
    __shared__ float red[8][256 + 8];
    const int cv = threadIdx.x & 31, rl = threadIdx.x >> 5;
    const int col = blockIdx.x * 256 + cv * 8;
    const int r0 = blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
    float a0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, a1[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (col < n) {
        if constexpr (kLn) {
#pragma unroll 4
            for (int r = r0 + rl; r < r1; r += 8) {
                float g[8], xv[8];
                load8(dy + static_cast<size_t>(r) * ld + col, g);
                load8(x + static_cast<size_t>(r) * ld + col, xv);
                const float mu = mean[r], rs = rstd[r];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    a0[q] = fmaf(g[q], (xv[q] - mu) * rs, a0[q]);
                    a1[q] += g[q];
                }
            }
        } else {
            // eight rows' 16-byte vectors in flight per thread (the pass is latency-bound)
            int r = r0 + rl;
            for (; r + 56 < r1; r += 64) {
                uint4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const uint4*>(dy + static_cast<size_t>(r + 8 * u) * ld + col);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const float2 f = ptx::unpack_bf16x2(w[t]);
                        a0[2 * t] += f.x;
                        a0[2 * t + 1] += f.y;
                    }
                }
            }
            for (; r < r1; r += 8) {
                float g[8];
                load8(dy + static_cast<size_t>(r) * ld + col, g);
#pragma unroll
                for (int q = 0; q < 8; ++q) a0[q] += g[q];
            }
        }
    }
    const int c = threadIdx.x;  // 256 columns of this block
    for (int pass = 0; pass < (kLn ? 2 : 1); ++pass) {
#pragma unroll
        for (int q = 0; q < 8; ++q) red[rl][cv * 8 + q] = pass == 0 ? a0[q] : a1[q];
        __syncthreads();
        if (blockIdx.x * 256 + c < n) {
            float s = 0.0f;
#pragma unroll
            for (int i = 0; i < 8; ++i) s += red[i][c];
            (pass == 0 ? part0 : part1)[static_cast<size_t>(blockIdx.y) * n + blockIdx.x * 256 + c] = s;
        }
        __syncthreads();
    }
}

// Row blocks so that the grid fills every SM with 8 CTAs; each block still sees >= 16 rows.
int colsum_row_blocks(int rows, int n) {
    const int col_blocks = (n + 255) / 256;
    const int want = (8 * 148 + col_blocks - 1) / col_blocks;
    return std::max(1, std::min(want, (rows + 15) / 16));
}

// ---- LayerNorm (one warp per row, up to NV 8-element vectors per lane) -------------------

template <int NV>
__global__ void k_ln_fwd(const bf16* __restrict__ x, const bf16* __restrict__ g, const bf16* __restrict__ b,
                         bf16* __restrict__ y, float* __restrict__ mean, float* __restrict__ rstd, int rows,
                         int h) {
    // R rows per warp (loads of all R rows in flight together).  R = 2 helped an older
    // version that was latency-bound; today R = 1 is faster (BERT-base microbatch,
    // CUDA-graph timed: 6.36 -> 5.78 us): fewer registers, twice the CTAs in flight.
    constexpr int R = 1;
    ptx::pdl_trigger();
    ptx::pdl_wait();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int row0 = warp * R;
    if (row0 >= rows) return;
    const int hv = h / 8;
    uint4 xp[R][NV], gp[NV], bp[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int vi = lane + 32 * i;
        if (vi < hv) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
                if (row0 + rr < rows) xp[rr][i] = *reinterpret_cast<const uint4*>(x + static_cast<size_t>(row0 + rr) * h + vi * 8);
            gp[i] = *reinterpret_cast<const uint4*>(g + vi * 8);
            bp[i] = *reinterpret_cast<const uint4*>(b + vi * 8);
        }
    }
    float v[R][NV][8];
    float sum[R], mu[R], var[R], rs[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
        sum[rr] = 0.0f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            if (lane + 32 * i < hv) {
                const uint32_t w[4] = {xp[rr][i].x, xp[rr][i].y, xp[rr][i].z, xp[rr][i].w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float2 f = ptx::unpack_bf16x2(w[t]);
                    v[rr][i][2 * t] = f.x;
                    v[rr][i][2 * t + 1] = f.y;
                    sum[rr] += f.x + f.y;
                }
            }
        }
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) mu[rr] = warp_sum(sum[rr]) / h;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
        var[rr] = 0.0f;
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if (lane + 32 * i < hv)
#pragma unroll
                for (int q = 0; q < 8; ++q) var[rr] += (v[rr][i][q] - mu[rr]) * (v[rr][i][q] - mu[rr]);
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) rs[rr] = rsqrtf(warp_sum(var[rr]) / h + 1e-5f);
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
        if (row0 + rr >= rows) break;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int vi = lane + 32 * i;
            if (vi < hv) {
                const uint32_t gw[4] = {gp[i].x, gp[i].y, gp[i].z, gp[i].w};
                const uint32_t bw[4] = {bp[i].x, bp[i].y, bp[i].z, bp[i].w};
                float o[8];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float2 gf = ptx::unpack_bf16x2(gw[t]), bf = ptx::unpack_bf16x2(bw[t]);
                    o[2 * t] = (v[rr][i][2 * t] - mu[rr]) * rs[rr] * gf.x + bf.x;
                    o[2 * t + 1] = (v[rr][i][2 * t + 1] - mu[rr]) * rs[rr] * gf.y + bf.y;
                }
                store8(y + static_cast<size_t>(row0 + rr) * h + vi * 8, o);
            }
        }
        if (lane == 0) {
            mean[row0 + rr] = mu[rr];
            rstd[row0 + rr] = rs[rr];
        }
    }
}

// Wide rows (h > 1024): a row is spread over WPR warps, each lane holding VPL 8-column
// vectors (vector k * 32 * WPR + warp * 32 + lane: coalesced), so a lane keeps 8 VPL
// values in registers instead of the one-warp kernel's h / 32 (h 1920: 60 -> 16, ~170 ->
// ~60 registers, four times the rows in flight).  The CTA's 8 warps work on 8 / WPR rows
// at a time and grid-stride over the rows with the next row's vectors loaded before the
// current row's two reductions (mean, then the centred variance -- exact two-pass, as the
// one-warp kernel), combined across a row's warps through SMEM under a named barrier.
template <int VPL, int WPR>
__global__ void __launch_bounds__(256) k_ln_fwd_wide(const bf16* __restrict__ x, const bf16* __restrict__ g,
                                                     const bf16* __restrict__ b, bf16* __restrict__ y,
                                                     float* __restrict__ mean, float* __restrict__ rstd, int rows,
                                                     int h) {
    constexpr int RPC = 8 / WPR;  // rows per CTA step
    __shared__ float red[2][2][RPC][WPR];  // [parity][stat][row group][warp]
    ptx::pdl_trigger();
    ptx::pdl_wait();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = warp / WPR, wi = warp % WPR;
    const int hv = h / 8;
    const float inv_h = 1.0f / static_cast<float>(h);
    int vi[VPL];
    bool ok[VPL];
    // packed fp32 pairs (FFMA2 / FADD2 / FMUL2) throughout: half the FP instructions
    unsigned long long g2[VPL][4], b2[VPL][4];
    uint4 cur[VPL], nxt[VPL];
    const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        vi[k] = k * 32 * WPR + wi * 32 + lane;
        ok[k] = vi[k] < hv;
        const uint4 gp = ok[k] ? *reinterpret_cast<const uint4*>(g + vi[k] * 8) : z4;
        const uint4 bp = ok[k] ? *reinterpret_cast<const uint4*>(b + vi[k] * 8) : z4;
        const uint32_t gw[4] = {gp.x, gp.y, gp.z, gp.w}, bw[4] = {bp.x, bp.y, bp.z, bp.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            g2[k][t] = ptx::bf2_to_f2(gw[t]);
            b2[k][t] = ptx::bf2_to_f2(bw[t]);
        }
    }
    const int step = gridDim.x * RPC;
    int r = blockIdx.x * RPC + grp;
    auto load = [&](int rr, uint4 (&dst)[VPL]) {
#pragma unroll
        for (int k = 0; k < VPL; ++k)
            dst[k] = (rr < rows && ok[k]) ? *reinterpret_cast<const uint4*>(x + static_cast<size_t>(rr) * h + vi[k] * 8)
                                          : z4;
    };
    load(r, cur);
    for (int it = 0; r - grp < rows; r += step, ++it) {
        load(r + step, nxt);  // the next row in flight during this row's reductions
        unsigned long long v[VPL][4];
        unsigned long long a1 = 0ull;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const uint32_t w[4] = {cur[k].x, cur[k].y, cur[k].z, cur[k].w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                v[k][t] = ptx::bf2_to_f2(w[t]);
                a1 = ptx::fadd2(a1, v[k][t]);
            }
        }
        const float2 f1 = ptx::f2_split(a1);
        const float s1 = warp_sum(f1.x + f1.y);
        float(*sl)[RPC][WPR] = red[it & 1];
        if (lane == 0) sl[0][grp][wi] = s1;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(WPR * 32) : "memory");
        float tot = 0.0f;
#pragma unroll
        for (int w = 0; w < WPR; ++w) tot += sl[0][grp][w];
        const float mu = tot * inv_h;
        const unsigned long long nmu2 = ptx::f2(-mu, -mu);
        unsigned long long a2 = 0ull;
#pragma unroll
        for (int k = 0; k < VPL; ++k)
            if (ok[k])
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const unsigned long long d = ptx::fadd2(v[k][t], nmu2);
                    a2 = ptx::ffma2(d, d, a2);
                }
        const float2 f2v = ptx::f2_split(a2);
        const float s2 = warp_sum(f2v.x + f2v.y);
        if (lane == 0) sl[1][grp][wi] = s2;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(WPR * 32) : "memory");
        float var = 0.0f;
#pragma unroll
        for (int w = 0; w < WPR; ++w) var += sl[1][grp][w];
        const float rs = rsqrtf(var * inv_h + 1e-5f);
        if (r < rows) {
            const unsigned long long rs2 = ptx::f2(rs, rs);
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                if (!ok[k]) continue;
                uint32_t ow[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {  // ((v - mu) rstd) g + b
                    const unsigned long long xh = ptx::fmul2(ptx::fadd2(v[k][t], nmu2), rs2);
                    ow[t] = ptx::f2_to_bf2(ptx::ffma2(xh, g2[k][t], b2[k][t]));
                }
                *reinterpret_cast<uint4*>(y + static_cast<size_t>(r) * h + vi[k] * 8) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
            }
            if (wi == 0 && lane == 0) {
                mean[r] = mu;
                rstd[r] = rs;
            }
        }
#pragma unroll
        for (int k = 0; k < VPL; ++k) cur[k] = nxt[k];
    }
}

// Fused LayerNorm backward.  Row part:
//   dx = rstd * (dxh - mean(dxh) - xh * mean(dxh * xh)) (+ dres),  dxh = dy * g
// Column part, accumulated in registers over the rows a thread visits and reduced
// over the CTA in SMEM -> one partial per CTA and statistic:
//   stat 0: sum_r dy * xh  (d gamma)     stat 1: sum_r dy  (d beta)
//   stat 2 (kSum): sum_r bf16(dx)  -- the bias gradient of the linear layer whose
//                  output gradient dx is (saves a separate pass over dx).
// A row is spread over a GROUP of wpr = ceil(h / 256) warps, one 8-column vector per
// lane, so each lane keeps only 8 columns of accumulators (24 registers) and a CTA of
// 768 threads works on G = 24 / wpr rows at a time, each group streaming its rows
// through an SMEM ring (k_ln_bwd below).  The two row sums are combined across the
// group's warps through SMEM (named barrier per group, fixed order: every warp of the
// group sees identical sums; deterministic).  dx may alias dy: a row is read (into
// the ring) before it is written, and the ring only fetches rows not yet written.
// Wide rows (h >= 1024) run with TWO vectors per lane (NVL = 2) in CTAs of 512 threads:
// a group of ceil(h / 512) warps per row, so the per-row shuffle / named-barrier / SMEM
// exchange work is spread over twice the elements (the kernel is issue-bound: ~300 SASS
// per warp-row at NVL = 1, h 1920).  P2BW_LN_BWD_NVL = 1 / 2 forces one layout.
template <int NVL>
constexpr int ln_bwd_threads() { return NVL == 1 ? 768 : 512; }  // 85 / 128 registers per thread

struct LnBwdShape {
    int nvl;  // 16-byte vectors per lane
    int wpr;  // warps per row
    int G;    // row groups per CTA
};

inline int ln_bwd_nvl(int h) {
    const char* env = std::getenv("P2BW_LN_BWD_NVL");  // read per call: tests switch it
    if (env && (env[0] == '1' || env[0] == '2')) return env[0] - '0';
    return h >= 1024 ? 2 : 1;
}

inline LnBwdShape ln_bwd_shape(int h, int nvl) {
    const int hv = h / 8;
    int wpr = (hv + 32 * nvl - 1) / (32 * nvl);
    if (wpr > 4) wpr = 8;  // instantiated group widths: 1, 2, 3, 4, 8
    int G = ((nvl == 1 ? ln_bwd_threads<1>() : ln_bwd_threads<2>()) / 32) / wpr;
    if (wpr > 1) G = std::min(G, 15);  // named barriers 1..15
    return {nvl, wpr, G};
}

// SMEM: red [G][h] fp32 | row-sum exchange [G][2][wpr][2] fp32 | row ring [G][NS] x
// {x, dy, dres} bf16 rows | ring barriers [G][NS].
inline size_t ln_bwd_fixed_bytes(int h, const LnBwdShape& sh) {
    const size_t f = (static_cast<size_t>(sh.G) * h + static_cast<size_t>(sh.G) * 2 * sh.wpr * 2) * sizeof(float);
    return (f + 127) & ~static_cast<size_t>(127);
}

// ring depth: G * 3 rows * h * 2 B ~ 24 * 256 * 6 B = 36 KB per slot for every h
// (G ~ 24 / ceil(h / 256)), so up to four slots fit beside the reduction buffer; the
// depth barely matters (the per-row reduction chain, not memory latency, bounds it)
// BERT-base (h 768, G 8 groups): 1 / 2 / 3 / 4 slots measured 16.1 / 16.0 / 16.2 / 16.5 us.
// Wide rows leave few groups per CTA (h 1920: G 3), so the ring deepens until ~16 rows
// per SM are in flight (Little's law at ~6.5 TB/s and ~1 us of latency: ~45 KB per SM).
inline int ln_bwd_ring_depth(int h, const LnBwdShape& sh) {
    const int G = sh.G;
    int ns = std::max(2, std::min(8, (16 + G - 1) / G));
    const size_t per_slot = static_cast<size_t>(G) * (3ull * h * 2 + 8);
    while (ns > 2 && ln_bwd_fixed_bytes(h, sh) + ns * per_slot > 200u * 1024u) --ns;
    return ns;
}

inline size_t ln_bwd_smem_bytes(int h, const LnBwdShape& sh) {
    return ln_bwd_fixed_bytes(h, sh) + static_cast<size_t>(sh.G) * ln_bwd_ring_depth(h, sh) * (3ull * h * 2 + 8);
}

__device__ __forceinline__ void group_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// LayerNorm backward + residual, persistent: 148 CTAs x G row groups of wpr warps (one
// row per group at a time, lane = NVL 8-column vectors, wpr * 32 columns apart).  Each
// group streams its rows (r, r + G * grid, ...) through an NS-deep SMEM ring filled by
// 1D bulk copies (x, dy, dres rows: NS rows in flight per group without holding them in
// registers -- the register-prefetch version kept one row in flight and ran at ~2.7 TB/s).
//   dx = rstd * (g*dy - mean(g*dy) - xhat * mean(g*dy*xhat)) + dres
// plus per-CTA partial column sums of dy*xhat (dgamma), dy (dbeta) and, kSum, bf16(dx).
template <bool kSum, int wpr, bool kRes, int NVL>
__global__ void __launch_bounds__(ln_bwd_threads<NVL>(), 1)
    k_ln_bwd(const bf16* __restrict__ dy, const bf16* __restrict__ x, const float* __restrict__ mean,
             const float* __restrict__ rstd, const bf16* __restrict__ g, const bf16* __restrict__ dres,
             bf16* dx, int rows, int h, int G, int fixed_bytes, int NS, float* __restrict__ part) {
    extern __shared__ __align__(128) uint8_t ln_raw[];
    float* ln_smem = reinterpret_cast<float*>(ln_raw);
    ptx::pdl_trigger();
    ptx::pdl_wait();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = warp / wpr, wi = warp % wpr;
    const int hv = h / 8;
    int vi[NVL];  // my 8-column vectors of every row
    bool act[NVL];
#pragma unroll
    for (int v = 0; v < NVL; ++v) {
        vi[v] = wi * 32 + lane + v * wpr * 32;
        act[v] = grp < G && vi[v] < hv;
    }
    constexpr bool has_res = kRes;  // residual gradient added to dx (compile-time: no per-row branches)
    const float inv_h = 1.0f / static_cast<float>(h);
    float* xs = ln_smem + static_cast<size_t>(G) * h;
    const int row_bytes = h * 2;
    const int stage_bytes = 3 * row_bytes;
    uint8_t* ring = ln_raw + fixed_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(G) * NS * stage_bytes);
    const int stride = gridDim.x * G;
    const int r0 = blockIdx.x * G + grp;
    const bool leader = grp < G && wi == 0 && lane == 0;
    uint8_t* my_ring = ring + static_cast<size_t>(grp) * NS * stage_bytes;
    uint64_t* my_bars = bars + grp * NS;
    auto issue = [&](int rr, int slot) {  // row rr into ring slot `slot`
        if (rr >= rows) return;
        uint64_t* bar = &my_bars[slot];
        uint8_t* dst = my_ring + slot * stage_bytes;
        const size_t o = static_cast<size_t>(rr) * h;
        ptx::mbar_arrive_expect_tx(bar, (has_res ? 3 : 2) * row_bytes);
        ptx::bulk_load_1d(dst, x + o, row_bytes, bar);
        ptx::bulk_load_1d(dst + row_bytes, dy + o, row_bytes, bar);
        if (has_res) ptx::bulk_load_1d(dst + 2 * row_bytes, dres + o, row_bytes, bar);
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < G * NS; ++i) ptx::mbar_init(&bars[i], 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (leader)
        for (int i = 0; i < NS; ++i) issue(r0 + i * stride, i);
    // the row math runs on packed fp32 pairs (FFMA2 / FADD2 / FMUL2): the kernel is issue-
    // bound, so half the FP instructions per element is what moves it
    unsigned long long g2[NVL][4];
#pragma unroll
    for (int v = 0; v < NVL; ++v) {
        g2[v][0] = g2[v][1] = g2[v][2] = g2[v][3] = 0ull;
        if (act[v]) {
            const uint4 gp = *reinterpret_cast<const uint4*>(g + vi[v] * 8);
            g2[v][0] = ptx::bf2_to_f2(gp.x), g2[v][1] = ptx::bf2_to_f2(gp.y), g2[v][2] = ptx::bf2_to_f2(gp.z),
            g2[v][3] = ptx::bf2_to_f2(gp.w);
        }
    }
    unsigned long long ag[NVL][4], ab[NVL][4], as[NVL][4];  // (0.0f, 0.0f) pairs
#pragma unroll
    for (int v = 0; v < NVL; ++v)
#pragma unroll
        for (int t = 0; t < 4; ++t) ag[v][t] = ab[v][t] = as[v][t] = 0ull;
    const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
    int r = r0;
    float mu = 0.0f, rs = 0.0f;
    if (grp < G && r < rows) {
        mu = mean[r];
        rs = rstd[r];
    }
    int slot = 0;
    uint32_t phase = 0;
    for (int it = 0; grp < G && r < rows; r += stride, ++it) {
        float nmu = 0.0f, nrs = 0.0f;
        if (r + stride < rows) {
            nmu = mean[r + stride];
            nrs = rstd[r + stride];
        }
        ptx::mbar_wait(&my_bars[slot], phase);
        const uint8_t* src = my_ring + slot * stage_bytes;
        uint4 rp[NVL];
        unsigned long long xh[NVL][4], dg[NVL][4];
        float s1, s2;
        {
            const unsigned long long rs2 = ptx::f2(rs, rs), sh2 = ptx::f2(-mu * rs, -mu * rs);
            unsigned long long a1 = 0ull, a2 = 0ull;
#pragma unroll
            for (int v = 0; v < NVL; ++v) {
                uint4 xp = z4, dp = z4;
                rp[v] = z4;
                if (act[v]) {
                    xp = *reinterpret_cast<const uint4*>(src + vi[v] * 16);
                    dp = *reinterpret_cast<const uint4*>(src + row_bytes + vi[v] * 16);
                    if (has_res) rp[v] = *reinterpret_cast<const uint4*>(src + 2 * row_bytes + vi[v] * 16);
                }
                const uint32_t xw[4] = {xp.x, xp.y, xp.z, xp.w}, dw[4] = {dp.x, dp.y, dp.z, dp.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const unsigned long long x2 = ptx::bf2_to_f2(xw[t]), d2 = ptx::bf2_to_f2(dw[t]);
                    xh[v][t] = ptx::ffma2(x2, rs2, sh2);  // (x - mu) rstd
                    dg[v][t] = ptx::fmul2(d2, g2[v][t]);
                    ag[v][t] = ptx::ffma2(d2, xh[v][t], ag[v][t]);  // inactive lanes hold zero data
                    ab[v][t] = ptx::fadd2(ab[v][t], d2);
                    a1 = ptx::fadd2(a1, dg[v][t]);
                    a2 = ptx::ffma2(dg[v][t], xh[v][t], a2);
                }
            }
            const float2 f1 = ptx::f2_split(a1), f2v = ptx::f2_split(a2);
            s1 = f1.x + f1.y;
            s2 = f2v.x + f2v.y;
        }
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        if constexpr (wpr > 1) {
            float* sl = xs + (static_cast<size_t>(grp) * 2 + (it & 1)) * wpr * 2;
            if (lane == 0) *reinterpret_cast<float2*>(sl + wi * 2) = make_float2(s1, s2);
            group_bar(1 + grp, wpr * 32);  // also: every warp of the group has read the slot
            s1 = 0.0f;
            s2 = 0.0f;
#pragma unroll
            for (int w = 0; w < wpr; ++w) {
                const float2 p = *reinterpret_cast<const float2*>(sl + w * 2);
                s1 += p.x;
                s2 += p.y;
            }
        } else {
            __syncwarp();
        }
        if (leader) issue(r + NS * stride, slot);  // refill the slot just read
        if (++slot == NS) {
            slot = 0;
            phase ^= 1;
        }
        // dx = rstd (dg - m1 - xh m2) = dg rstd + xh (-rstd m2) + (-rstd m1)
        const float c1 = -rs * s1 * inv_h, c2 = -rs * s2 * inv_h;
        const unsigned long long rs2 = ptx::f2(rs, rs), c12 = ptx::f2(c1, c1), c22 = ptx::f2(c2, c2);
#pragma unroll
        for (int v = 0; v < NVL; ++v) {
            if (act[v]) {
                const uint32_t rw[4] = {rp[v].x, rp[v].y, rp[v].z, rp[v].w};
                uint32_t ow[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    unsigned long long o = ptx::ffma2(xh[v][t], c22, ptx::ffma2(dg[v][t], rs2, c12));
                    if (has_res) o = ptx::fadd2(o, ptx::bf2_to_f2(rw[t]));
                    ow[t] = ptx::f2_to_bf2(o);
                    if constexpr (kSum) as[v][t] = ptx::fadd2(as[v][t], ptx::bf2_to_f2(ow[t]));  // what the next GEMM reads
                }
                *reinterpret_cast<uint4*>(dx + static_cast<size_t>(r) * h + vi[v] * 8) =
                    make_uint4(ow[0], ow[1], ow[2], ow[3]);
            }
        }
        mu = nmu;
        rs = nrs;
    }
    // CTA reduction over the row groups, one statistic at a time, fixed order
    for (int st = 0; st < (kSum ? 3 : 2); ++st) {
        __syncthreads();
#pragma unroll
        for (int v = 0; v < NVL; ++v) {
            if (act[v]) {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float2 q = ptx::f2_split(st == 0 ? ag[v][t] : (st == 1 ? ab[v][t] : as[v][t]));
                    *reinterpret_cast<float2*>(ln_smem + static_cast<size_t>(grp) * h + vi[v] * 8 + 2 * t) = q;
                }
            }
        }
        __syncthreads();
        for (int c = threadIdx.x; c < h; c += blockDim.x) {
            float sum = 0.0f;
            for (int gg = 0; gg < G; ++gg) sum += ln_smem[static_cast<size_t>(gg) * h + c];
            part[(static_cast<size_t>(st) * gridDim.x + blockIdx.x) * h + c] = sum;
        }
    }
}

int ln_bwd_blocks(int rows) { return std::max(1, std::min(148, (rows + 15) / 16)); }

// ---- softmax cross-entropy ------------------------------------------------------------

__global__ void __launch_bounds__(256) k_softmax_xent(bf16* __restrict__ logits, const int* __restrict__ targets,
                                                      int vocab, int vp, float grad_scale,
                                                      float* __restrict__ row_loss) {
    __shared__ float sm[8], ss[8];
    __shared__ float s_lse, s_tgt;
    const int row = blockIdx.x;
    bf16* lr = logits + static_cast<size_t>(row) * vp;
    const int tgt = targets[row];
    if (threadIdx.x == 0) s_tgt = __bfloat162float(lr[tgt]);
    float m = -INFINITY, sum = 0.0f;
    const int nv = vp / 8;
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        float x[8];
        load8(lr + v * 8, x);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (v * 8 + q < vocab) {
                const float t = x[q] * kLog2e;
                if (t > m) {
                    sum = sum * exp2f(m - t) + 1.0f;
                    m = t;
                } else {
                    sum += exp2f(t - m);
                }
            }
        }
    }
    // warp-combine (m, sum)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, sum, o);
        const float nm = fmaxf(m, om);
        sum = (m == -INFINITY ? 0.0f : sum * exp2f(m - nm)) + (om == -INFINITY ? 0.0f : os * exp2f(om - nm));
        m = nm;
    }
    if ((threadIdx.x & 31) == 0) {
        sm[threadIdx.x >> 5] = m;
        ss[threadIdx.x >> 5] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = -INFINITY, S = 0.0f;
        for (int w = 0; w < 8; ++w) {
            const float nm = fmaxf(M, sm[w]);
            S = (M == -INFINITY ? 0.0f : S * exp2f(M - nm)) + (sm[w] == -INFINITY ? 0.0f : ss[w] * exp2f(sm[w] - nm));
            M = nm;
        }
        s_lse = (M + log2f(S)) / kLog2e;
        row_loss[row] = s_lse - s_tgt;
    }
    __syncthreads();
    const float lse2 = s_lse * kLog2e;
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        float x[8];
        load8(lr + v * 8, x);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int c = v * 8 + q;
            const float p = c < vocab ? exp2f(x[q] * kLog2e - lse2) : 0.0f;
            x[q] = (p - (c == tgt ? 1.0f : 0.0f)) * grad_scale;
        }
        store8(lr + v * 8, x);
    }
}

// Register-resident variant (vp <= 256 * 8 * NVT): the row is read from HBM once into
// packed bf16 registers; max, then sum of exp2, then the gradient are computed from
// registers (the two-pass kernel above reads every row twice).  Same row loss and
// gradient definitions; the max is exact, so only the summation order differs.
// bf16x2 -> 2 x f32 that the compiler may not hoist or merge across the passes below
// (a hoisted fp32 copy of the row would double its register footprint)
__device__ __forceinline__ float2 unpack_bf16x2_opaque(uint32_t w) {
    uint32_t lo, hi;
    asm volatile("shl.b32 %0, %1, 16;" : "=r"(lo) : "r"(w));
    asm volatile("and.b32 %0, %1, 0xffff0000;" : "=r"(hi) : "r"(w));
    return make_float2(__uint_as_float(lo), __uint_as_float(hi));
}

template <int NVT>
__global__ void __launch_bounds__(256, NVT <= 25 ? 2 : 1) k_softmax_xent_reg(bf16* __restrict__ logits, const int* __restrict__ targets,
                                                          int vocab, int vp, float grad_scale,
                                                          float* __restrict__ row_loss) {
    __shared__ float red[8];
    __shared__ float s_b;
    const int row = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    bf16* lr = logits + static_cast<size_t>(row) * vp;
    const int tgt = targets[row];
    const int nv = vp / 8;
    constexpr uint32_t kNegInf2 = 0xFF80FF80u;  // two bf16 -inf: padded columns drop out of every pass
    uint4 u[NVT];
#pragma unroll
    for (int k = 0; k < NVT; ++k) {
        const int v = threadIdx.x + 256 * k;
        u[k] = v < nv ? *reinterpret_cast<const uint4*>(lr + v * 8) : make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
        if (v < nv && v * 8 + 8 > vocab) {  // the vector that straddles the vocabulary end
            uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
            for (int q = 0; q < 8; ++q)
                if (v * 8 + q >= vocab) w[q / 2] = (q & 1) ? ((w[q / 2] & 0xFFFFu) | 0xFF800000u) : ((w[q / 2] & 0xFFFF0000u) | 0xFF80u);
            u[k] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    const float t_tgt = __bfloat162float(lr[tgt]) * kLog2e;
    auto block_reduce = [&](float x, bool is_max) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float y = __shfl_xor_sync(0xffffffffu, x, o);
            x = is_max ? fmaxf(x, y) : x + y;
        }
        if (lane == 0) red[warp] = x;
        __syncthreads();
        if (threadIdx.x == 0) {
            float r = red[0];
            for (int w = 1; w < 8; ++w) r = is_max ? fmaxf(r, red[w]) : r + red[w];
            s_b = r;
        }
        __syncthreads();
        const float r = s_b;
        __syncthreads();  // red / s_b reused by the next reduction
        return r;
    };
    // pass 1: row max
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < NVT; ++k) {
        const uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float2 f = unpack_bf16x2_opaque(w[t]);
            m = fmaxf(m, fmaxf(f.x, f.y));
        }
    }
    const float M = block_reduce(m, true) * kLog2e;
    // pass 2: sum of exp2(t - M)
    float sum = 0.0f;
#pragma unroll
    for (int k = 0; k < NVT; ++k) {
        const uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float2 f = unpack_bf16x2_opaque(w[t]);
            sum += exp2f(fmaf(f.x, kLog2e, -M)) + exp2f(fmaf(f.y, kLog2e, -M));
        }
    }
    const float S = block_reduce(sum, false);
    const float lse2 = M + log2f(S);
    if (threadIdx.x == 0) row_loss[row] = (lse2 - t_tgt) / kLog2e;
    // pass 3: dlogits = (softmax - onehot) * grad_scale, in place
#pragma unroll
    for (int k = 0; k < NVT; ++k) {
        const int v = threadIdx.x + 256 * k;
        if (v < nv) {
            const uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
            float x[8];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float2 f = unpack_bf16x2_opaque(w[t]);
                x[2 * t] = exp2f(fmaf(f.x, kLog2e, -lse2)) * grad_scale;
                x[2 * t + 1] = exp2f(fmaf(f.y, kLog2e, -lse2)) * grad_scale;
            }
            const int d = tgt - v * 8;
            if (d >= 0 && d < 8) x[d] -= grad_scale;
            store8(lr + v * 8, x);
        }
    }
}

__global__ void k_sum_scaled(const float* __restrict__ in, int n, float scale, float* __restrict__ out) {
    __shared__ float red[256];
    float acc = 0.0f;
    for (int i = threadIdx.x; i < n; i += 256) acc += in[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0] * scale;
}

// ---- optimizer / init -----------------------------------------------------------------

__global__ void k_sgd(float4* __restrict__ w, float4* __restrict__ v, const float4* __restrict__ g,
                      uint2* __restrict__ out, size_t n4, float inv_count, float lr, float beta) {
    const float damp = 1.0f - beta;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const float4 gg = g[i];
        float4 vv = v[i], ww = w[i];
        vv.x = beta * vv.x + damp * (gg.x * inv_count);
        vv.y = beta * vv.y + damp * (gg.y * inv_count);
        vv.z = beta * vv.z + damp * (gg.z * inv_count);
        vv.w = beta * vv.w + damp * (gg.w * inv_count);
        ww.x -= lr * vv.x;
        ww.y -= lr * vv.y;
        ww.z -= lr * vv.z;
        ww.w -= lr * vv.w;
        v[i] = vv;
        w[i] = ww;
        out[i] = make_uint2(ptx::pack_bf16x2(ww.x, ww.y), ptx::pack_bf16x2(ww.z, ww.w));
    }
}

// Adam with bias correction: g = grad / count; m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
// w -= lr * (m / c1) / (sqrt(v / c2) + eps), c1 = 1 - b1^t, c2 = 1 - b2^t.
__global__ void k_adam(float4* __restrict__ w, float4* __restrict__ m1, float4* __restrict__ m2,
                       const float4* __restrict__ g, uint2* __restrict__ out, size_t n4, float inv_count, float lr,
                       float b1, float b2, float eps, float inv_c1, float inv_c2) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const float4 gg = g[i];
        float4 a = m1[i], b = m2[i], ww = w[i];
        const float gv[4] = {gg.x * inv_count, gg.y * inv_count, gg.z * inv_count, gg.w * inv_count};
        float* ap = &a.x;
        float* bp = &b.x;
        float* wp = &ww.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            ap[e] = b1 * ap[e] + (1.0f - b1) * gv[e];
            bp[e] = b2 * bp[e] + (1.0f - b2) * gv[e] * gv[e];
            wp[e] -= lr * (ap[e] * inv_c1) / (sqrtf(bp[e] * inv_c2) + eps);
        }
        m1[i] = a;
        m2[i] = b;
        w[i] = ww;
        out[i] = make_uint2(ptx::pack_bf16x2(ww.x, ww.y), ptx::pack_bf16x2(ww.z, ww.w));
    }
}

// The AllReduce fused into the optimizer over peer memory (tkernels.h ReplicaShard).
struct ShardArgs {
    const float4* g[kMaxReplicas];
    float4* w[kMaxReplicas];
    uint2* out[kMaxReplicas];
};

template <bool kAdam>
__global__ void k_opt_replicas(ShardArgs a, int nrep, int rank, float4* __restrict__ s1, float4* __restrict__ s2,
                               size_t lo, size_t hi, float inv_count, float lr, float b1, float b2, float eps,
                               float inv_c1, float inv_c2) {
    for (size_t i = lo + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < hi;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        float4 gq[kMaxReplicas];
#pragma unroll
        for (int q = 0; q < kMaxReplicas; ++q)  // every replica's loads in flight together
            if (q < nrep) gq[q] = a.g[q][i];
        float4 gg = gq[0];
#pragma unroll
        for (int q = 1; q < kMaxReplicas; ++q)
            if (q < nrep) gg.x += gq[q].x, gg.y += gq[q].y, gg.z += gq[q].z, gg.w += gq[q].w;
        float4 ww = a.w[rank][i], m = s1[i];
        float* mp = &m.x;
        float* wp = &ww.x;
        const float gv[4] = {gg.x * inv_count, gg.y * inv_count, gg.z * inv_count, gg.w * inv_count};
        if constexpr (kAdam) {
            float4 v = s2[i];
            float* vp = &v.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                mp[e] = b1 * mp[e] + (1.0f - b1) * gv[e];
                vp[e] = b2 * vp[e] + (1.0f - b2) * gv[e] * gv[e];
                wp[e] -= lr * (mp[e] * inv_c1) / (sqrtf(vp[e] * inv_c2) + eps);
            }
            s2[i] = v;
        } else {
            const float damp = 1.0f - b1;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                mp[e] = b1 * mp[e] + damp * gv[e];
                wp[e] -= lr * mp[e];
            }
        }
        s1[i] = m;
        const uint2 o = make_uint2(ptx::pack_bf16x2(ww.x, ww.y), ptx::pack_bf16x2(ww.z, ww.w));
#pragma unroll
        for (int q = 0; q < kMaxReplicas; ++q)
            if (q < nrep) {
                a.w[q][i] = ww;
                a.out[q][i] = o;
            }
    }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__global__ void k_init_uniform(float* __restrict__ w, size_t n, uint64_t key, float hw) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = mix64(key + i * 0xd1b54a32d192ed03ULL);
        const double u = static_cast<double>(r >> 11) * (1.0 / 9007199254740992.0);
        w[i] = static_cast<float>((u - 0.5) * 2.0 * hw);
    }
}

__global__ void k_fill(float* __restrict__ w, size_t n, float v) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        w[i] = v;
}

__global__ void k_cast_f2b(const float* __restrict__ in, bf16* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = __float2bfloat16_rn(in[i]);
}

__global__ void k_cast_b2f(const bf16* __restrict__ in, float* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = __bfloat162float(in[i]);
}

__global__ void k_gather_rows(const bf16* __restrict__ in, const int* __restrict__ idx, bf16* __restrict__ out,
                              int rows, int h, int scatter) {
    const int hv = h / 8;
    const size_t total = static_cast<size_t>(rows) * hv;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / hv), c = static_cast<int>(i % hv) * 8;
        const size_t src = scatter ? static_cast<size_t>(r) : static_cast<size_t>(idx[r]);
        const size_t dst = scatter ? static_cast<size_t>(idx[r]) : static_cast<size_t>(r);
        *reinterpret_cast<uint4*>(out + dst * h + c) = *reinterpret_cast<const uint4*>(in + src * h + c);
    }
}

}  // namespace

// ---- host wrappers ---------------------------------------------------------------------
// Each wrapper opens a prof::Scope with its algorithmic HBM bytes (reads + writes
// of the tensors it must touch once) for the roofline report.

void embed_fwd(const int* ids, const bf16* tok, const bf16* pos, bf16* x0, int tokens, int seq, int h,
               cudaStream_t s) {
    const double th = static_cast<double>(tokens) * h;
    prof::Scope scope("embed_fwd", 0.0, 6.0 * th + 4.0 * tokens, 1, s);
    k_embed_fwd<<<grid_for(static_cast<size_t>(tokens) * h / 8, 256), 256, 0, s>>>(ids, tok, pos, x0, tokens,
                                                                                  seq, h);
    check_cuda(cudaGetLastError(), "embed_fwd");
}

void embed_bwd(const int* ids, const bf16* dx0, float* dtok, float* dpos, int tokens, int seq, int h,
               bool overwrite_pos, cudaStream_t s) {
    const double th = static_cast<double>(tokens) * h;
    prof::Scope scope("embed_bwd", 0.0, 2.0 * th * 2 + 8.0 * th + 8.0 * seq * h, 2, s);
    k_embed_bwd_tok<<<grid_for(static_cast<size_t>(tokens) * h / 8, 256), 256, 0, s>>>(ids, dx0, dtok, tokens, h);
    k_embed_bwd_pos<<<grid_for(static_cast<size_t>(seq) * h / 8, 128), 128, 0, s>>>(
        dx0, dpos, tokens / seq, seq, h, overwrite_pos ? 1 : 0);
    check_cuda(cudaGetLastError(), "embed_bwd");
}

void layernorm_fwd(const bf16* x, const bf16* g, const bf16* b, bf16* y, float* mean, float* rstd, int rows,
                   int h, cudaStream_t s) {
    if (h % 8 != 0 || h > 2048) throw Error("layernorm: hidden must be a multiple of 8 and <= 2048");
    prof::Scope scope("layernorm_fwd", 0.0, 4.0 * rows * h + 8.0 * rows, 1, s);
    const int nv = (h / 8 + 31) / 32;
    if (nv > 4) {  // h > 1024: a row over WPR warps of two vectors per lane
        const int wpr = (h / 8 + 63) / 64;
        const int rpc = wpr <= 2 ? 8 / 2 : (wpr <= 4 ? 2 : 1);
        const int grid = std::max(1, std::min((rows + rpc - 1) / rpc, 148 * 8));
        if (wpr <= 2)
            launch_pdl(k_ln_fwd_wide<2, 2>, dim3(grid), dim3(256), 0, s, "k_ln_fwd", x, g, b, y, mean, rstd, rows, h);
        else if (wpr <= 4)
            launch_pdl(k_ln_fwd_wide<2, 4>, dim3(grid), dim3(256), 0, s, "k_ln_fwd", x, g, b, y, mean, rstd, rows, h);
        else
            launch_pdl(k_ln_fwd_wide<2, 8>, dim3(grid), dim3(256), 0, s, "k_ln_fwd", x, g, b, y, mean, rstd, rows, h);
        check_cuda(cudaGetLastError(), "layernorm_fwd");
        return;
    }
    const int grid = (rows + 7) / 8;  // 8 warps x 1 row
    switch (nv) {
        case 1: launch_pdl(k_ln_fwd<1>, dim3(grid), dim3(256), 0, s, "k_ln_fwd", x, g, b, y, mean, rstd, rows, h); break;
        case 2: launch_pdl(k_ln_fwd<2>, dim3(grid), dim3(256), 0, s, "k_ln_fwd", x, g, b, y, mean, rstd, rows, h); break;
        case 3: launch_pdl(k_ln_fwd<3>, dim3(grid), dim3(256), 0, s, "k_ln_fwd", x, g, b, y, mean, rstd, rows, h); break;
        case 4: launch_pdl(k_ln_fwd<4>, dim3(grid), dim3(256), 0, s, "k_ln_fwd", x, g, b, y, mean, rstd, rows, h); break;
        default: launch_pdl(k_ln_fwd<8>, dim3(grid), dim3(256), 0, s, "k_ln_fwd", x, g, b, y, mean, rstd, rows, h); break;
    }
    check_cuda(cudaGetLastError(), "layernorm_fwd");
}

size_t layernorm_bwd_scratch_floats(int rows, int h) { return static_cast<size_t>(ln_bwd_blocks(rows)) * h * 3; }

template <bool kSum, int NVL>
void launch_ln_bwd_nvl(int grid, const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* g,
                       const bf16* dres, bf16* dx, int rows, int h, float* part, cudaStream_t s) {
    const LnBwdShape sh = ln_bwd_shape(h, NVL);
    const size_t smem = ln_bwd_smem_bytes(h, sh);
    auto go = [&](auto kern) {
        if (smem > 48 * 1024)
            check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                       "cudaFuncSetAttribute(ln bwd smem)");
        launch_pdl(kern, dim3(grid), dim3(ln_bwd_threads<NVL>()), smem, s, "k_ln_bwd", dy, x, mean, rstd, g, dres, dx,
                   rows, h, sh.G, static_cast<int>(ln_bwd_fixed_bytes(h, sh)), ln_bwd_ring_depth(h, sh), part);
    };
    switch (sh.wpr) {
        case 1: dres ? go(k_ln_bwd<kSum, 1, true, NVL>) : go(k_ln_bwd<kSum, 1, false, NVL>); break;
        case 2: dres ? go(k_ln_bwd<kSum, 2, true, NVL>) : go(k_ln_bwd<kSum, 2, false, NVL>); break;
        case 3: dres ? go(k_ln_bwd<kSum, 3, true, NVL>) : go(k_ln_bwd<kSum, 3, false, NVL>); break;
        case 4: dres ? go(k_ln_bwd<kSum, 4, true, NVL>) : go(k_ln_bwd<kSum, 4, false, NVL>); break;
        default:
            if constexpr (NVL == 1) dres ? go(k_ln_bwd<kSum, 8, true, 1>) : go(k_ln_bwd<kSum, 8, false, 1>);
            else throw Error("layernorm_bwd: no 8-warp group at two vectors per lane");
            break;
    }
}

template <bool kSum>
void launch_ln_bwd(int grid, const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* g,
                   const bf16* dres, bf16* dx, int rows, int h, float* part, cudaStream_t s) {
    if (ln_bwd_nvl(h) == 2) launch_ln_bwd_nvl<kSum, 2>(grid, dy, x, mean, rstd, g, dres, dx, rows, h, part, s);
    else launch_ln_bwd_nvl<kSum, 1>(grid, dy, x, mean, rstd, g, dres, dx, rows, h, part, s);
}

void layernorm_bwd(const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* g,
                   const bf16* dres, bf16* dx, float* dg, float* db, bool overwrite, int rows, int h,
                   float* scratch, cudaStream_t s, float* dsum) {
    if (h % 8 != 0 || h > 2048) throw Error("layernorm: hidden must be a multiple of 8 and <= 2048");
    prof::Scope scope("layernorm_bwd", 0.0, (dres ? 8.0 : 6.0) * rows * h + 8.0 * rows, 2, s);
    const int grid = ln_bwd_blocks(rows);
    if (dsum) launch_ln_bwd<true>(grid, dy, x, mean, rstd, g, dres, dx, rows, h, scratch, s);
    else launch_ln_bwd<false>(grid, dy, x, mean, rstd, g, dres, dx, rows, h, scratch, s);
    ReduceOut o{{dg, db, dsum}};
    launch_pdl(k_reduce_parts, dim3((h + 7) / 8, dsum ? 3 : 2), dim3(256), 0, s, "k_reduce_parts",
               static_cast<const float*>(scratch), grid, h, o, overwrite ? 1 : 0);
    check_cuda(cudaGetLastError(), "layernorm_bwd");
}

void reduce_partials(const float* part, int parts, int n, float* out, bool overwrite, cudaStream_t s) {
    reduce_parts(part, parts, n, out, overwrite, s);
    check_cuda(cudaGetLastError(), "reduce_partials");
}

size_t colsum_scratch_floats(int rows, int n) { return static_cast<size_t>(colsum_row_blocks(rows, n)) * n; }

void colsum_bf16(const bf16* x, int rows, int n, int ld, float* out, bool overwrite, float* scratch,
                 cudaStream_t s) {
    if (n % 8 != 0) throw Error("colsum: columns must be a multiple of 8");
    prof::Scope scope("bias_grad", 0.0, 2.0 * rows * n + 8.0 * n, 2, s);
    const int rb = colsum_row_blocks(rows, n);
    const int rpb = (rows + rb - 1) / rb;
    launch_pdl(k_colstats<false>, dim3((n + 255) / 256, rb), dim3(256), 0, s, "k_colstats", x,
               static_cast<const bf16*>(nullptr), static_cast<const float*>(nullptr),
               static_cast<const float*>(nullptr), rows, n, ld, rpb, scratch, static_cast<float*>(nullptr));
    reduce_parts(scratch, rb, n, out, overwrite, s);
    check_cuda(cudaGetLastError(), "colsum");
}

bool xent_two_per_sm() {  // P2BW_XENT_2CTA=0: the one-CTA-per-SM <32> instantiation (A/B knob)
    static const bool on = [] {
        const char* e = std::getenv("P2BW_XENT_2CTA");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return on;
}

void softmax_xent(bf16* logits, const int* targets, int rows, int vocab, int vp, float grad_scale,
                  float* row_loss, cudaStream_t s) {
    if (vp % 8 != 0) throw Error("softmax_xent: padded vocab must be a multiple of 8");
    prof::Scope scope("softmax_xent", 0.0, 4.0 * rows * static_cast<double>(vp) + 8.0 * rows, 1, s);
    const int nvt = (vp / 8 + 255) / 256;  // 16-byte vectors per thread for a register-resident row
    if (nvt <= 16) k_softmax_xent_reg<16><<<rows, 256, 0, s>>>(logits, targets, vocab, vp, grad_scale, row_loss);
    // <= 25 vectors per thread (V <= 51200): <= 128 registers, so two rows share an SM and
    // one row's exponentials overlap the other's loads (one CTA per SM left the memory pipe
    // idle during the exp passes: 548 us per 8192-row GPT-2.2B head at 3.1 TB/s)
    else if (nvt <= 25 && xent_two_per_sm()) k_softmax_xent_reg<25><<<rows, 256, 0, s>>>(logits, targets, vocab, vp, grad_scale, row_loss);
    else if (nvt <= 32) k_softmax_xent_reg<32><<<rows, 256, 0, s>>>(logits, targets, vocab, vp, grad_scale, row_loss);
    else k_softmax_xent<<<rows, 256, 0, s>>>(logits, targets, vocab, vp, grad_scale, row_loss);
    check_cuda(cudaGetLastError(), "softmax_xent");
}

void sum_scaled(const float* row_loss, int rows, float scale, float* loss_out, cudaStream_t s) {
    prof::Scope scope("loss_sum", 0.0, 4.0 * rows, 1, s);
    k_sum_scaled<<<1, 256, 0, s>>>(row_loss, rows, scale, loss_out);
    check_cuda(cudaGetLastError(), "sum_scaled");
}

void sgd_momentum_update(float* master, float* vel, const float* grad, bf16* out_bf16, size_t n,
                         float inv_count, float lr, float beta, cudaStream_t s) {
    if (n % 4 != 0) throw Error("optimizer: parameter count must be a multiple of 4");
    // reads w, v, g (12 B) + writes w, v (8 B) + bf16 copy (2 B) = 22 B/param
    prof::Scope scope("optimizer", 0.0, 22.0 * static_cast<double>(n), 1, s);
    k_sgd<<<grid_for(n / 4, 256), 256, 0, s>>>(reinterpret_cast<float4*>(master), reinterpret_cast<float4*>(vel),
                                              reinterpret_cast<const float4*>(grad),
                                              reinterpret_cast<uint2*>(out_bf16), n / 4, inv_count, lr, beta);
    check_cuda(cudaGetLastError(), "sgd_momentum_update");
}

void adam_update(float* master, float* m1, float* m2, const float* grad, bf16* out_bf16, size_t n, float inv_count,
                 float lr, float b1, float b2, float eps, int step, cudaStream_t s) {
    if (n % 4 != 0) throw Error("optimizer: parameter count must be a multiple of 4");
    // reads w, m, v, g (16 B) + writes w, m, v (12 B) + bf16 copy (2 B) = 30 B/param
    prof::Scope scope("optimizer", 0.0, 30.0 * static_cast<double>(n), 1, s);
    const float inv_c1 = static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(b1), step)));
    const float inv_c2 = static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(b2), step)));
    k_adam<<<grid_for(n / 4, 256), 256, 0, s>>>(reinterpret_cast<float4*>(master), reinterpret_cast<float4*>(m1),
                                               reinterpret_cast<float4*>(m2), reinterpret_cast<const float4*>(grad),
                                               reinterpret_cast<uint2*>(out_bf16), n / 4, inv_count, lr, b1, b2, eps,
                                               inv_c1, inv_c2);
    check_cuda(cudaGetLastError(), "adam_update");
}

namespace {
template <bool kAdam>
void opt_replicas(const ReplicaShard& r, float* s1, float* s2, size_t n, float inv_count, float lr, float b1,
                  float b2, float eps, float inv_c1, float inv_c2, cudaStream_t s) {
    if (n % 4 != 0) throw Error("optimizer: parameter count must be a multiple of 4");
    if (r.w < 1 || r.w > kMaxReplicas || r.rank < 0 || r.rank >= r.w)
        throw Error("replica update: bad width / rank");
    ShardArgs a{};
    for (int q = 0; q < r.w; ++q) {
        if (!r.grad[q] || !r.master[q] || !r.version[q]) throw Error("replica update: missing peer buffer");
        a.g[q] = reinterpret_cast<const float4*>(r.grad[q]);
        a.w[q] = reinterpret_cast<float4*>(r.master[q]);
        a.out[q] = reinterpret_cast<uint2*>(r.version[q]);
    }
    const size_t n4 = n / 4;
    const size_t lo = n4 * static_cast<size_t>(r.rank) / r.w, hi = n4 * static_cast<size_t>(r.rank + 1) / r.w;
    // per shard parameter: w gradient reads, the local state (w, m[, v]) read + written,
    // w fp32 master + w bf16 version stores
    const double per = 4.0 * r.w + (kAdam ? 24.0 : 16.0) + 6.0 * r.w;
    prof::Scope scope("optimizer", 0.0, per * 4.0 * static_cast<double>(hi - lo), 1, s);
    k_opt_replicas<kAdam><<<grid_for(hi - lo, 256), 256, 0, s>>>(a, r.w, r.rank, reinterpret_cast<float4*>(s1),
                                                                  reinterpret_cast<float4*>(s2), lo, hi, inv_count, lr,
                                                                  b1, b2, eps, inv_c1, inv_c2);
    check_cuda(cudaGetLastError(), "optimizer (replicas)");
}
}  // namespace

void sgd_momentum_update_replicas(const ReplicaShard& r, float* vel, size_t n, float inv_count, float lr,
                                  float beta, cudaStream_t s) {
    opt_replicas<false>(r, vel, nullptr, n, inv_count, lr, beta, 0.0f, 0.0f, 1.0f, 1.0f, s);
}

void adam_update_replicas(const ReplicaShard& r, float* m1, float* m2, size_t n, float inv_count, float lr,
                          float b1, float b2, float eps, int step, cudaStream_t s) {
    const float inv_c1 = static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(b1), step)));
    const float inv_c2 = static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(b2), step)));
    opt_replicas<true>(r, m1, m2, n, inv_count, lr, b1, b2, eps, inv_c1, inv_c2, s);
}

void init_uniform(float* w, size_t n, uint64_t seed, uint64_t uid, float half_width, cudaStream_t s) {
    prof::Scope scope("init", 0.0, 4.0 * static_cast<double>(n), 1, s);
    const uint64_t key = seed * 0x9e3779b97f4a7c15ULL + uid * 0xbf58476d1ce4e5b9ULL;
    k_init_uniform<<<grid_for(n, 256), 256, 0, s>>>(w, n, key, half_width);
    check_cuda(cudaGetLastError(), "init_uniform");
}

void fill_f32(float* w, size_t n, float v, cudaStream_t s) {
    prof::Scope scope("init", 0.0, 4.0 * static_cast<double>(n), 1, s);
    k_fill<<<grid_for(n, 256), 256, 0, s>>>(w, n, v);
    check_cuda(cudaGetLastError(), "fill_f32");
}

void cast_f32_bf16(const float* in, bf16* out, size_t n, cudaStream_t s) {
    prof::Scope scope("cast", 0.0, 6.0 * static_cast<double>(n), 1, s);
    k_cast_f2b<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
    check_cuda(cudaGetLastError(), "cast_f32_bf16");
}

void cast_bf16_f32(const bf16* in, float* out, size_t n, cudaStream_t s) {
    prof::Scope scope("cast", 0.0, 6.0 * static_cast<double>(n), 1, s);
    k_cast_b2f<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
    check_cuda(cudaGetLastError(), "cast_bf16_f32");
}

void gather_rows(const bf16* in, const int* idx, bf16* out, int rows, int h, cudaStream_t s) {
    prof::Scope scope("head_rows", 0.0, 4.0 * rows * h, 1, s);
    k_gather_rows<<<grid_for(static_cast<size_t>(rows) * h / 8, 256), 256, 0, s>>>(in, idx, out, rows, h, 0);
    check_cuda(cudaGetLastError(), "gather_rows");
}

void scatter_rows(const bf16* in, const int* idx, bf16* out, int rows, int h, cudaStream_t s) {
    prof::Scope scope("head_rows", 0.0, 4.0 * rows * h, 1, s);
    k_gather_rows<<<grid_for(static_cast<size_t>(rows) * h / 8, 256), 256, 0, s>>>(in, idx, out, rows, h, 1);
    check_cuda(cudaGetLastError(), "scatter_rows");
}

}  // namespace p2bw
