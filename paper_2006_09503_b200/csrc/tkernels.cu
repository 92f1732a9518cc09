// Transformer-stage kernels other than the tcgen05 GEMM: embedding, LayerNorm,
// deterministic column reductions (bias / LN-parameter gradients), fused
// softmax cross-entropy, the fused momentum optimizer and synthetic init.
// All are HBM-bound: 16-byte vector accesses, one warp (LN) or one CTA (CE)
// per row, grids sized to the SM count where a reduction follows.
#include <cuda_bf16.h>

#include <algorithm>

#include "profiler.h"
#include "ptx.cuh"
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
        float* dst = dtok + static_cast<size_t>(ids[t]) * h + c;
#pragma unroll
        for (int q = 0; q < 8; ++q) atomicAdd(dst + q, g[q]);
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
        for (int b = 0; b < batch; ++b) {
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

// out[c] (=|+=) sum_{p < parts} part[p * n + c], fixed order; 32 columns x 8 part lanes.
__global__ void k_reduce_parts(const float* __restrict__ part, int parts, int n,
                               float* __restrict__ out, int overwrite) {
    __shared__ float red[8][33];
    const int col = blockIdx.x * 32 + (threadIdx.x & 31);
    const int lane8 = threadIdx.x >> 5;
    // four independent accumulators (parts p, p+8, p+16, p+24 of each stride of 32)
    // keep four loads in flight; combined in a fixed order, so still deterministic
    float a[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (col < n) {
        int p = lane8;
        for (; p + 24 < parts; p += 32) {
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] += part[static_cast<size_t>(p + 8 * u) * n + col];
        }
        for (int u = 0; p < parts; p += 8, ++u) a[u & 3] += part[static_cast<size_t>(p) * n + col];
    }
    const float acc = (a[0] + a[1]) + (a[2] + a[3]);
    red[lane8][threadIdx.x & 31] = acc;
    __syncthreads();
    if (lane8 == 0 && col < n) {
        float s = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += red[i][threadIdx.x & 31];
        out[col] = overwrite ? s : out[col] + s;
    }
}

void reduce_parts(const float* part, int parts, int n, float* out, bool overwrite, cudaStream_t s) {
    k_reduce_parts<<<(n + 31) / 32, 256, 0, s>>>(part, parts, n, out, overwrite ? 1 : 0);
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
    __shared__ float red[8][256 + 8];
    const int cv = threadIdx.x & 31, rl = threadIdx.x >> 5;
    const int col = blockIdx.x * 256 + cv * 8;
    const int r0 = blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
    float a0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, a1[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (col < n) {
#pragma unroll 4
        for (int r = r0 + rl; r < r1; r += 8) {
            float g[8];
            load8(dy + static_cast<size_t>(r) * ld + col, g);
            if constexpr (kLn) {
                float xv[8];
                load8(x + static_cast<size_t>(r) * ld + col, xv);
                const float mu = mean[r], rs = rstd[r];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    a0[q] = fmaf(g[q], (xv[q] - mu) * rs, a0[q]);
                    a1[q] += g[q];
                }
            } else {
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

// Row blocks so that the grid has >= ~4 CTAs per SM; each block still sees >= 16 rows.
int colsum_row_blocks(int rows, int n) {
    const int col_blocks = (n + 255) / 256;
    const int want = (4 * 148 + col_blocks - 1) / col_blocks;
    return std::max(1, std::min(want, (rows + 15) / 16));
}

// ---- LayerNorm (one warp per row, up to NV 8-element vectors per lane) -------------------

template <int NV>
__global__ void k_ln_fwd(const bf16* __restrict__ x, const bf16* __restrict__ g, const bf16* __restrict__ b,
                         bf16* __restrict__ y, float* __restrict__ mean, float* __restrict__ rstd, int rows,
                         int h) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const int hv = h / 8;
    const bf16* xr = x + static_cast<size_t>(warp) * h;
    float v[NV][8];
    float sum = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int vi = lane + 32 * i;
        if (vi < hv) {
            load8(xr + vi * 8, v[i]);
#pragma unroll
            for (int q = 0; q < 8; ++q) sum += v[i][q];
        }
    }
    const float mu = warp_sum(sum) / h;
    float var = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i)
        if (lane + 32 * i < hv)
#pragma unroll
            for (int q = 0; q < 8; ++q) var += (v[i][q] - mu) * (v[i][q] - mu);
    const float rs = rsqrtf(warp_sum(var) / h + 1e-5f);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int vi = lane + 32 * i;
        if (vi < hv) {
            float gg[8], bb[8], o[8];
            load8(g + vi * 8, gg);
            load8(b + vi * 8, bb);
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = (v[i][q] - mu) * rs * gg[q] + bb[q];
            store8(y + static_cast<size_t>(warp) * h + vi * 8, o);
        }
    }
    if (lane == 0) {
        mean[warp] = mu;
        rstd[warp] = rs;
    }
}

// dx = rstd * (dxh - mean(dxh) - xh * mean(dxh * xh)) (+ dres), dxh = dy * g;
// one warp per row, no cross-row state (gamma / beta gradients: k_colstats<true>).
template <int NV>
__global__ void __launch_bounds__(256) k_ln_bwd_dx(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                                   const float* __restrict__ mean, const float* __restrict__ rstd,
                                                   const bf16* __restrict__ g, const bf16* __restrict__ dres,
                                                   bf16* __restrict__ dx, int rows, int h) {
    const int lane = threadIdx.x & 31;
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= rows) return;
    const int hv = h / 8;
    const float mu = mean[r], rs = rstd[r];
    float xh[NV][8], dxh[NV][8];
    float s1 = 0.0f, s2 = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int vi = lane + 32 * i;
        if (vi < hv) {
            float xv[8], dv[8], gv[8];
            load8(x + static_cast<size_t>(r) * h + vi * 8, xv);
            load8(dy + static_cast<size_t>(r) * h + vi * 8, dv);
            load8(g + vi * 8, gv);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                xh[i][q] = (xv[q] - mu) * rs;
                dxh[i][q] = dv[q] * gv[q];
                s1 += dxh[i][q];
                s2 += dxh[i][q] * xh[i][q];
            }
        }
    }
    const float m1 = warp_sum(s1) / h, m2 = warp_sum(s2) / h;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int vi = lane + 32 * i;
        if (vi < hv) {
            float o[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = rs * (dxh[i][q] - m1 - xh[i][q] * m2);
            if (dres != nullptr) {
                float rv[8];
                load8(dres + static_cast<size_t>(r) * h + vi * 8, rv);
#pragma unroll
                for (int q = 0; q < 8; ++q) o[q] += rv[q];
            }
            store8(dx + static_cast<size_t>(r) * h + vi * 8, o);
        }
    }
}

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
    const int grid = (rows + 7) / 8;
    switch (nv) {
        case 1: k_ln_fwd<1><<<grid, 256, 0, s>>>(x, g, b, y, mean, rstd, rows, h); break;
        case 2: k_ln_fwd<2><<<grid, 256, 0, s>>>(x, g, b, y, mean, rstd, rows, h); break;
        case 3: k_ln_fwd<3><<<grid, 256, 0, s>>>(x, g, b, y, mean, rstd, rows, h); break;
        case 4: k_ln_fwd<4><<<grid, 256, 0, s>>>(x, g, b, y, mean, rstd, rows, h); break;
        default: k_ln_fwd<8><<<grid, 256, 0, s>>>(x, g, b, y, mean, rstd, rows, h); break;
    }
    check_cuda(cudaGetLastError(), "layernorm_fwd");
}

size_t layernorm_bwd_scratch_floats(int rows, int h) {
    return static_cast<size_t>(colsum_row_blocks(rows, h)) * h * 2;
}

void layernorm_bwd(const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* g,
                   const bf16* dres, bf16* dx, float* dg, float* db, bool overwrite, int rows, int h,
                   float* scratch, cudaStream_t s) {
    if (h % 8 != 0 || h > 2048) throw Error("layernorm: hidden must be a multiple of 8 and <= 2048");
    prof::Scope scope("layernorm_bwd", 0.0, (dres ? 10.0 : 8.0) * rows * h + 8.0 * rows, 5, s);
    // gamma / beta statistics first: dx may alias dy (in-place LN backward)
    const int rb = colsum_row_blocks(rows, h);
    const int rpb = (rows + rb - 1) / rb;
    float* pg = scratch;
    float* pb = scratch + static_cast<size_t>(rb) * h;
    k_colstats<true><<<dim3((h + 255) / 256, rb), 256, 0, s>>>(dy, x, mean, rstd, rows, h, h, rpb, pg, pb);
    reduce_parts(pg, rb, h, dg, overwrite, s);
    reduce_parts(pb, rb, h, db, overwrite, s);
    const int nv = (h / 8 + 31) / 32;
    const int grid = (rows + 7) / 8;
    switch (nv) {
        case 1: k_ln_bwd_dx<1><<<grid, 256, 0, s>>>(dy, x, mean, rstd, g, dres, dx, rows, h); break;
        case 2: k_ln_bwd_dx<2><<<grid, 256, 0, s>>>(dy, x, mean, rstd, g, dres, dx, rows, h); break;
        case 3: k_ln_bwd_dx<3><<<grid, 256, 0, s>>>(dy, x, mean, rstd, g, dres, dx, rows, h); break;
        case 4: k_ln_bwd_dx<4><<<grid, 256, 0, s>>>(dy, x, mean, rstd, g, dres, dx, rows, h); break;
        default: k_ln_bwd_dx<8><<<grid, 256, 0, s>>>(dy, x, mean, rstd, g, dres, dx, rows, h); break;
    }
    check_cuda(cudaGetLastError(), "layernorm_bwd");
}

size_t colsum_scratch_floats(int rows, int n) { return static_cast<size_t>(colsum_row_blocks(rows, n)) * n; }

void colsum_bf16(const bf16* x, int rows, int n, int ld, float* out, bool overwrite, float* scratch,
                 cudaStream_t s) {
    if (n % 8 != 0) throw Error("colsum: columns must be a multiple of 8");
    prof::Scope scope("bias_grad", 0.0, 2.0 * rows * n + 8.0 * n, 2, s);
    const int rb = colsum_row_blocks(rows, n);
    const int rpb = (rows + rb - 1) / rb;
    k_colstats<false><<<dim3((n + 255) / 256, rb), 256, 0, s>>>(x, nullptr, nullptr, nullptr, rows, n, ld, rpb,
                                                                  scratch, nullptr);
    reduce_parts(scratch, rb, n, out, overwrite, s);
    check_cuda(cudaGetLastError(), "colsum");
}

void softmax_xent(bf16* logits, const int* targets, int rows, int vocab, int vp, float grad_scale,
                  float* row_loss, cudaStream_t s) {
    if (vp % 8 != 0) throw Error("softmax_xent: padded vocab must be a multiple of 8");
    prof::Scope scope("softmax_xent", 0.0, 4.0 * rows * static_cast<double>(vp) + 8.0 * rows, 1, s);
    k_softmax_xent<<<rows, 256, 0, s>>>(logits, targets, vocab, vp, grad_scale, row_loss);
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
