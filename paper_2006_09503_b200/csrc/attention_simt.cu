// Softmax attention (head dim 64) on CUDA cores: the correctness-first path.
// Forward: one warp per query row; scores for all keys of the row are held in
// registers (seq <= 512), exact softmax, then P.V with the row's weights
// broadcast by shuffles.  Backward: a query-parallel pass (dQ, delta = rowsum(dO*O))
// and a key-parallel pass (dK, dV) that recompute P from the saved log-sum-exp.
// K/V (or Q/dO) of one (sequence, head) are staged in shared memory with a
// 72-element row pitch (16-byte aligned, 4-way bank spread for row-wise reads).
#include <cuda_bf16.h>

#include "profiler.h"
#include "ptx.cuh"
#include "tkernels.h"
#include "util.h"

namespace p2bw {
namespace {

constexpr int kD = 64;        // head dim
constexpr int kPitch = 72;    // smem row pitch (elements)
constexpr int kQB = 64;       // queries (or keys) per CTA
constexpr int kMaxSeq = 512;  // register-resident score row
constexpr float kLog2e = 1.4426950408889634f;

// dot(q, row) with q as 64 floats in smem (broadcast) and row as bf16 in smem.
__device__ __forceinline__ float dot64(const float* __restrict__ q, const bf16* __restrict__ row) {
    float acc = 0.0f;
#pragma unroll
    for (int c = 0; c < kD; c += 8) {
        const uint4 u = *reinterpret_cast<const uint4*>(row + c);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = ptx::unpack_bf16x2(w[i]);
            acc = fmaf(q[c + 2 * i], f.x, acc);
            acc = fmaf(q[c + 2 * i + 1], f.y, acc);
        }
    }
    return acc;
}

// Stage rows [r0, r1) of a [T x ld] matrix at column `col` into smem rows 0..r1-r0.
__device__ __forceinline__ void stage_rows(bf16* sm, const bf16* g, size_t ld, int r0, int r1) {
    const int n = (r1 - r0) * (kD / 8);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int r = i / (kD / 8), c = (i % (kD / 8)) * 8;
        *reinterpret_cast<uint4*>(sm + r * kPitch + c) =
            *reinterpret_cast<const uint4*>(g + static_cast<size_t>(r0 + r) * ld + c);
    }
}

template <bool kCausal>
__global__ void __launch_bounds__(256) k_attn_fwd(const bf16* __restrict__ qkv, bf16* __restrict__ out,
                                                  float* __restrict__ lse, int seq, int heads) {
    extern __shared__ __align__(16) uint8_t smem[];
    bf16* sk = reinterpret_cast<bf16*>(smem);
    bf16* sv = sk + kMaxSeq * kPitch;
    float* sq = reinterpret_cast<float*>(sv + kMaxSeq * kPitch);  // [8 warps][64]
    const int bh = blockIdx.x, b = bh / heads, hd = bh % heads;
    const int h = heads * kD;
    const size_t ld = 3 * static_cast<size_t>(h);
    const bf16* base = qkv + static_cast<size_t>(b) * seq * ld;
    const int q0 = blockIdx.y * kQB;
    const int kv_len = kCausal ? min(seq, q0 + kQB) : seq;
    stage_rows(sk, base + h + hd * kD, ld, 0, kv_len);
    stage_rows(sv, base + 2 * h + hd * kD, ld, 0, kv_len);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float sc = 0.125f * kLog2e;  // 1/sqrt(64) in the log2 domain
    float* q = sq + warp * kD;
    for (int qi = warp; qi < kQB; qi += 8) {
        const int i = q0 + qi;
        if (i >= seq) break;
        const bf16* qrow = base + static_cast<size_t>(i) * ld + hd * kD;
        const float2 qf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(qrow + 2 * lane));
        q[2 * lane] = qf.x * sc;
        q[2 * lane + 1] = qf.y * sc;
        __syncwarp();
        const int n_keys = kCausal ? i + 1 : kv_len;
        float s[kMaxSeq / 32];
        float m = -INFINITY;
#pragma unroll
        for (int c = 0; c < kMaxSeq / 32; ++c) {
            const int j = lane + 32 * c;
            s[c] = j < n_keys ? dot64(q, sk + j * kPitch) : -INFINITY;
            m = fmaxf(m, s[c]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float l = 0.0f;
#pragma unroll
        for (int c = 0; c < kMaxSeq / 32; ++c) {
            s[c] = exp2f(s[c] - m);
            l += s[c];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        float o0 = 0.0f, o1 = 0.0f;
#pragma unroll
        for (int c = 0; c < kMaxSeq / 32; ++c) {
            if (32 * c >= n_keys) break;
            for (int src = 0; src < 32; ++src) {
                const int j = 32 * c + src;
                const float p = __shfl_sync(0xffffffffu, s[c], src);
                if (j < n_keys) {
                    const float2 v = __bfloat1622float2(
                        *reinterpret_cast<const __nv_bfloat162*>(sv + j * kPitch + 2 * lane));
                    o0 = fmaf(p, v.x, o0);
                    o1 = fmaf(p, v.y, o1);
                }
            }
        }
        const float inv = 1.0f / l;
        *reinterpret_cast<__nv_bfloat162*>(out + (static_cast<size_t>(b) * seq + i) * h + hd * kD + 2 * lane) =
            __floats2bfloat162_rn(o0 * inv, o1 * inv);
        if (lane == 0) lse[static_cast<size_t>(bh) * seq + i] = (m + log2f(l)) / kLog2e;
        __syncwarp();
    }
}

// dQ and delta, one warp per query row.
template <bool kCausal>
__global__ void __launch_bounds__(256) k_attn_bwd_q(const bf16* __restrict__ qkv, const bf16* __restrict__ o,
                                                    const bf16* __restrict__ dout, const float* __restrict__ lse,
                                                    bf16* __restrict__ dqkv, float* __restrict__ delta, int seq,
                                                    int heads) {
    extern __shared__ __align__(16) uint8_t smem[];
    bf16* sk = reinterpret_cast<bf16*>(smem);
    bf16* sv = sk + kMaxSeq * kPitch;
    float* sq = reinterpret_cast<float*>(sv + kMaxSeq * kPitch);  // [8][64] q
    float* sd = sq + 8 * kD;                                      // [8][64] dO
    const int bh = blockIdx.x, b = bh / heads, hd = bh % heads;
    const int h = heads * kD;
    const size_t ld = 3 * static_cast<size_t>(h);
    const bf16* base = qkv + static_cast<size_t>(b) * seq * ld;
    const int q0 = blockIdx.y * kQB;
    const int kv_len = kCausal ? min(seq, q0 + kQB) : seq;
    stage_rows(sk, base + h + hd * kD, ld, 0, kv_len);
    stage_rows(sv, base + 2 * h + hd * kD, ld, 0, kv_len);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float sc = 0.125f * kLog2e;
    float* q = sq + warp * kD;
    float* dov = sd + warp * kD;
    for (int qi = warp; qi < kQB; qi += 8) {
        const int i = q0 + qi;
        if (i >= seq) break;
        const size_t t = static_cast<size_t>(b) * seq + i;
        const float2 qf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(base + i * ld + hd * kD + 2 * lane));
        const float2 df = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dout + t * h + hd * kD + 2 * lane));
        const float2 of = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(o + t * h + hd * kD + 2 * lane));
        q[2 * lane] = qf.x * sc;
        q[2 * lane + 1] = qf.y * sc;
        dov[2 * lane] = df.x;
        dov[2 * lane + 1] = df.y;
        float dd = df.x * of.x + df.y * of.y;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, off);
        __syncwarp();
        const float l2 = lse[static_cast<size_t>(bh) * seq + i] * kLog2e;
        const int n_keys = kCausal ? i + 1 : kv_len;
        float ds[kMaxSeq / 32];
#pragma unroll
        for (int c = 0; c < kMaxSeq / 32; ++c) {
            const int j = lane + 32 * c;
            if (j < n_keys) {
                const float p = exp2f(dot64(q, sk + j * kPitch) - l2);
                const float dp = dot64(dov, sv + j * kPitch);
                ds[c] = p * (dp - dd);
            } else {
                ds[c] = 0.0f;
            }
        }
        float g0 = 0.0f, g1 = 0.0f;
#pragma unroll
        for (int c = 0; c < kMaxSeq / 32; ++c) {
            if (32 * c >= n_keys) break;
            for (int src = 0; src < 32; ++src) {
                const int j = 32 * c + src;
                const float w = __shfl_sync(0xffffffffu, ds[c], src);
                if (j < n_keys) {
                    const float2 kf = __bfloat1622float2(
                        *reinterpret_cast<const __nv_bfloat162*>(sk + j * kPitch + 2 * lane));
                    g0 = fmaf(w, kf.x, g0);
                    g1 = fmaf(w, kf.y, g1);
                }
            }
        }
        *reinterpret_cast<__nv_bfloat162*>(dqkv + t * ld + hd * kD + 2 * lane) =
            __floats2bfloat162_rn(g0 * 0.125f, g1 * 0.125f);
        if (lane == 0) delta[static_cast<size_t>(bh) * seq + i] = dd;
        __syncwarp();
    }
}

// dK and dV, one warp per key row (queries staged in smem).
template <bool kCausal>
__global__ void __launch_bounds__(256) k_attn_bwd_kv(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                     const float* __restrict__ lse, const float* __restrict__ delta,
                                                     bf16* __restrict__ dqkv, int seq, int heads) {
    extern __shared__ __align__(16) uint8_t smem[];
    bf16* sq = reinterpret_cast<bf16*>(smem);
    bf16* sdo = sq + kMaxSeq * kPitch;
    float* sl = reinterpret_cast<float*>(sdo + kMaxSeq * kPitch);  // lse2 [seq]
    float* sdd = sl + kMaxSeq;                                      // delta [seq]
    float* skv = sdd + kMaxSeq;                                     // [8][2][64]
    const int bh = blockIdx.x, b = bh / heads, hd = bh % heads;
    const int h = heads * kD;
    const size_t ld = 3 * static_cast<size_t>(h);
    const bf16* base = qkv + static_cast<size_t>(b) * seq * ld;
    const int k0 = blockIdx.y * kQB;
    const int qs = kCausal ? k0 : 0;  // first query that can see this key block
    stage_rows(sq, base + static_cast<size_t>(qs) * ld + hd * kD, ld, 0, seq - qs);
    stage_rows(sdo, dout + (static_cast<size_t>(b) * seq + qs) * h + hd * kD, h, 0, seq - qs);
    for (int i = threadIdx.x; i < seq - qs; i += blockDim.x) {
        sl[i] = lse[static_cast<size_t>(bh) * seq + qs + i] * kLog2e;
        sdd[i] = delta[static_cast<size_t>(bh) * seq + qs + i];
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float sc = 0.125f * kLog2e;
    float* kf = skv + warp * 2 * kD;
    float* vf = kf + kD;
    for (int ki = warp; ki < kQB; ki += 8) {
        const int j = k0 + ki;
        if (j >= seq) break;
        const float2 kk = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(base + j * ld + h + hd * kD + 2 * lane));
        const float2 vv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(base + j * ld + 2 * h + hd * kD + 2 * lane));
        kf[2 * lane] = kk.x * sc;
        kf[2 * lane + 1] = kk.y * sc;
        vf[2 * lane] = vv.x;
        vf[2 * lane + 1] = vv.y;
        __syncwarp();
        const int first = kCausal ? j - qs : 0;  // local index of the first query that sees key j
        const int nq = seq - qs;
        float pv[kMaxSeq / 32], dsv[kMaxSeq / 32];
#pragma unroll
        for (int c = 0; c < kMaxSeq / 32; ++c) {
            const int il = lane + 32 * c;
            if (il < nq && il >= first) {
                const float p = exp2f(dot64(kf, sq + il * kPitch) - sl[il]);
                const float dp = dot64(vf, sdo + il * kPitch);
                pv[c] = p;
                dsv[c] = p * (dp - sdd[il]);
            } else {
                pv[c] = 0.0f;
                dsv[c] = 0.0f;
            }
        }
        float dv0 = 0.0f, dv1 = 0.0f, dk0 = 0.0f, dk1 = 0.0f;
#pragma unroll
        for (int c = 0; c < kMaxSeq / 32; ++c) {
            if (32 * c >= nq) break;
            for (int src = 0; src < 32; ++src) {
                const int il = 32 * c + src;
                const float p = __shfl_sync(0xffffffffu, pv[c], src);
                const float w = __shfl_sync(0xffffffffu, dsv[c], src);
                if (il < nq) {
                    const float2 d2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sdo + il * kPitch + 2 * lane));
                    const float2 q2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sq + il * kPitch + 2 * lane));
                    dv0 = fmaf(p, d2.x, dv0);
                    dv1 = fmaf(p, d2.y, dv1);
                    dk0 = fmaf(w, q2.x, dk0);
                    dk1 = fmaf(w, q2.y, dk1);
                }
            }
        }
        const size_t t = static_cast<size_t>(b) * seq + j;
        *reinterpret_cast<__nv_bfloat162*>(dqkv + t * ld + h + hd * kD + 2 * lane) =
            __floats2bfloat162_rn(dk0 * 0.125f, dk1 * 0.125f);
        *reinterpret_cast<__nv_bfloat162*>(dqkv + t * ld + 2 * h + hd * kD + 2 * lane) = __floats2bfloat162_rn(dv0, dv1);
        __syncwarp();
    }
}

constexpr size_t kFwdSmem = 2 * kMaxSeq * kPitch * sizeof(bf16) + 8 * kD * sizeof(float);
constexpr size_t kBwdQSmem = 2 * kMaxSeq * kPitch * sizeof(bf16) + 16 * kD * sizeof(float);
constexpr size_t kBwdKVSmem = 2 * kMaxSeq * kPitch * sizeof(bf16) + 2 * kMaxSeq * sizeof(float) + 16 * kD * sizeof(float);

template <class K>
void set_smem(K kern, size_t bytes) {
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)),
               "cudaFuncSetAttribute(attention smem)");
}

void check_shape(int seq, int heads) {
    if (seq < 1 || seq > kMaxSeq) throw Error("attention: sequence length must be in [1, 512]");
    if (heads < 1) throw Error("attention: heads must be >= 1");
}

}  // namespace

void attention_fwd(const bf16* qkv, bf16* o, float* lse, int batch, int seq, int heads, bool causal,
                   cudaStream_t s) {
    check_shape(seq, heads);
    const double flops = 4.0 * batch * heads * 64.0 * seq * seq * (causal ? 0.5 : 1.0);
    prof::Scope scope("attention_fwd", flops, 2.0 * batch * seq * heads * 64.0 * 4, 1, s);
    if (attention_tc_supported(seq)) {  // tensor-core path: seq in {128, 256, 384, 512}
        attention_fwd_tc(qkv, o, lse, batch, seq, heads, causal, s);
        return;
    }
    dim3 grid(batch * heads, (seq + kQB - 1) / kQB);
    if (causal) {
        set_smem(k_attn_fwd<true>, kFwdSmem);
        k_attn_fwd<true><<<grid, 256, kFwdSmem, s>>>(qkv, o, lse, seq, heads);
    } else {
        set_smem(k_attn_fwd<false>, kFwdSmem);
        k_attn_fwd<false><<<grid, 256, kFwdSmem, s>>>(qkv, o, lse, seq, heads);
    }
    check_cuda(cudaGetLastError(), "attention_fwd");
}

size_t attention_bwd_scratch_floats(int batch, int seq, int heads) {
    return attention_tc_supported(seq) ? attention_bwd_tc_scratch_floats(batch, seq, heads) : 0;
}

void attention_bwd(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, bf16* dqkv, float* delta,
                   float* scratch, int batch, int seq, int heads, bool causal, cudaStream_t s) {
    check_shape(seq, heads);
    const double flops = 8.0 * batch * heads * 64.0 * seq * seq * (causal ? 0.5 : 1.0);
    if (attention_tc_supported(seq)) {  // tensor-core path
        prof::Scope scope("attention_bwd", flops, 2.0 * batch * seq * heads * 64.0 * 8, 3, s);
        attention_bwd_tc(qkv, o, dout, lse, dqkv, delta, scratch, batch, seq, heads, causal, s);
        return;
    }
    prof::Scope scope("attention_bwd", flops, 2.0 * batch * seq * heads * 64.0 * 8, 2, s);
    dim3 grid(batch * heads, (seq + kQB - 1) / kQB);
    if (causal) {
        set_smem(k_attn_bwd_q<true>, kBwdQSmem);
        set_smem(k_attn_bwd_kv<true>, kBwdKVSmem);
        k_attn_bwd_q<true><<<grid, 256, kBwdQSmem, s>>>(qkv, o, dout, lse, dqkv, delta, seq, heads);
        k_attn_bwd_kv<true><<<grid, 256, kBwdKVSmem, s>>>(qkv, dout, lse, delta, dqkv, seq, heads);
    } else {
        set_smem(k_attn_bwd_q<false>, kBwdQSmem);
        set_smem(k_attn_bwd_kv<false>, kBwdKVSmem);
        k_attn_bwd_q<false><<<grid, 256, kBwdQSmem, s>>>(qkv, o, dout, lse, dqkv, delta, seq, heads);
        k_attn_bwd_kv<false><<<grid, 256, kBwdKVSmem, s>>>(qkv, dout, lse, delta, dqkv, seq, heads);
    }
    check_cuda(cudaGetLastError(), "attention_bwd");
}

}  // namespace p2bw
