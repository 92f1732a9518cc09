// Launch interface of the transformer-stage kernels (bf16 activations, fp32
// statistics / gradients / master weights).  All launches are asynchronous on
// the given stream and fail loudly on launch errors.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "util.h"

namespace p2bw {

// x0[t] = tok[ids[t]] + pos[t % seq]                                  [T x h]
void embed_fwd(const int* ids, const bf16* tok, const bf16* pos, bf16* x0, int tokens, int seq,
               int h, cudaStream_t s);
// dtok[ids[t]] += dx0[t] (fp32 atomics; rows of dtok must be zeroed first);
// dpos[p] (=|+=) sum_b dx0[b*seq + p]                                  deterministic
void embed_bwd(const int* ids, const bf16* dx0, float* dtok, float* dpos, int tokens, int seq, int h,
               bool overwrite_pos, cudaStream_t s);

// y = LN(x) * g + b ; mean / rstd per row saved for the backward.
void layernorm_fwd(const bf16* x, const bf16* g, const bf16* b, bf16* y, float* mean, float* rstd,
                   int rows, int h, cudaStream_t s);
// dx = LN'(dy) (+ dres); dg / db (=|+=) column sums, deterministic two-phase; with
// dsum != nullptr also dsum (=|+=) sum_r bf16(dx[r, :]) (the bias gradient of the
// layer that consumes dx as its output gradient).  dx may alias dy.
void layernorm_bwd(const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* g,
                   const bf16* dres, bf16* dx, float* dg, float* db, bool overwrite, int rows, int h,
                   float* scratch, cudaStream_t s, float* dsum = nullptr);
size_t layernorm_bwd_scratch_floats(int rows, int h);

// out[n] (=|+=) sum_r x[r, n]  (bias gradients), deterministic two-phase.
void colsum_bf16(const bf16* x, int rows, int n, int ld, float* out, bool overwrite, float* scratch,
                 cudaStream_t s);
size_t colsum_scratch_floats(int rows, int n);

// Fused softmax cross-entropy over logits [rows x vp] (first `vocab` columns valid):
// row_loss[r] = lse - logit[target]; logits <- (softmax - onehot) * grad_scale (in place).
void softmax_xent(bf16* logits, const int* targets, int rows, int vocab, int vp, float grad_scale,
                  float* row_loss, cudaStream_t s);
// loss_out = sum(row_loss[0:rows]) * scale  (one block, fixed order)
void sum_scaled(const float* row_loss, int rows, float scale, float* loss_out, cudaStream_t s);

// Attention over qkv [T x 3h] (q | k | v, heads of head_dim = 64 or 128), output o [T x h],
// lse [b*nh*seq].
void attention_fwd(const bf16* qkv, bf16* o, float* lse, int batch, int seq, int heads, bool causal,
                   cudaStream_t s, int head_dim = 64);
// The tcgen05 kernels cover seq % 128 == 0 (attention.cu rejects anything else).
bool attention_tc_supported(int seq);
// Debug: per-CTA phase timestamps of the tcgen05 forward into dev_buf[cta * 16 + slot] (null: off).
void attention_debug_timing(unsigned long long* dev_buf);
// Debug: phase timestamps of the tcgen05 attention backward (64 per CTA, null: off).
void attention_bwd_debug_timing(unsigned long long* dev_buf);
void attention_fwd_tc(const bf16* qkv, bf16* o, float* lse, int batch, int seq, int heads, bool causal,
                      cudaStream_t s, int head_dim);
size_t attention_bwd_tc_scratch_floats(int batch, int seq, int heads, int head_dim);
void attention_bwd_tc(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, bf16* dqkv,
                      float* delta, float* dq_part, int batch, int seq, int heads, bool causal, cudaStream_t s,
                      int head_dim, float* dq_alt = nullptr, int phase = 0, bool last = true);
// dqkv [T x 3h] from do [T x h]; delta: [b*nh*seq] floats; scratch: attention_bwd_scratch_floats.
// A run of consecutive calls on one stream (a stage's layers in one Backward) may pass a
// second dQ accumulator dq_alt ([T x h] floats) with phase = 0, 1, ... and last on the
// final call: the accumulators alternate and each call's kernel zeroes the next one's.
size_t attention_bwd_scratch_floats(int batch, int seq, int heads, int head_dim = 64);
void attention_bwd(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, bf16* dqkv,
                   float* delta, float* scratch, int batch, int seq, int heads, bool causal, cudaStream_t s,
                   int head_dim = 64, float* dq_alt = nullptr, int phase = 0, bool last = true);

// Momentum SGD with dampening (semantics.cpp:153-165) on the flat fp32 master:
//   g = grad / count; v = beta v + (1-beta) g; w -= lr v; out_bf16 = bf16(w)
void sgd_momentum_update(float* master, float* vel, const float* grad, bf16* out_bf16, size_t n,
                         float inv_count, float lr, float beta, cudaStream_t s);

// Data-parallel replicas on one node (CUDA IPC; Engine::join_replicas_ipc): the
// AllReduce op fused into the optimizer.  Replica `rank` of `w` owns parameter shard
// [rank n / w, (rank + 1) n / w) (in 4-element vectors): it sums that shard of every
// replica's coalesced gradient (peer loads over NVLink, replica order 0 .. w-1 -- one
// writer per element, so every replica ends bit-identical), updates the shard's
// optimizer state (local) and stores the new fp32 master and bf16 version of the shard
// into every replica (peer stores): reduce-scatter, update and all-gather in one pass,
// (w - 1) / w x (4 + 4 + 2) bytes per parameter over the links.
struct ReplicaShard {
    const float* grad[kMaxReplicas];
    float* master[kMaxReplicas];
    bf16* version[kMaxReplicas];
    int w = 1, rank = 0;
};
void sgd_momentum_update_replicas(const ReplicaShard& r, float* vel, size_t n, float inv_count, float lr,
                                  float beta, cudaStream_t s);
void adam_update_replicas(const ReplicaShard& r, float* m1, float* m2, size_t n, float inv_count, float lr,
                          float b1, float b2, float eps, int step, cudaStream_t s);

// out[c] (=|+=) sum_{p < parts} part[p * n + c], fixed order (deterministic).
void reduce_partials(const float* part, int parts, int n, float* out, bool overwrite, cudaStream_t s);

// Adam (bias-corrected, step = 1-based update count) on the flat fp32 master; m1 / m2
// are the first / second moment buffers.
void adam_update(float* master, float* m1, float* m2, const float* grad, bf16* out_bf16, size_t n, float inv_count,
                 float lr, float b1, float b2, float eps, int step, cudaStream_t s);

// Deterministic synthetic init: w = (u - 0.5) * 2a with u from splitmix64(seed, uid, i).
void init_uniform(float* w, size_t n, uint64_t seed, uint64_t uid, float half_width, cudaStream_t s);
void fill_f32(float* w, size_t n, float v, cudaStream_t s);
void cast_f32_bf16(const float* in, bf16* out, size_t n, cudaStream_t s);
void cast_bf16_f32(const bf16* in, float* out, size_t n, cudaStream_t s);

// Row gather / scatter for masked-position heads: out[r] = in[idx[r]]; out[idx[r]] = in[r].
void gather_rows(const bf16* in, const int* idx, bf16* out, int rows, int h, cudaStream_t s);
void scatter_rows(const bf16* in, const int* idx, bf16* out, int rows, int h, cudaStream_t s);

}  // namespace p2bw
