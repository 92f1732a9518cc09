// Attention entry points of the transformer stage: shape checks, profiler scopes and
// the tcgen05 kernels (attention_tc.cu forward, attention_tc_bwd.cu backward).  There is
// one implementation per pass -- no CUDA-core fallback: a shape the tensor-core tiles do
// not cover (sequence length not a multiple of 128) is an error, not a slower path.
#include "profiler.h"
#include "tkernels.h"
#include "util.h"

namespace p2bw {
namespace {

void check_shape(int seq, int heads, int head_dim) {
    if (head_dim != 64 && head_dim != 128) throw Error("attention: head dim must be 64 or 128");
    if (!attention_tc_supported(seq))
        throw Error("attention: sequence length " + std::to_string(seq) +
                    " is not a positive multiple of 128 (the tcgen05 query / key tiles)");
    if (heads < 1) throw Error("attention: heads must be >= 1");
}

}  // namespace

bool attention_tc_supported(int seq) { return seq >= 128 && seq % 128 == 0; }

void attention_fwd(const bf16* qkv, bf16* o, float* lse, int batch, int seq, int heads, bool causal,
                   cudaStream_t s, int head_dim) {
    check_shape(seq, heads, head_dim);
    const double flops = 4.0 * batch * heads * head_dim * seq * seq * (causal ? 0.5 : 1.0);
    prof::Scope scope("attention_fwd", flops, 2.0 * batch * seq * heads * head_dim * 4.0, 1, s);
    attention_fwd_tc(qkv, o, lse, batch, seq, heads, causal, s, head_dim);
}

size_t attention_bwd_scratch_floats(int batch, int seq, int heads, int head_dim) {
    check_shape(seq, heads, head_dim);
    return attention_bwd_tc_scratch_floats(batch, seq, heads, head_dim);
}

void attention_bwd(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, bf16* dqkv, float* delta,
                   float* scratch, int batch, int seq, int heads, bool causal, cudaStream_t s, int head_dim,
                   float* dq_alt, int phase, bool last) {
    check_shape(seq, heads, head_dim);
    const double flops = 8.0 * batch * heads * head_dim * seq * seq * (causal ? 0.5 : 1.0);
    prof::Scope scope("attention_bwd", flops, 2.0 * batch * seq * heads * head_dim * 8.0, 3, s);
    attention_bwd_tc(qkv, o, dout, lse, dqkv, delta, scratch, batch, seq, heads, causal, s, head_dim, dq_alt, phase,
                     last);
}

}  // namespace p2bw
