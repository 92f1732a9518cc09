// C-ABI entry points that expose single stage kernels for parity tests
// (p2bw_kernel_*).  Device pointers in, status code out; see include/p2bw.h.
#include "capi_internal.h"
#include "kernels.h"
#include "tkernels.h"
#include "util.h"
#include "p2bw.h"

using namespace p2bw;

extern "C" int p2bw_kernel_gemm_bf16(const void* a, long long lda, int a_major, const void* b,
                                     long long ldb, int b_major, int m, int n, int k,
                                     const p2bw_gemm_epilogue* epi, void* stream) {
    return guarded([&] {
        if (epi == nullptr) throw Error("epilogue descriptor is NULL");
        GemmOperand A{static_cast<const bf16*>(a), lda, a_major ? Major::MN : Major::K};
        GemmOperand B{static_cast<const bf16*>(b), ldb, b_major ? Major::MN : Major::K};
        GemmEpilogue e;
        e.kind = static_cast<EpiKind>(epi->kind);
        e.d = epi->d;
        e.ldd = epi->ldd;
        e.bias = static_cast<const bf16*>(epi->bias);
        e.residual = static_cast<const bf16*>(epi->residual);
        e.ldr = epi->ldr;
        e.preact = static_cast<bf16*>(epi->preact);
        e.gelu = epi->gelu != 0;
        e.aux = static_cast<const bf16*>(epi->aux);
        e.alpha = epi->alpha;
        e.beta = epi->beta;
        e.workspace = static_cast<float*>(epi->workspace);
        e.workspace_floats = epi->workspace_floats;
        e.bias_grad = static_cast<float*>(epi->bias_grad);
        e.bias_grad_accumulate = epi->bias_grad_accumulate != 0;
        e.bias_scratch = static_cast<float*>(epi->bias_scratch);
        e.bias_scratch_floats = epi->bias_scratch_floats;
        gemm_bf16(A, B, m, n, k, e, static_cast<cudaStream_t>(stream));
    });
}

namespace {
cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }
const bf16* cb(const void* p) { return static_cast<const bf16*>(p); }
bf16* mb(void* p) { return static_cast<bf16*>(p); }
}  // namespace

extern "C" int p2bw_kernel_attention_fwd_hd(const void* qkv, void* o, void* lse, int batch, int seq, int heads,
                                            int head_dim, int causal, void* stream) {
    return guarded([&] {
        attention_fwd(cb(qkv), mb(o), static_cast<float*>(lse), batch, seq, heads, causal != 0, as_stream(stream),
                      head_dim);
    });
}

extern "C" int p2bw_kernel_attention_fwd(const void* qkv, void* o, void* lse, int batch, int seq, int heads,
                                         int causal, void* stream) {
    return p2bw_kernel_attention_fwd_hd(qkv, o, lse, batch, seq, heads, 64, causal, stream);
}

extern "C" int p2bw_kernel_attention_bwd_hd(const void* qkv, const void* o, const void* dout, const void* lse,
                                            void* dqkv, void* delta, int batch, int seq, int heads, int head_dim,
                                            int causal, void* stream) {
    return guarded([&] {
        float* scratch = nullptr;
        const size_t n = attention_bwd_scratch_floats(batch, seq, heads, head_dim);
        if (n) check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&scratch), n * sizeof(float), as_stream(stream)),
                          "cudaMallocAsync");
        attention_bwd(cb(qkv), cb(o), cb(dout), static_cast<const float*>(lse), mb(dqkv),
                      static_cast<float*>(delta), scratch, batch, seq, heads, causal != 0, as_stream(stream),
                      head_dim);
        if (n) check_cuda(cudaFreeAsync(scratch, as_stream(stream)), "cudaFreeAsync");
    });
}

extern "C" int p2bw_kernel_attention_bwd(const void* qkv, const void* o, const void* dout, const void* lse,
                                         void* dqkv, void* delta, int batch, int seq, int heads, int causal,
                                         void* stream) {
    return p2bw_kernel_attention_bwd_hd(qkv, o, dout, lse, dqkv, delta, batch, seq, heads, 64, causal, stream);
}

extern "C" int p2bw_kernel_layernorm_fwd(const void* x, const void* g, const void* b, void* y, void* mean,
                                         void* rstd, int rows, int h, void* stream) {
    return guarded([&] {
        layernorm_fwd(cb(x), cb(g), cb(b), mb(y), static_cast<float*>(mean), static_cast<float*>(rstd), rows, h,
                      as_stream(stream));
    });
}

extern "C" int p2bw_kernel_layernorm_bwd(const void* dy, const void* x, const void* mean, const void* rstd,
                                         const void* g, const void* dres, void* dx, void* dg, void* db,
                                         void* dsum, int overwrite, int rows, int h, void* stream) {
    return guarded([&] {
        float* scratch = nullptr;
        check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                                   layernorm_bwd_scratch_floats(rows, h) * sizeof(float), as_stream(stream)),
                   "cudaMallocAsync");
        layernorm_bwd(cb(dy), cb(x), static_cast<const float*>(mean), static_cast<const float*>(rstd), cb(g),
                      cb(dres), mb(dx), static_cast<float*>(dg), static_cast<float*>(db), overwrite != 0, rows, h,
                      scratch, as_stream(stream), static_cast<float*>(dsum));
        check_cuda(cudaFreeAsync(scratch, as_stream(stream)), "cudaFreeAsync");
    });
}

extern "C" int p2bw_kernel_softmax_xent(void* logits, const void* targets, int rows, int vocab, int vp,
                                        float grad_scale, void* row_loss, void* stream) {
    return guarded([&] {
        softmax_xent(mb(logits), static_cast<const int*>(targets), rows, vocab, vp, grad_scale,
                     static_cast<float*>(row_loss), as_stream(stream));
    });
}

extern "C" int p2bw_debug_attention_timing(void* dev_buf) {
    return guarded([&] {
        attention_debug_timing(static_cast<unsigned long long*>(dev_buf));
        attention_bwd_debug_timing(static_cast<unsigned long long*>(dev_buf));
    });
}

extern "C" int p2bw_debug_gemm_timing(void* dev_buf) {
    return guarded([&] { gemm_debug_timing(static_cast<unsigned long long*>(dev_buf)); });
}

extern "C" int p2bw_debug_gemm_plan(int m, int n, int k, int a_major, int b_major, int kind, int bias_grad,
                                    int* out) {
    return guarded([&] { gemm_plan(m, n, k, a_major != 0, b_major != 0, kind == 1, bias_grad != 0, out); });
}

extern "C" int p2bw_kernel_colsum(const void* x, int rows, int n, int ld, void* out, int overwrite, void* stream) {
    return guarded([&] {
        float* scratch = nullptr;
        check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&scratch), colsum_scratch_floats(rows, n) * sizeof(float),
                                   as_stream(stream)), "cudaMallocAsync");
        colsum_bf16(cb(x), rows, n, ld, static_cast<float*>(out), overwrite != 0, scratch, as_stream(stream));
        check_cuda(cudaFreeAsync(scratch, as_stream(stream)), "cudaFreeAsync");
    });
}
