// Host-side launch interface of the sm_100a stage kernels.  Internal to
// libp2bw.so: the engine (engine.cpp) and the C-ABI test hooks (capi.cpp)
// call these; nothing outside the library sees them.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace p2bw {

using bf16 = __nv_bfloat16;

// Storage order of a GEMM operand relative to its (row, k) indexing.
//   K  : element (r, k) at ptr[r * ld + k]   (k contiguous)
//   MN : element (r, k) at ptr[k * ld + r]   (r contiguous)
enum class Major : int { K = 0, MN = 1 };

struct GemmOperand {
    const bf16* ptr = nullptr;
    int64_t ld = 0;
    Major major = Major::K;
};

enum class EpiKind : int {
    StoreBF16 = 0,  // D_bf16 = [gelu](alpha*acc + bias) [+ residual]; preact stored before gelu
    StoreF32 = 1,   // D_f32 = beta*D_f32 + alpha*acc
    DGeluBF16 = 2,  // D_bf16 = alpha*acc * gelu'(u)
};

struct GemmEpilogue {
    EpiKind kind = EpiKind::StoreBF16;
    void* d = nullptr;
    int64_t ldd = 0;
    const bf16* bias = nullptr;      // [N]
    const bf16* residual = nullptr;  // [M x ldr]
    int64_t ldr = 0;
    bf16* preact = nullptr;          // [M x ldd] pre-GELU copy (StoreBF16 with gelu)
    bool gelu = false;
    const bf16* aux = nullptr;       // u for DGeluBF16, [M x ldd]
    float alpha = 1.0f;
    float beta = 0.0f;
    // Optional fp32 [M x N] workspace: a plain bf16 store (no bias / GELU / residual)
    // with few output tiles and a long K may then run split-K into it and be cast.
    float* workspace = nullptr;
    int64_t workspace_floats = 0;
    // The bias gradient of the layer whose output gradient A is, summed from the A tiles
    // already in SMEM by two otherwise idle warps (single-CTA tiles):
    //   A MN-major (wgrad, fp32 store): bias_grad[r] (=|+=) sum over K of A[r, :];
    //     bias_scratch >= splits * M floats (splits <= K / 512);
    //   A K-major (dgrad, any store): bias_grad[c] (=|+=) sum over M of A[:, c];
    //     bias_scratch >= 2 * ceil(M / 128) * K floats.
    float* bias_grad = nullptr;
    bool bias_grad_accumulate = false;
    float* bias_scratch = nullptr;
    int64_t bias_scratch_floats = 0;
};

// D[M x N] = A[M x K] . B[N x K]^T on tcgen05 (TMA -> SMEM -> UMMA -> TMEM -> epilogue).
// Requirements: N % 32 == 0, leading dims multiple of 8 elements, 16-byte aligned pointers.
// Debug: per-CTA phase timestamps of the GEMM kernel (8 u64 per CTA; null = off).
void gemm_debug_timing(unsigned long long* dev_buf);
// The main-path launch plan of gemm_bf16 for a shape: {BN, cluster, split-K, tail K
// parts (1 = no tail split)}.  (The plain-bf16 workspace split-K path is not included.)
void gemm_plan(int m, int n, int k, bool amn, bool bmn, bool f32, bool bias_grad, int out[4]);

void gemm_bf16(const GemmOperand& a, const GemmOperand& b, int m, int n, int k,
               const GemmEpilogue& epi, cudaStream_t stream);

int num_sms();

}  // namespace p2bw
