// C-ABI entry points that expose single stage kernels for parity tests
// (p2bw_kernel_*).  Device pointers in, status code out; see include/p2bw.h.
#include "capi_internal.h"
#include "kernels.h"
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
        gemm_bf16(A, B, m, n, k, e, static_cast<cudaStream_t>(stream));
    });
}
