/*
 * p2bw.h — C-ABI of libp2bw.so, the B200-native PipeDream-2BW engine.
 *
 * This is the drop-in boundary for the reference's pipelined training path
 * (pipesim, /root/reference/proj/core/include/pipesim/*.hpp).  The reference
 * has no FFI of its own; every entry point below names the C++ interface it
 * replaces (file:line, relative to /root/reference/proj).  Plain pointers and
 * sizes only: no torch / C++ types cross this boundary.
 *
 * Conventions
 *   - Every function returns P2BW_OK (0) or a nonzero status; the message of
 *     the last failure on the calling thread is p2bw_last_error().  The message
 *     text keeps the reference's pipesim::Error wording (core/include/pipesim/
 *     error.hpp:9-12) so callers can rethrow it unchanged.
 *   - Host buffers are borrowed for the duration of the call only.
 *   - An engine is not reentrant (the reference is single-threaded,
 *     SPEC.md:83); internally it drives one CUDA stream per pipeline stage.
 */
#ifndef P2BW_H
#define P2BW_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define P2BW_OK 0
#define P2BW_ERR 1     /* pipesim::Error equivalent (invariant / infeasible / CUDA failure) */
#define P2BW_ERR_ARG 2 /* malformed argument */

/* ---- library ------------------------------------------------------------ */

const char* p2bw_last_error(void);
const char* p2bw_version(void);

/* ---- policies and ops: schedule.hpp:10-51 ---------------------------------- */

/* == pipesim::PipelinePolicy (schedule.hpp:10-16), same order. */
enum {
    P2BW_POLICY_NONE = 0,
    P2BW_POLICY_GPIPE = 1,
    P2BW_POLICY_1F1B = 2,
    P2BW_POLICY_FLUSH = 3,
    P2BW_POLICY_2BW = 4
};

/* == pipesim::OpKind (schedule.hpp:21-32), same order. */
enum {
    P2BW_OP_FORWARD = 0,
    P2BW_OP_BACKWARD = 1,
    P2BW_OP_RECOMPUTE = 2,
    P2BW_OP_UPDATE = 3,
    P2BW_OP_FLUSH = 4,
    P2BW_OP_ACT_SEND = 5,
    P2BW_OP_ACT_RECV = 6,
    P2BW_OP_GRAD_SEND = 7,
    P2BW_OP_GRAD_RECV = 8,
    P2BW_OP_ALLREDUCE = 9
};

#define P2BW_LATEST_VERSION (-1) /* == pipesim::kLatestVersion (schedule.hpp:36) */

/* == pipesim::ScheduledOp (schedule.hpp:40-46). */
typedef struct {
    int kind;
    int microbatch;
    int weight_version;
} p2bw_op;

/* ---- stage kernels (parity-test hooks; device pointers, CUDA stream) ------- */

/* Epilogue of p2bw_kernel_gemm_bf16. kind: 0 = bf16 store with optional
 * bias / GELU (pre-activation copy in preact) / residual; 1 = fp32
 * D = beta*D + alpha*acc (wgrad accumulation, semantics.cpp:329);
 * 2 = bf16 D = alpha*acc*gelu'(aux). */
typedef struct {
    int kind;
    void* d;
    long long ldd;
    const void* bias;
    const void* residual;
    long long ldr;
    void* preact;
    int gelu;
    const void* aux;
    float alpha;
    float beta;
} p2bw_gemm_epilogue;

/* D[m x n] = A[m x k] . B[n x k]^T on tcgen05 tensor cores (bf16 in, fp32 acc).
 * major 0: element (r,k) at ptr[r*ld+k]; major 1: at ptr[k*ld+r].
 * Replaces matmul / matmul_tn / matmul_nt (semantics.hpp:23-25). */
int p2bw_kernel_gemm_bf16(const void* a, long long lda, int a_major, const void* b,
                          long long ldb, int b_major, int m, int n, int k,
                          const p2bw_gemm_epilogue* epi, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* P2BW_H */
