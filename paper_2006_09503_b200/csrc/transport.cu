// Cross-process stage hand-off primitives (CUDA IPC pipelines, engine.cpp).
//
// A stage that sends to a neighbour in another process copies its staging slot
// into the neighbour's receive ring (cudaMemcpyAsync over NVLink, copy stream)
// and then bumps a sequence flag in the neighbour's receive block.  The consumer
// never polls remote memory: every flag lives in the block of the stage that
// waits on it, and the wait is a stream memory operation (cuStreamWaitValue32),
// so a waiting stream occupies no SM.  Reference ordering being reproduced:
// semantics.cpp:279 (forward needs the upstream out_act) and :301 (backward
// needs the downstream grad_to_prev).
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>
#include <string>

#include "profiler.h"
#include "transport.h"
#include "util.h"

namespace p2bw {
namespace {

__global__ void k_signal(uint32_t* flag, uint32_t value) {
    // Every write of the preceding stream work (kernels and the copy engine) is
    // complete when this kernel starts; publish it system-wide, then the flag.
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

WaitValueFn wait_fn() {
    static WaitValueFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        check_cuda(cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &p, 12000, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPointByVersion(cuStreamWaitValue32)");
        if (p == nullptr || q != cudaDriverEntryPointSuccess)
            throw Error("cuStreamWaitValue32 is unavailable in this driver");
        fn = reinterpret_cast<WaitValueFn>(p);
    });
    return fn;
}

struct FlagList {
    uint32_t* f[8];
};

__global__ void k_signal_many(FlagList l, int n, uint32_t value) {
    __threadfence_system();
    if (static_cast<int>(threadIdx.x) < n)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(l.f[threadIdx.x]), "r"(value) : "memory");
}

using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

}  // namespace

void stream_signal_many(uint32_t* const* flags, int n, uint32_t value, cudaStream_t s) {
    if (n <= 0) return;
    if (n > 8) throw Error("stream_signal_many: at most 8 flags");
    FlagList l{};
    for (int i = 0; i < n; ++i) l.f[i] = flags[i];
    k_signal_many<<<1, 32, 0, s>>>(l, n, value);
    check_cuda(cudaGetLastError(), "k_signal_many launch");
    prof::add_launches(1);
}

void* allocation_base(const void* p, size_t* offset) {
    static AddrRangeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* q = nullptr;
        cudaDriverEntryPointQueryResult r{};
        check_cuda(cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &q, 12000, cudaEnableDefault, &r),
                   "cudaGetDriverEntryPointByVersion(cuMemGetAddressRange)");
        if (q == nullptr || r != cudaDriverEntryPointSuccess) throw Error("cuMemGetAddressRange is unavailable");
        fn = reinterpret_cast<AddrRangeFn>(q);
    });
    CUdeviceptr base = 0;
    size_t size = 0;
    const CUresult e = fn(&base, &size, reinterpret_cast<CUdeviceptr>(p));
    if (e != CUDA_SUCCESS) throw Error("cuMemGetAddressRange failed: " + std::to_string(static_cast<int>(e)));
    *offset = static_cast<size_t>(reinterpret_cast<CUdeviceptr>(p) - base);
    return reinterpret_cast<void*>(base);
}

void stream_signal(uint32_t* flag, uint32_t value, cudaStream_t s) {
    k_signal<<<1, 1, 0, s>>>(flag, value);
    check_cuda(cudaGetLastError(), "k_signal launch");
    prof::add_launches(1);
}

void stream_wait_geq(const uint32_t* flag, uint32_t value, cudaStream_t s) {
    const CUresult r = wait_fn()(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), value,
                                 CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) throw Error("cuStreamWaitValue32 failed: " + std::to_string(static_cast<int>(r)));
}

}  // namespace p2bw
