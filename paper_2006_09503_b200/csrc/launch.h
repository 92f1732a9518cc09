// Kernel launches with Programmatic Dependent Launch (PDL).
//
// A stage issues ~1300 dependent kernels per batch on each stream.  Launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, a kernel's CTAs may be
// scheduled as soon as every CTA of the previous kernel on the stream has executed
// griddepcontrol.launch_dependents (pdl_begin, at the top of every hot kernel) --
// i.e. onto the SMs the previous kernel's ragged last wave leaves idle -- and then
// run their local prologue (barriers, TMEM allocation, descriptor prefetch) before
// griddepcontrol.wait blocks them until the previous grid has completed and its
// memory is visible (pdl_wait, before any global access).
//
// Measured on BERT-base (bench.py): with the early trigger, waiting dependent CTAs
// hold the SMs a kernel's tail frees, which the stage's other streams (forward,
// weight-gradient side stream) use better: -1.7%.  With the trigger at exit (the
// implicit one) the next kernel's launch is prepared while this one drains: neutral
// before the stream priorities, +0.7% (8 paired same-box runs, every pair positive)
// with them.  So PDL launches are the default (P2BW_PDL=0 switches them off); the
// early trigger is compiled in only with -DP2BW_PDL_EARLY_TRIGGER.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

#include "util.h"

namespace p2bw {

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("P2BW_PDL");
        return e == nullptr || e[0] != '0';
    }();
    return on;
}

// cudaLaunchKernelEx with the PDL attribute (and an optional 1-D cluster).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, const char* what,
                Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    check_cuda(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), what);
}

}  // namespace p2bw
