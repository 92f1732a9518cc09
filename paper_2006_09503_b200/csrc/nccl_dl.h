// Run-time-loaded NCCL (see nccl_dl.cpp).  Types come from the system nccl.h.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>

namespace p2bw {

ncclUniqueId nccl_unique_id();
ncclComm_t nccl_comm_init(const ncclUniqueId& id, int nranks, int rank);
void nccl_comm_destroy(ncclComm_t c);
void nccl_allreduce_sum(void* buf, size_t count, ncclDataType_t dt, ncclComm_t c, cudaStream_t s);

}  // namespace p2bw
