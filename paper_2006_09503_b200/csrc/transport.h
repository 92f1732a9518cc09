// Stream-ordered flags for cross-process stage hand-offs (transport.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace p2bw {

// After all prior work on `s`: *flag = value (release, system scope; flag may be
// a peer-mapped address in another process's allocation).
void stream_signal(uint32_t* flag, uint32_t value, cudaStream_t s);
// Work enqueued on `s` after this call waits until (int32)(*flag - value) >= 0.
// `flag` is local device memory.
// After all prior work on `s`: *flags[i] = value for i < n (n <= 8), one launch.
void stream_signal_many(uint32_t* const* flags, int n, uint32_t value, cudaStream_t s);
// Base of the cudaMalloc allocation holding p (for CUDA IPC export) and p's offset in it.
void* allocation_base(const void* p, size_t* offset);
void stream_wait_geq(const uint32_t* flag, uint32_t value, cudaStream_t s);

}  // namespace p2bw
