// Stream-ordered flags for cross-process stage hand-offs (transport.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace p2bw {

// After all prior work on `s`: *flag = value (release, system scope; flag may be
// a peer-mapped address in another process's allocation).
void stream_signal(uint32_t* flag, uint32_t value, cudaStream_t s);
// Work enqueued on `s` after this call waits until (int32)(*flag - value) >= 0.
// `flag` is local device memory.
void stream_wait_geq(const uint32_t* flag, uint32_t value, cudaStream_t s);

}  // namespace p2bw
