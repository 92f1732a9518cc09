// Error plumbing shared by the engine, the kernels and the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace p2bw {

// Every failure inside libp2bw.so is a p2bw::Error; the C-ABI converts it to a
// nonzero status plus p2bw_last_error() text (mirrors pipesim::Error, error.hpp:9-12).
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        throw Error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
    }
}

}  // namespace p2bw
