// Error plumbing shared by the engine, the kernels and the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

namespace p2bw {

// Data-parallel replicas of one stage in a peer-memory group (Engine::join_replicas_ipc).
constexpr int kMaxReplicas = 8;

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

// A stage's streams by role ("main" = the stage stream, "fwd", "data", "side" =
// weight gradients, "update").  Lower = more urgent, clamped to the device range.
// Default: side -3, main -2, fwd -1, the rest 0 -- weight-gradient GEMMs take the SMs
// a dgrad / attention / LayerNorm tail frees, then the stage stream's chain, then the
// next Forward (BERT-base paired runs: side-first +0.6-0.8% over equal priorities;
// fwd above data / update a further ~+0.3%; main or side demoted: -1.2 to -1.8%).
// P2BW_STREAM_PRIO="main=-2,fwd=-1,..." replaces the whole table (omitted roles: 0).
inline cudaStream_t make_stage_stream(const char* role) {
    int prio = std::strcmp(role, "side") == 0   ? -3
               : std::strcmp(role, "main") == 0 ? -2
               : std::strcmp(role, "fwd") == 0  ? -1
                                                : 0;
    if (const char* e = std::getenv("P2BW_STREAM_PRIO")) {
        prio = 0;
        const size_t n = std::strlen(role);
        for (const char* p = e; p && *p;) {
            if (std::strncmp(p, role, n) == 0 && p[n] == '=') {
                prio = std::atoi(p + n + 1);
                break;
            }
            p = std::strchr(p, ',');
            if (p) ++p;
        }
    }
    int least = 0, greatest = 0;
    check_cuda(cudaDeviceGetStreamPriorityRange(&least, &greatest), "cudaDeviceGetStreamPriorityRange");
    if (prio < greatest) prio = greatest;
    if (prio > least) prio = least;
    cudaStream_t s = nullptr;
    check_cuda(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio), (std::string("cudaStreamCreate(") + role + ")").c_str());
    return s;
}

}  // namespace p2bw
