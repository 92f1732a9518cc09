// B200 block profiler -> the reference's profile document (block_profiler.cpp).
#pragma once

#include <string>
#include <vector>

#include "engine.h"

namespace p2bw {

// Times every transformer block of `base` (one layer per block; embedding folded into
// block 0, LM head + loss into the last) at each microbatch size and returns the
// document load_model_profile (profile.cpp:162-193) reads.
std::string profile_transformer_blocks(const EngineConfig& base, const std::vector<int>& sizes, int warmup,
                                       int iters, const std::string& name);

}  // namespace p2bw
