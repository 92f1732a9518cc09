// Transformer stage (placeholder until the block kernels land).
#include "engine.h"

namespace p2bw {

std::unique_ptr<StageModel> make_transformer_stage(const EngineConfig&, int, int, int, int, int) {
    throw Error("transformer stages are not built yet");
}

}  // namespace p2bw
