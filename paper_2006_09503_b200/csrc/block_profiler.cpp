// B200 block profiler: measures the per-block costs the reference planner consumes
// and writes them as the reference's profile document (profile.cpp:162-193,
// load_model_profile), closing the loop  B200 kernels -> ModelProfile -> plan().
//
// The reference's profile is a list of blocks with per-microbatch-size tables
// fwd_ms / bwd_ms / act_total_bytes / act_input_bytes / act_boundary_bytes and a
// scalar weight_bytes (profile.hpp:18-28).  Here a block is one transformer layer;
// the embedding is folded into block 0 and the final LayerNorm + LM head + loss into
// the last block (that is where partition_equal puts them, profile.cpp:104-131).
//
// Each microbatch size b is timed on three one-layer stage models of a depth-3
// pipeline -- first (embedding + layer), middle (layer only), last (layer + head) --
// running the same Forward / Backward code the engine issues for a real stage, with
// CUDA events on the stage stream around `iters` repetitions after `warmup` ones.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <nlohmann/json.hpp>
#include <string>
#include <vector>

#include "block_profiler.h"
#include "engine.h"

namespace p2bw {
namespace {

using json = nlohmann::json;

struct Timed {
    double fwd_ms = 0.0, bwd_ms = 0.0;
};

struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) { check_cuda(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc(profile)"); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// Deterministic small-magnitude bf16 fill (a random-looking activation / gradient).
void fill_pattern(void* p, size_t bytes, cudaStream_t s) {
    std::vector<uint16_t> host(bytes / 2);
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (auto& v : host) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        // bf16 in [-0.5, 0.5): sign | exponent 0x3E/0x3F range | mantissa
        const uint16_t mant = static_cast<uint16_t>(x & 0x7F);
        const uint16_t exp = static_cast<uint16_t>(0x7C + ((x >> 8) & 0x1));
        v = static_cast<uint16_t>(((x >> 9) & 1) << 15 | exp << 7 | mant);
    }
    check_cuda(cudaMemcpyAsync(p, host.data(), bytes, cudaMemcpyHostToDevice, s), "H2D profile fill");
    check_cuda(cudaStreamSynchronize(s), "profile fill sync");
}

Timed time_stage(StageModel& m, bool first, bool last, size_t boundary, int warmup, int iters, cudaStream_t s) {
    DevBuf xin(boundary), xout(boundary), gin(boundary), gout(boundary);
    fill_pattern(xin.p, boundary, s);
    fill_pattern(gin.p, boundary, s);
    cudaEvent_t e[3];
    for (auto& ev : e) check_cuda(cudaEventCreate(&ev), "cudaEventCreate");
    auto fwd = [&] { m.forward(1, 0, 0, first ? nullptr : xin.p, last ? nullptr : xout.p, s); };
    auto bwd = [&] { m.backward(1, 0, 0, last ? nullptr : gin.p, first ? nullptr : gout.p, true, s); };
    for (int i = 0; i < warmup; ++i) {
        fwd();
        bwd();
    }
    // forwards timed back to back, then backwards (each backward re-reads the stash of
    // the last forward, which is what it reads inside a pipeline too)
    check_cuda(cudaEventRecord(e[0], s), "event");
    for (int i = 0; i < iters; ++i) fwd();
    check_cuda(cudaEventRecord(e[1], s), "event");
    for (int i = 0; i < iters; ++i) bwd();
    check_cuda(cudaEventRecord(e[2], s), "event");
    check_cuda(cudaEventSynchronize(e[2]), "event sync");
    float f = 0.0f, b = 0.0f;
    check_cuda(cudaEventElapsedTime(&f, e[0], e[1]), "elapsed");
    check_cuda(cudaEventElapsedTime(&b, e[1], e[2]), "elapsed");
    for (auto& ev : e) cudaEventDestroy(ev);
    return Timed{f / iters, b / iters};
}

}  // namespace

std::string profile_transformer_blocks(const EngineConfig& base, const std::vector<int>& sizes, int warmup,
                                       int iters, const std::string& name) {
    if (base.model_kind != P2BW_MODEL_TRANSFORMER) throw Error("block profiler: transformer models only");
    if (base.layers < 1) throw Error("block profiler: layers must be >= 1");
    if (sizes.empty()) throw Error("block profiler: no microbatch sizes");
    if (iters < 1 || warmup < 0) throw Error("block profiler: iters must be >= 1");
    for (int b : sizes)
        if (b < 1) throw Error("block profiler: microbatch sizes must be >= 1");
    const int L = base.layers;
    const double h = base.hidden, seq = base.seq_len, V = base.vocab, heads = base.heads;
    const double rows_per_seq = base.head_rows > 0 ? base.head_rows : seq;
    const double vp = std::ceil(V / 128.0) * 128.0;
    // parameters (the flat fp32 layout of model_transformer.cu, 64-element aligned tensors)
    auto al = [](double n) { return std::ceil(n / 64.0) * 64.0; };
    const double layer_params = 4 * al(h) + al(3 * h * h) + al(3 * h) + al(h * h) + al(h) + al(4 * h * h) +
                                al(4 * h) + al(4 * h * h) + al(h);
    const double emb_params = al(vp * h) + al(seq * h);
    const double head_params = 2 * al(h) + al(vp * h);
    // weight_bytes: the cost model charges required_versions x weight_bytes per stage
    // (costmodel.cpp:93-99) and has no term for optimizer or gradient state, so the field
    // carries the 2BW stage's whole parameter state split over its two versions: fp32
    // master + momentum (8 B) + two fp32 coalesced-gradient buffers (8 B) + two bf16
    // versions (4 B) = 20 B/param / 2.  (allreduce_seconds, costmodel.cpp:23-27, then
    // prices 10 B/param where NCCL moves the 4 B/param fp32 gradient: conservative.)
    constexpr double kBytesPerParam = 10.0;

    cudaStream_t s = nullptr;
    check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate(profile)");
    std::vector<Timed> tf, tm, tl;
    try {
        for (int b : sizes) {
            EngineConfig c = base;
            c.microbatch_size = b;
            c.depth = 3;
            c.layers = 3;
            c.microbatches = 1;
            auto first = make_transformer_stage(c, 0, 0, 1, 1, 1);
            auto mid = make_transformer_stage(c, 1, 1, 2, 1, 1);
            auto last = make_transformer_stage(c, 2, 2, 3, 1, 1);
            const int T = b * base.seq_len;
            const int R = static_cast<int>(b * rows_per_seq);
            std::vector<int> ids(static_cast<size_t>(T)), tg(static_cast<size_t>(R));
            uint64_t x = base.seed * 2654435761ull + 12345;
            for (auto& v : ids) v = static_cast<int>((x = x * 6364136223846793005ull + 1442695040888963407ull) >> 33) % base.vocab;
            for (auto& v : tg) v = static_cast<int>((x = x * 6364136223846793005ull + 1442695040888963407ull) >> 33) % base.vocab;
            for (auto* m : {first.get(), mid.get(), last.get()}) {
                m->bind_stream(s);
                m->init_weights(base.seed);
                m->set_data(ids.data(), tg.data(), 1, 1);
            }
            const size_t boundary = mid->boundary_bytes();
            tf.push_back(time_stage(*first, true, false, boundary, warmup, iters, s));
            tm.push_back(time_stage(*mid, false, false, boundary, warmup, iters, s));
            tl.push_back(time_stage(*last, false, true, boundary, warmup, iters, s));
            check_cuda(cudaStreamSynchronize(s), "profile sync");
        }
    } catch (...) {
        cudaStreamDestroy(s);
        throw;
    }
    cudaStreamDestroy(s);

    json doc;
    doc["model"] = name;
    doc["blocks"] = json::array();
    for (int l = 0; l < L; ++l) {
        json fwd = json::object(), bwd = json::object(), at = json::object(), ai = json::object(),
             ab = json::object();
        for (size_t k = 0; k < sizes.size(); ++k) {
            const int b = sizes[k];
            const std::string key = std::to_string(b);
            double f = tm[k].fwd_ms, bw = tm[k].bwd_ms;
            if (l == 0) f += tf[k].fwd_ms - tm[k].fwd_ms, bw += tf[k].bwd_ms - tm[k].bwd_ms;
            if (l == L - 1) f += tl[k].fwd_ms - tm[k].fwd_ms, bw += tl[k].bwd_ms - tm[k].bwd_ms;
            fwd[key] = std::max(f, 1e-6);
            bwd[key] = std::max(bw, 1e-6);
            const double T = static_cast<double>(b) * seq;
            const double R = static_cast<double>(b) * rows_per_seq;
            // the stash slot of model_transformer.cu: 16 bf16 [T x h]-sized tensors
            // (x, LN1, qkv (3), attn out, x1, LN2, u (4), gelu (4)), LN stats, lse
            double act = 32.0 * T * h + 16.0 * T + 4.0 * b * heads * seq;
            if (l == L - 1) act += 2.0 * T * h + 4.0 * R * h + 2.0 * R * vp + 8.0 * R;  // xl, head rows, LNf, logits
            at[key] = act;
            ai[key] = 2.0 * T * h;
            ab[key] = 4.0 * T * h;
        }
        double params = layer_params;
        if (l == 0) params += emb_params;
        if (l == L - 1) params += head_params;
        doc["blocks"].push_back({{"fwd_ms", fwd},
                                 {"bwd_ms", bwd},
                                 {"weight_bytes", params * kBytesPerParam},
                                 {"act_total_bytes", at},
                                 {"act_input_bytes", ai},
                                 {"act_boundary_bytes", ab}});
    }
    return doc.dump(2);
}

}  // namespace p2bw
