// pipesim semantics API (semantics.hpp) on top of the B200 stage executor.
// Host-side pieces (Mat helpers, ToyModel::make's splitmix64 generator) restate
// reference core/src/semantics.cpp; every trainer entry point reaches the GPU
// only through the C-ABI in include/p2bw.h.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <sstream>

#include "p2bw.h"
#include "pipesim/semantics.hpp"

namespace pipesim {

namespace {

void ok(int status) {
    if (status != P2BW_OK) throw Error(p2bw_last_error());
}

// splitmix64 (semantics.cpp:64-75): uniform doubles in [-0.5, 0.5).
class SplitMix64 {
public:
    explicit SplitMix64(std::uint64_t seed) : s_(seed) {}
    std::uint64_t bits() {
        std::uint64_t z = (s_ += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(bits() >> 11) * (1.0 / 9007199254740992.0) - 0.5; }

private:
    std::uint64_t s_;
};

Mat uniform_mat(int r, int c, SplitMix64& g) {
    Mat m(r, c);
    for (double& v : m.data) v = g.uniform();
    return m;
}

// I + scale * U[-0.5, 0.5)  (semantics.cpp:91-94, 98-100)
Mat near_identity(int n, double scale, SplitMix64& g) {
    Mat m = uniform_mat(n, n, g);
    for (double& v : m.data) v *= scale;
    for (int i = 0; i < n; ++i) m.at(i, i) += 1.0;
    return m;
}

// Stage devices from P2BW_DEVICES ("0,1,2,..."); empty -> all on the current device.
std::vector<int> stage_devices(int depth) {
    std::vector<int> devs;
    if (const char* env = std::getenv("P2BW_DEVICES")) {
        std::stringstream ss(env);
        std::string tok;
        while (std::getline(ss, tok, ',')) devs.push_back(std::stoi(tok));
        if (devs.empty()) return {};
        std::vector<int> out;
        for (int s = 0; s < depth; ++s) out.push_back(devs[static_cast<size_t>(s) % devs.size()]);
        return out;
    }
    return {};
}

struct EngineHandle {
    p2bw_engine* e = nullptr;
    ~EngineHandle() { p2bw_engine_destroy(e); }
};

struct Run {
    PipelinedResult result;
    std::vector<double> losses;  // per microbatch
};

// The linear-chain model executed by the GPU engine: fp64 parity mode, or the bf16
// production path; loop_scaling selects reference_loop's 1/m gradient scaling.
Run run_on_engine(const ToyModel& model, const TrainerConfig& cfg, PipelinePolicy policy,
                  int depth, bool want_losses, EnginePrecision precision = EnginePrecision::Fp64Exact,
                  bool loop_scaling = false) {
    cfg.validate();
    const int layers = model.num_layers();
    if (depth < 1 || layers % depth != 0)
        throw Error("block count " + std::to_string(layers) + " not divisible by depth " +
                    std::to_string(depth));
    const int m = cfg.microbatches_per_batch;
    const int total = m * cfg.num_batches;
    if (static_cast<int>(model.dataset.size()) < total)
        throw Error("toy dataset has too few microbatches for the requested run");
    const int per = layers / depth;
    const int b = model.microbatch_samples();
    const size_t act = static_cast<size_t>(model.dim) * b;
    const size_t mat = static_cast<size_t>(model.dim) * model.dim;

    const std::vector<int> devs = stage_devices(depth);
    p2bw_desc d{};
    d.model_kind = precision == EnginePrecision::Bf16TensorCore ? P2BW_MODEL_LINEAR_BF16 : P2BW_MODEL_LINEAR_F64;
    d.loop_scaling = loop_scaling ? 1 : 0;
    d.policy = static_cast<int>(policy);
    d.depth = depth;
    d.width = 1;
    d.microbatches = m;
    d.microbatch_size = b;
    d.layers = layers;
    d.dim = model.dim;
    d.learning_rate = cfg.learning_rate;
    d.momentum = cfg.momentum;
    d.devices = devs.empty() ? nullptr : devs.data();
    EngineHandle h;
    ok(p2bw_engine_create(&d, &h.e));

    std::vector<double> buf(per * mat);
    for (int s = 0; s < depth; ++s) {
        for (int l = 0; l < per; ++l) {
            const Mat& w = model.init_weights[static_cast<size_t>(s * per + l)];
            std::copy(w.data.begin(), w.data.end(), buf.begin() + static_cast<long>(l * mat));
        }
        ok(p2bw_engine_load_stage_weights(h.e, s, buf.data(), buf.size() * sizeof(double)));
    }
    std::vector<double> xs(static_cast<size_t>(total) * act), ys(xs.size());
    for (int k = 0; k < total; ++k) {
        const auto& [x, y] = model.dataset[static_cast<size_t>(k)];
        std::copy(x.data.begin(), x.data.end(), xs.begin() + static_cast<long>(k * act));
        std::copy(y.data.begin(), y.data.end(), ys.begin() + static_cast<long>(k * act));
    }
    ok(p2bw_engine_set_data(h.e, xs.data(), ys.data(), 1, total));
    ok(p2bw_engine_run_schedule(h.e, cfg.num_batches, /*snapshot_updates=*/1));
    ok(p2bw_engine_sync(h.e));

    Run run;
    p2bw_counters c{};
    ok(p2bw_engine_counters(h.e, &c));
    run.result.version_consistent = c.version_consistent != 0;
    run.result.max_versions_held = c.max_versions_held;
    // Trajectory assembly (semantics.cpp:363-373): W^(t) = the t-th update of every stage.
    const int updates_per_batch = policy == PipelinePolicy::PipeDream1F1B ? m : 1;
    run.result.trajectory.push_back(model.init_weights);
    for (int t = 1; t <= cfg.num_batches; ++t) {
        WeightSet full;
        for (int s = 0; s < depth; ++s) {
            ok(p2bw_engine_read_snapshot(h.e, s, t * updates_per_batch, buf.data(),
                                         buf.size() * sizeof(double)));
            for (int l = 0; l < per; ++l) {
                Mat w(model.dim, model.dim);
                std::copy(buf.begin() + static_cast<long>(l * mat),
                          buf.begin() + static_cast<long>((l + 1) * mat), w.data.begin());
                full.push_back(std::move(w));
            }
        }
        run.result.trajectory.push_back(std::move(full));
    }
    if (want_losses) {
        run.losses.resize(static_cast<size_t>(total));
        ok(p2bw_engine_losses(h.e, 1, total, run.losses.data()));
    }
    return run;
}

std::vector<double> batch_losses(const std::vector<double>& per_mb, int m) {
    std::vector<double> out;
    for (size_t i = 0; i + static_cast<size_t>(m) <= per_mb.size(); i += static_cast<size_t>(m)) {
        double s = 0.0;
        for (int j = 0; j < m; ++j) s += per_mb[i + static_cast<size_t>(j)];
        out.push_back(s / m);
    }
    return out;
}

}  // namespace

// ---- host helpers of the reference API (semantics.cpp:9-59) ----------------

Mat matmul(const Mat& a, const Mat& b) {
    if (a.cols != b.rows) throw Error("matmul: shape mismatch");
    Mat c(a.rows, b.cols);
    for (int j = 0; j < b.cols; ++j)
        for (int k = 0; k < a.cols; ++k) {
            const double s = b.at(k, j);
            for (int i = 0; i < a.rows; ++i) c.at(i, j) += a.at(i, k) * s;
        }
    return c;
}

Mat matmul_tn(const Mat& a, const Mat& b) {
    if (a.rows != b.rows) throw Error("matmul_tn: shape mismatch");
    Mat c(a.cols, b.cols);
    for (int j = 0; j < b.cols; ++j)
        for (int i = 0; i < a.cols; ++i) {
            double acc = 0.0;
            for (int k = 0; k < a.rows; ++k) acc += a.at(k, i) * b.at(k, j);
            c.at(i, j) = acc;
        }
    return c;
}

Mat matmul_nt(const Mat& a, const Mat& b) {
    if (a.cols != b.cols) throw Error("matmul_nt: shape mismatch");
    Mat c(a.rows, b.rows);
    for (int j = 0; j < b.rows; ++j)
        for (int k = 0; k < a.cols; ++k) {
            const double s = b.at(j, k);
            for (int i = 0; i < a.rows; ++i) c.at(i, j) += a.at(i, k) * s;
        }
    return c;
}

void axpy(double alpha, const Mat& x, Mat& y) {
    if (x.rows != y.rows || x.cols != y.cols) throw Error("axpy: shape mismatch");
    for (size_t i = 0; i < x.data.size(); ++i) y.data[i] += alpha * x.data[i];
}

double max_rel_diff(const Mat& a, const Mat& b) {
    if (a.rows != b.rows || a.cols != b.cols) throw Error("max_rel_diff: shape mismatch");
    double worst = 0.0;
    for (size_t i = 0; i < a.data.size(); ++i) {
        const double scale = std::max({std::abs(a.data[i]), std::abs(b.data[i]), 1e-12});
        worst = std::max(worst, std::abs(a.data[i] - b.data[i]) / scale);
    }
    return worst;
}

// semantics.cpp:85-109 — weights, then the hidden target map, then x per microbatch.
ToyModel ToyModel::make(int dim, int num_layers, int microbatch_size, int num_microbatches,
                        std::uint64_t seed) {
    if (dim < 1 || num_layers < 1 || microbatch_size < 1 || num_microbatches < 1)
        throw Error("toy model dimensions must be >= 1");
    SplitMix64 g(seed);
    ToyModel model;
    model.dim = dim;
    for (int l = 0; l < num_layers; ++l) model.init_weights.push_back(near_identity(dim, 0.2, g));
    const Mat target_map = near_identity(dim, 0.3, g);
    for (int k = 0; k < num_microbatches; ++k) {
        Mat x = uniform_mat(dim, microbatch_size, g);
        Mat y = matmul(target_map, x);
        model.dataset.emplace_back(std::move(x), std::move(y));
    }
    return model;
}

// semantics.cpp:111-116
void TrainerConfig::validate() const {
    if (learning_rate < 0) throw Error("learning rate must be >= 0");
    if (momentum < 0 || momentum >= 1) throw Error("momentum must be in [0, 1)");
    if (microbatches_per_batch < 1) throw Error("m must be >= 1");
    if (num_batches < 1) throw Error("num_batches must be >= 1");
}

// ---- trainers on the GPU engine ---------------------------------------------

// Vanilla minibatch SGD == a one-stage flushed pipeline (version t-1 for batch t),
// with reference_loop's per-microbatch 1/m scaling (semantics.cpp:145): bit-identical
// to the reference for every m.
Trajectory reference_vanilla(const ToyModel& model, const TrainerConfig& cfg) {
    return run_on_engine(model, cfg, PipelinePolicy::GPipe, 1, false, EnginePrecision::Fp64Exact, true)
        .result.trajectory;
}

// Delay-1 SGD == a one-stage 2BW pipeline (version max(t-2,0) for batch t).
Trajectory reference_2bw(const ToyModel& model, const TrainerConfig& cfg) {
    return run_on_engine(model, cfg, PipelinePolicy::TwoBW, 1, false, EnginePrecision::Fp64Exact, true)
        .result.trajectory;
}

PipelinedResult pipelined_execute(const ToyModel& model, const TrainerConfig& cfg,
                                  PipelinePolicy policy, int depth) {
    return run_on_engine(model, cfg, policy, depth, false).result;
}

PipelinedResult pipelined_execute(const ToyModel& model, const TrainerConfig& cfg,
                                  PipelinePolicy policy, int depth, EnginePrecision precision) {
    return run_on_engine(model, cfg, policy, depth, false, precision).result;
}

// semantics.cpp:377-388, with per-batch losses measured by the engine's forward passes.
LossCurves loss_curve_compare(const ToyModel& model, const TrainerConfig& cfg) {
    LossCurves curves;
    const int m = cfg.microbatches_per_batch;
    curves.vanilla = batch_losses(
        run_on_engine(model, cfg, PipelinePolicy::GPipe, 1, true, EnginePrecision::Fp64Exact, true).losses, m);
    curves.twobw = batch_losses(
        run_on_engine(model, cfg, PipelinePolicy::TwoBW, 1, true, EnginePrecision::Fp64Exact, true).losses, m);
    for (double v : curves.vanilla) curves.loss_scale = std::max(curves.loss_scale, v);
    for (size_t i = curves.vanilla.size() / 2; i < curves.vanilla.size(); ++i)
        curves.tail_max_gap = std::max(curves.tail_max_gap, std::abs(curves.vanilla[i] - curves.twobw[i]));
    return curves;
}

}  // namespace pipesim
