// C entry points over the REFERENCE pipesim library (test infrastructure).
// Compiled together with /root/reference/proj/core/src/*.cpp into
// oracle/_ref/libpipesim_ref.so by oracle/Makefile; used only by tests/ and by
// bench.py's reference / cpu_baseline arm, never by the product path.
#include <cstdlib>
#include <cstring>
#include <string>

#include "pipesim/planner.hpp"
#include "pipesim/profile.hpp"
#include "pipesim/schedule.hpp"
#include "pipesim/semantics.hpp"

namespace {
thread_local std::string g_err;

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

pipesim::TrainerConfig trainer(double lr, double beta, int m, int T) {
    pipesim::TrainerConfig c;
    c.learning_rate = lr;
    c.momentum = beta;
    c.microbatches_per_batch = m;
    c.num_batches = T;
    return c;
}

void flatten(const pipesim::Trajectory& traj, double* out) {
    size_t off = 0;
    for (const auto& ws : traj)
        for (const auto& w : ws) {
            std::memcpy(out + off, w.data.data(), w.data.size() * sizeof(double));
            off += w.data.size();
        }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

int ref_weight_version_2bw(int k, int m, int* out) {
    return guard([&] { *out = pipesim::weight_version_2bw(k, m); });
}

int ref_schedule_text(int policy, int d, int m, int T, char** out) {
    return guard([&] {
        *out = dup(pipesim::serialize_programs(
            pipesim::generate_schedule(static_cast<pipesim::PipelinePolicy>(policy), d, m, T)));
    });
}

int ref_plan_json(const char* model_json, const char* cluster_json, long long max_batch,
                  int policy, int as_text, char** out) {
    return guard([&] {
        const auto r = pipesim::plan(pipesim::load_model_profile(model_json),
                                     pipesim::load_cluster_spec(cluster_json), max_batch,
                                     static_cast<pipesim::PipelinePolicy>(policy));
        *out = dup(as_text ? pipesim::plan_to_text(r) : pipesim::plan_to_json(r));
    });
}

// ToyModel::make: weights [L][dim*dim], x/y [nmb][dim*b] (column-major).
int ref_toy_make(int dim, int layers, int b, int nmb, unsigned long long seed, double* w,
                 double* x, double* y) {
    return guard([&] {
        const auto model = pipesim::ToyModel::make(dim, layers, b, nmb, seed);
        for (int l = 0; l < layers; ++l)
            std::memcpy(w + static_cast<size_t>(l) * dim * dim, model.init_weights[l].data.data(),
                        sizeof(double) * dim * dim);
        for (int k = 0; k < nmb; ++k) {
            std::memcpy(x + static_cast<size_t>(k) * dim * b, model.dataset[k].first.data.data(),
                        sizeof(double) * dim * b);
            std::memcpy(y + static_cast<size_t>(k) * dim * b, model.dataset[k].second.data.data(),
                        sizeof(double) * dim * b);
        }
    });
}

// pipelined_execute on ToyModel::make(dim, layers, b, m*T, seed); trajectory out:
// (T+1) x layers x dim*dim doubles.
int ref_pipelined_execute(int dim, int layers, int b, unsigned long long seed, double lr,
                          double beta, int m, int T, int policy, int depth, double* traj,
                          int* version_consistent, int* max_versions_held) {
    return guard([&] {
        const auto model = pipesim::ToyModel::make(dim, layers, b, m * T, seed);
        const auto r = pipesim::pipelined_execute(model, trainer(lr, beta, m, T),
                                                  static_cast<pipesim::PipelinePolicy>(policy), depth);
        if (traj) flatten(r.trajectory, traj);
        if (version_consistent) *version_consistent = r.version_consistent ? 1 : 0;
        if (max_versions_held) *max_versions_held = r.max_versions_held;
    });
}

// reference_vanilla (delayed=0) / reference_2bw (delayed=1).
int ref_reference_loop(int dim, int layers, int b, unsigned long long seed, double lr,
                       double beta, int m, int T, int delayed, double* traj) {
    return guard([&] {
        const auto model = pipesim::ToyModel::make(dim, layers, b, m * T, seed);
        const auto cfg = trainer(lr, beta, m, T);
        flatten(delayed ? pipesim::reference_2bw(model, cfg) : pipesim::reference_vanilla(model, cfg),
                traj);
    });
}

}  // extern "C"
