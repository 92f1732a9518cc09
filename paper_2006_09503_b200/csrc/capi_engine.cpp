// C-ABI over the stage executor (include/p2bw.h, "the stage executor").
#include <algorithm>
#include <cstring>
#include <memory>

#include "capi_internal.h"
#include "block_profiler.h"
#include "engine.h"
#include "nccl_dl.h"
#include "p2bw.h"
#include "pipesim/schedule.hpp"

struct p2bw_engine {
    std::unique_ptr<p2bw::Engine> impl;
};

using p2bw::guarded;

namespace {

p2bw::Engine& eng_of(p2bw_engine* e) {
    if (e == nullptr || !e->impl) throw std::invalid_argument("engine is NULL");
    return *e->impl;
}

void check_stage(p2bw::Engine& e, int stage) {
    if (stage < 0 || stage >= e.depth()) throw std::invalid_argument("stage out of range");
}

p2bw::EngineConfig config_from_desc(const p2bw_desc& dd) {
    const p2bw_desc* d = &dd;
    p2bw::EngineConfig c;
    c.model_kind = d->model_kind;
    c.policy = d->policy;
    c.depth = d->depth;
    c.microbatches = d->microbatches;
    c.microbatch_size = d->microbatch_size;
    c.layers = d->layers;
    c.dim = d->dim;
    c.hidden = d->hidden;
    c.heads = d->heads;
    c.seq_len = d->seq_len;
    c.vocab = d->vocab;
    c.causal = d->causal;
    c.head_rows = d->head_rows;
    c.lr = d->learning_rate;
    c.momentum = d->momentum;
    c.seed = d->seed;
    if (d->devices != nullptr) c.devices.assign(d->devices, d->devices + d->depth);
    c.first_local = d->first_local_stage;
    c.local_count = d->local_stages;
    c.recompute = d->recompute != 0;
    c.optimizer = d->optimizer;
    c.loop_scaling = d->loop_scaling != 0;
    if (d->stage_layers != nullptr) c.stage_layers.assign(d->stage_layers, d->stage_layers + d->depth);
    if (c.loop_scaling && c.model_kind != P2BW_MODEL_LINEAR_F64)
        throw p2bw::Error("loop_scaling applies to the fp64 linear chain only");
    if (c.optimizer != P2BW_OPT_MOMENTUM_SGD && c.optimizer != P2BW_OPT_ADAM)
        throw std::invalid_argument("unknown optimizer " + std::to_string(c.optimizer));
    if (c.optimizer == P2BW_OPT_ADAM) {
        c.beta2 = d->beta2;
        c.eps = d->eps;
        if (!(c.beta2 >= 0 && c.beta2 < 1) || !(c.eps > 0)) throw p2bw::Error("Adam needs beta2 in [0, 1) and eps > 0");
        if (c.model_kind != P2BW_MODEL_TRANSFORMER) throw p2bw::Error("Adam is available for transformer stages only");
    }
    if (c.lr < 0) throw p2bw::Error("learning rate must be >= 0");
    if (c.momentum < 0 || c.momentum >= 1) throw p2bw::Error("momentum must be in [0, 1)");
    return c;
}

}  // namespace

extern "C" {

int p2bw_engine_create(const p2bw_desc* d, p2bw_engine** out) {
    return guarded([&] {
        if (d == nullptr || out == nullptr) throw std::invalid_argument("NULL argument");
        if (d->width != 1 && d->width != 0)
            throw p2bw::Error("width > 1 runs one replica per process (see DESIGN.md); "
                              "this engine instance drives a single pipeline");
        auto e = std::make_unique<p2bw_engine>();
        e->impl = std::make_unique<p2bw::Engine>(config_from_desc(*d));
        *out = e.release();
    });
}

int p2bw_profile_blocks(const p2bw_desc* d, const int* microbatch_sizes, int n_sizes, int warmup, int iters,
                        const char* name, char** out_json) {
    return guarded([&] {
        if (d == nullptr || microbatch_sizes == nullptr || out_json == nullptr)
            throw std::invalid_argument("NULL argument");
        if (n_sizes < 1) throw std::invalid_argument("no microbatch sizes");
        const std::vector<int> sizes(microbatch_sizes, microbatch_sizes + n_sizes);
        *out_json = p2bw::dup_string(p2bw::profile_transformer_blocks(config_from_desc(*d), sizes, warmup, iters,
                                                                      name ? name : "p2bw-transformer"));
    });
}

void p2bw_engine_destroy(p2bw_engine* eng) { delete eng; }

int p2bw_engine_stage_weight_bytes(p2bw_engine* eng, int stage, size_t* bytes) {
    return guarded([&] {
        auto& e = eng_of(eng);
        check_stage(e, stage);
        if (bytes == nullptr) throw std::invalid_argument("bytes is NULL");
        *bytes = e.model(stage).weight_bytes_public();
    });
}

int p2bw_engine_load_stage_weights(p2bw_engine* eng, int stage, const void* host, size_t bytes) {
    return guarded([&] {
        auto& e = eng_of(eng);
        check_stage(e, stage);
        if (host == nullptr) throw std::invalid_argument("host buffer is NULL");
        e.load_stage_weights(stage, host, bytes);
    });
}

int p2bw_engine_init_weights(p2bw_engine* eng) {
    return guarded([&] {
        auto& e = eng_of(eng);
        for (int s = 0; s < e.depth(); ++s)
            if (e.is_local(s)) e.model(s).init_weights(e.config().seed);
    });
}

int p2bw_engine_set_data(p2bw_engine* eng, const void* inputs, const void* targets, int first_mb,
                         int count) {
    return guarded([&] {
        auto& e = eng_of(eng);
        if (first_mb < 1) throw std::invalid_argument("microbatch ids are 1-based");
        // Inputs feed stage 0, targets the last stage (they may be the same stage);
        // a process without either stage ignores the call.
        if (e.is_local(0)) {
            e.before_data_set(0);
            e.model(0).set_data(inputs, e.depth() == 1 ? targets : nullptr, first_mb, count);
            e.after_data_set(0, first_mb, count);
        }
        if (e.depth() > 1 && e.is_local(e.depth() - 1)) {
            e.before_data_set(e.depth() - 1);
            e.model(e.depth() - 1).set_data(nullptr, targets, first_mb, count);
            e.after_data_set(e.depth() - 1, first_mb, count);
        }
    });
}

int p2bw_engine_make_toy_data(p2bw_engine* eng, int first_mb, int count) {
    return guarded([&] {
        auto& e = eng_of(eng);
        if (first_mb < 1) throw std::invalid_argument("microbatch ids are 1-based");
        const uint64_t seed = e.config().seed;
        // inputs on stage 0, targets on the last stage (one stage plays both at depth 1)
        std::vector<int> stages{0};
        if (e.depth() > 1) stages.push_back(e.depth() - 1);
        for (int s : stages) {
            if (!e.is_local(s)) continue;
            e.before_data_set(s);
            e.model(s).make_toy_data(seed, first_mb, count);
            e.after_data_set(s, first_mb, count);
        }
    });
}

int p2bw_engine_run(p2bw_engine* eng, const p2bw_op* const* programs, const size_t* n_ops,
                    int snapshot_updates) {
    return guarded([&] {
        auto& e = eng_of(eng);
        if (programs == nullptr || n_ops == nullptr) throw std::invalid_argument("NULL programs");
        std::vector<p2bw::Program> progs(static_cast<size_t>(e.depth()));
        for (int s = 0; s < e.depth(); ++s) {
            for (size_t i = 0; i < n_ops[s]; ++i) {
                const p2bw_op& op = programs[s][i];
                progs[s].push_back({op.kind, op.microbatch, op.weight_version});
            }
        }
        e.set_snapshot_every_update(snapshot_updates != 0);
        e.run(progs);
    });
}

int p2bw_engine_run_schedule_graph(p2bw_engine* eng, int num_batches, int launches, double* ms_per_launch) {
    return guarded([&] {
        auto& e = eng_of(eng);
        const auto& c = e.config();
        const auto programs = pipesim::generate_schedule(
            static_cast<pipesim::PipelinePolicy>(c.policy), c.depth, c.microbatches, num_batches);
        std::vector<p2bw::Program> progs;
        for (const auto& p : programs) {
            p2bw::Program prog;
            for (const auto& op : p.ops)
                prog.push_back({static_cast<int>(op.kind), op.microbatch, op.weight_version});
            progs.push_back(std::move(prog));
        }
        e.set_snapshot_every_update(false);
        const double ms = e.run_graph(progs, launches);
        if (ms_per_launch) *ms_per_launch = ms;
    });
}

int p2bw_engine_run_schedule(p2bw_engine* eng, int num_batches, int snapshot_updates) {
    return guarded([&] {
        auto& e = eng_of(eng);
        const auto& c = e.config();
        const auto programs = pipesim::generate_schedule(
            static_cast<pipesim::PipelinePolicy>(c.policy), c.depth, c.microbatches, num_batches);
        std::vector<p2bw::Program> progs;
        for (const auto& p : programs) {
            p2bw::Program prog;
            for (const auto& op : p.ops)
                prog.push_back({static_cast<int>(op.kind), op.microbatch, op.weight_version});
            progs.push_back(std::move(prog));
        }
        e.set_snapshot_every_update(snapshot_updates != 0);
        e.run(progs);
    });
}

int p2bw_engine_begin(p2bw_engine* eng, int num_batches) {
    return guarded([&] {
        auto& e = eng_of(eng);
        const auto& c = e.config();
        const auto programs = pipesim::generate_schedule(
            static_cast<pipesim::PipelinePolicy>(c.policy), c.depth, c.microbatches, num_batches);
        std::vector<p2bw::Program> progs;
        for (const auto& p : programs) {
            p2bw::Program prog;
            for (const auto& op : p.ops)
                prog.push_back({static_cast<int>(op.kind), op.microbatch, op.weight_version});
            progs.push_back(std::move(prog));
        }
        e.set_snapshot_every_update(false);
        e.begin(progs);
    });
}

int p2bw_engine_issue(p2bw_engine* eng, int upto_batch) {
    return guarded([&] { eng_of(eng).issue(upto_batch); });
}

int p2bw_engine_finish(p2bw_engine* eng) {
    return guarded([&] { eng_of(eng).finish(); });
}

int p2bw_engine_update_elapsed_ms(p2bw_engine* eng, int stage, int u0, int u1, double* ms) {
    return guarded([&] {
        auto& e = eng_of(eng);
        check_stage(e, stage);
        if (ms == nullptr) throw std::invalid_argument("ms is NULL");
        *ms = e.update_elapsed_ms(stage, u0, u1);
    });
}

int p2bw_nccl_unique_id(void* out, size_t bytes) {
    return guarded([&] {
        if (out == nullptr || bytes != sizeof(ncclUniqueId))
            throw std::invalid_argument("unique id buffer must be " + std::to_string(sizeof(ncclUniqueId)) + " bytes");
        const ncclUniqueId id = p2bw::nccl_unique_id();
        std::memcpy(out, &id, sizeof(id));
    });
}

int p2bw_engine_join_replicas(p2bw_engine* eng, const void* ids, int nranks, int rank) {
    return guarded([&] {
        if (ids == nullptr) throw std::invalid_argument("ids is NULL");
        eng_of(eng).join_replicas(ids, nranks, rank);
    });
}

int p2bw_engine_is_local(p2bw_engine* eng, int stage, int* out) {
    return guarded([&] {
        auto& e = eng_of(eng);
        check_stage(e, stage);
        if (out == nullptr) throw std::invalid_argument("out is NULL");
        *out = e.is_local(stage) ? 1 : 0;
    });
}

int p2bw_engine_export_stage(p2bw_engine* eng, int stage, void* blob, size_t bytes) {
    static_assert(sizeof(p2bw::StageBlob) <= P2BW_STAGE_BLOB_BYTES, "stage blob does not fit");
    return guarded([&] {
        auto& e = eng_of(eng);
        check_stage(e, stage);
        if (blob == nullptr || bytes != P2BW_STAGE_BLOB_BYTES)
            throw std::invalid_argument("stage blob buffer must be P2BW_STAGE_BLOB_BYTES bytes");
        const p2bw::StageBlob b = e.export_stage(stage);
        std::memset(blob, 0, bytes);
        std::memcpy(blob, &b, sizeof(b));
    });
}

int p2bw_engine_connect_stage(p2bw_engine* eng, const void* blob, size_t bytes) {
    return guarded([&] {
        auto& e = eng_of(eng);
        if (blob == nullptr || bytes != P2BW_STAGE_BLOB_BYTES)
            throw std::invalid_argument("stage blob buffer must be P2BW_STAGE_BLOB_BYTES bytes");
        p2bw::StageBlob b;
        std::memcpy(&b, blob, sizeof(b));
        e.connect_stage(b);
    });
}

int p2bw_engine_export_replica(p2bw_engine* eng, int stage, void* blob, size_t bytes) {
    static_assert(sizeof(p2bw::ReplicaBlob) <= P2BW_REPLICA_BLOB_BYTES, "replica blob does not fit");
    return guarded([&] {
        auto& e = eng_of(eng);
        check_stage(e, stage);
        if (blob == nullptr || bytes != P2BW_REPLICA_BLOB_BYTES)
            throw std::invalid_argument("replica blob buffer must be P2BW_REPLICA_BLOB_BYTES bytes");
        const p2bw::ReplicaBlob b = e.export_replica(stage);
        std::memset(blob, 0, bytes);
        std::memcpy(blob, &b, sizeof(b));
    });
}

int p2bw_engine_join_replicas_ipc(p2bw_engine* eng, int stage, const void* blobs, int nranks, int rank) {
    return guarded([&] {
        auto& e = eng_of(eng);
        check_stage(e, stage);
        if (blobs == nullptr) throw std::invalid_argument("blobs is NULL");
        if (nranks < 1 || nranks > p2bw::kMaxReplicas) throw std::invalid_argument("nranks must be in [1, 8]");
        std::vector<p2bw::ReplicaBlob> v(static_cast<size_t>(nranks));
        for (int q = 0; q < nranks; ++q)
            std::memcpy(&v[static_cast<size_t>(q)], static_cast<const uint8_t*>(blobs) + q * P2BW_REPLICA_BLOB_BYTES,
                        sizeof(p2bw::ReplicaBlob));
        e.join_replicas_ipc(stage, v, rank);
    });
}

int p2bw_engine_sync(p2bw_engine* eng) {
    return guarded([&] { eng_of(eng).sync(); });
}

int p2bw_engine_set_trace(p2bw_engine* eng, int on) {
    return guarded([&] { eng_of(eng).set_trace(on != 0); });
}

int p2bw_engine_trace_report(p2bw_engine* eng, char** out_json) {
    return guarded([&] {
        if (out_json == nullptr) throw std::invalid_argument("NULL argument");
        *out_json = p2bw::dup_string(eng_of(eng).trace_report());
    });
}

int p2bw_engine_counters(p2bw_engine* eng, p2bw_counters* out) {
    return guarded([&] {
        auto& e = eng_of(eng);
        if (out == nullptr) throw std::invalid_argument("out is NULL");
        out->version_consistent = e.stats().version_consistent ? 1 : 0;
        out->max_versions_held = e.stats().max_versions_held;
        out->ops_executed = e.stats().ops_executed;
        out->last_run_ms = e.elapsed_ms_last_run();
    });
}

int p2bw_engine_read_snapshot(p2bw_engine* eng, int stage, int update_index, void* host,
                              size_t bytes) {
    return guarded([&] {
        auto& e = eng_of(eng);
        check_stage(e, stage);
        e.sync();
        const auto& snaps = e.snapshots(stage);
        if (update_index < 1 || update_index > static_cast<int>(snaps.size()))
            throw p2bw::Error("no snapshot for update " + std::to_string(update_index));
        const auto& buf = snaps[static_cast<size_t>(update_index - 1)];
        if (bytes != buf.size()) throw std::invalid_argument("snapshot size mismatch");
        std::memcpy(host, buf.data(), bytes);
    });
}

int p2bw_engine_read_version(p2bw_engine* eng, int stage, int version, void* host, size_t bytes) {
    return guarded([&] {
        auto& e = eng_of(eng);
        check_stage(e, stage);
        e.sync();
        e.read_version(stage, version, host, bytes);
    });
}

int p2bw_engine_read_master(p2bw_engine* eng, int stage, void* host, size_t bytes) {
    return guarded([&] {
        auto& e = eng_of(eng);
        check_stage(e, stage);
        if (host == nullptr) throw std::invalid_argument("host buffer is NULL");
        e.sync();
        e.model(stage).read_master(host, bytes);
    });
}

int p2bw_engine_losses_async(p2bw_engine* eng, int first_mb, int count, float* host) {
    return guarded([&] {
        auto& e = eng_of(eng);
        if (host == nullptr || count < 1) throw std::invalid_argument("bad loss buffer");
        e.copy_losses_async(host, first_mb, count);
    });
}

int p2bw_engine_losses(p2bw_engine* eng, int first_mb, int count, double* out) {
    return guarded([&] {
        auto& e = eng_of(eng);
        if (out == nullptr || count < 0) throw std::invalid_argument("bad loss buffer");
        e.sync();
        const auto l = e.losses(first_mb, count);
        std::copy(l.begin(), l.end(), out);
    });
}

}  // extern "C"
