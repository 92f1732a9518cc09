// C-ABI over the host-side pipesim API (schedule, planner, partition).
#include <cstdlib>
#include <cstring>

#include <nlohmann/json.hpp>

#include "capi_internal.h"
#include "p2bw.h"
#include "pipesim/planner.hpp"
#include "pipesim/profile.hpp"
#include "pipesim/schedule.hpp"

struct p2bw_schedule {
    std::vector<pipesim::StageProgram> programs;
    std::vector<std::vector<p2bw_op>> flat;
    void flatten() {
        flat.clear();
        for (const auto& p : programs) {
            std::vector<p2bw_op> ops;
            ops.reserve(p.ops.size());
            for (const auto& op : p.ops)
                ops.push_back({static_cast<int>(op.kind), op.microbatch, op.weight_version});
            flat.push_back(std::move(ops));
        }
    }
};

using p2bw::guarded;

namespace p2bw {

char* dup_string(const std::string& s) {
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    if (out == nullptr) throw std::bad_alloc();
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}

}  // namespace p2bw

using p2bw::dup_string;

namespace {

pipesim::PipelinePolicy as_policy(int p) {
    if (p < P2BW_POLICY_NONE || p > P2BW_POLICY_2BW)
        throw std::invalid_argument("unknown policy code " + std::to_string(p));
    return static_cast<pipesim::PipelinePolicy>(p);
}

void need(const void* p, const char* what) {
    if (p == nullptr) throw std::invalid_argument(std::string(what) + " is NULL");
}

}  // namespace

extern "C" {

void p2bw_free(void* p) { std::free(p); }

int p2bw_weight_version_2bw(int k, int m, int* out) {
    return guarded([&] {
        need(out, "out");
        *out = pipesim::weight_version_2bw(k, m);
    });
}

int p2bw_required_versions(int policy, int d, int m, int* out) {
    return guarded([&] {
        need(out, "out");
        *out = pipesim::required_versions(as_policy(policy), d, m);
    });
}

int p2bw_schedule_generate(int policy, int d, int m, int num_batches, p2bw_schedule** out) {
    return guarded([&] {
        need(out, "out");
        auto* s = new p2bw_schedule;
        try {
            s->programs = pipesim::generate_schedule(as_policy(policy), d, m, num_batches);
            s->flatten();
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

int p2bw_schedule_parse(const char* text, p2bw_schedule** out) {
    return guarded([&] {
        need(text, "text");
        need(out, "out");
        auto* s = new p2bw_schedule;
        try {
            s->programs = pipesim::parse_programs(text);
            s->flatten();
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

int p2bw_schedule_num_stages(const p2bw_schedule* sched, int* out) {
    return guarded([&] {
        need(sched, "schedule");
        need(out, "out");
        *out = static_cast<int>(sched->programs.size());
    });
}

int p2bw_schedule_ops(const p2bw_schedule* sched, int stage, const p2bw_op** ops, size_t* n) {
    return guarded([&] {
        need(sched, "schedule");
        need(ops, "ops");
        need(n, "n");
        if (stage < 0 || stage >= static_cast<int>(sched->flat.size()))
            throw std::invalid_argument("stage out of range");
        *ops = sched->flat[stage].data();
        *n = sched->flat[stage].size();
    });
}

int p2bw_schedule_serialize(const p2bw_schedule* sched, char** text) {
    return guarded([&] {
        need(sched, "schedule");
        need(text, "text");
        *text = dup_string(pipesim::serialize_programs(sched->programs));
    });
}

void p2bw_schedule_destroy(p2bw_schedule* sched) { delete sched; }

int p2bw_policy_name(int policy, const char** name) {
    return guarded([&] {
        need(name, "name");
        static const char* const names[] = {"none", "gpipe", "1f1b", "flush", "2bw"};
        as_policy(policy);
        *name = names[policy];
    });
}

int p2bw_policy_parse(const char* name, int* policy) {
    return guarded([&] {
        need(name, "name");
        need(policy, "policy");
        *policy = static_cast<int>(pipesim::parse_policy(name));
    });
}

int p2bw_plan(const char* model_json, const char* cluster_json, long long max_batch, int policy,
              int as_text, char** out) {
    return guarded([&] {
        need(model_json, "model_json");
        need(cluster_json, "cluster_json");
        need(out, "out");
        const auto model = pipesim::load_model_profile(model_json);
        const auto cluster = pipesim::load_cluster_spec(cluster_json);
        const auto result = pipesim::plan(model, cluster, max_batch, as_policy(policy));
        *out = dup_string(as_text ? pipesim::plan_to_text(result) : pipesim::plan_to_json(result));
    });
}

int p2bw_partition_balanced(const char* model_json, int d, int b, char** out_json) {
    return guarded([&] {
        need(model_json, "model_json");
        need(out_json, "out_json");
        const auto bounds = pipesim::partition_balanced(pipesim::load_model_profile(model_json), d, b);
        *out_json = dup_string(nlohmann::json(bounds).dump());
    });
}

int p2bw_partition_equal(const char* model_json, int d, char** out_json) {
    return guarded([&] {
        need(model_json, "model_json");
        need(out_json, "out_json");
        const auto stages = pipesim::partition_equal(pipesim::load_model_profile(model_json), d);
        auto table = [](const pipesim::BTable& t) {
            nlohmann::json j = nlohmann::json::object();
            for (const auto& [b, v] : t) j[std::to_string(b)] = v;
            return j;
        };
        nlohmann::json arr = nlohmann::json::array();
        for (const auto& s : stages) {
            arr.push_back({{"fwd_time", table(s.fwd_time)},
                           {"bwd_time", table(s.bwd_time)},
                           {"weight_bytes", s.weight_bytes},
                           {"act_total_bytes", table(s.act_total_bytes)},
                           {"act_input_bytes", table(s.act_input_bytes)},
                           {"act_output_bytes", table(s.act_output_bytes)}});
        }
        *out_json = dup_string(arr.dump(2));
    });
}

}  // extern "C"
