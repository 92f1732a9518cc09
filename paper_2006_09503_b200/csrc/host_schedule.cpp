// Stage-program generator: the op streams the B200 executor interprets.
// Behaviour (op order, versions, error text) follows reference
// core/src/schedule.cpp; each function cites the lines it restates.
#include <algorithm>
#include <array>
#include <sstream>
#include <utility>

#include "pipesim/schedule.hpp"

namespace pipesim {
namespace {

constexpr std::array<std::pair<PipelinePolicy, const char*>, 5> kPolicyNames{{
    {PipelinePolicy::NoPipelining, "none"},
    {PipelinePolicy::GPipe, "gpipe"},
    {PipelinePolicy::PipeDream1F1B, "1f1b"},
    {PipelinePolicy::PipeDreamFlush, "flush"},
    {PipelinePolicy::TwoBW, "2bw"},
}};

constexpr std::array<std::pair<OpKind, const char*>, 10> kOpNames{{
    {OpKind::Forward, "forward"},
    {OpKind::Backward, "backward"},
    {OpKind::Recompute, "recompute"},
    {OpKind::WeightUpdate, "update"},
    {OpKind::FlushBarrier, "flush"},
    {OpKind::ActivationSend, "act_send"},
    {OpKind::ActivationRecv, "act_recv"},
    {OpKind::GradSend, "grad_send"},
    {OpKind::GradRecv, "grad_recv"},
    {OpKind::AllReduce, "allreduce"},
}};

bool carries_microbatch(OpKind k) {
    return k == OpKind::Forward || k == OpKind::Backward || k == OpKind::Recompute;
}

// Program builder: appends ops to one stage's list.
struct Emitter {
    std::vector<ScheduledOp>& ops;
    void fwd(int k, int v) { ops.push_back({OpKind::Forward, k, v}); }
    void bwd(int k, int v) { ops.push_back({OpKind::Backward, k, v}); }
    // End of a batch: [flush barrier,] all-reduce, update (schedule.cpp:80-84).
    void update(bool with_flush) {
        if (with_flush) ops.push_back({OpKind::FlushBarrier, 0, 0});
        ops.push_back({OpKind::AllReduce, 0, 0});
        ops.push_back({OpKind::WeightUpdate, 0, 0});
    }
};

// GPipe (all F then all B, flush) and no-pipelining (F/B alternating), one
// weight version per batch (schedule.cpp:88-105).
void emit_batched(Emitter& e, bool gpipe, int m, int batches) {
    for (int t = 0; t < batches; ++t) {
        const int first = t * m + 1;
        if (gpipe) {
            for (int k = first; k < first + m; ++k) e.fwd(k, t);
            for (int k = first; k < first + m; ++k) e.bwd(k, t);
        } else {
            for (int k = first; k < first + m; ++k) {
                e.fwd(k, t);
                e.bwd(k, t);
            }
        }
        e.update(gpipe);
    }
}

// PipeDream-Flush: per batch, 1F1B with a warm-up of min(d - s, m) forwards,
// then a flush (schedule.cpp:109-123).
void emit_flush(Emitter& e, int stage, int d, int m, int batches) {
    const int warm = std::min(d - stage, m);
    for (int t = 0; t < batches; ++t) {
        const int base = t * m;
        for (int j = 1; j <= warm; ++j) e.fwd(base + j, t);
        for (int j = 1; j <= m; ++j) {
            e.bwd(base + j, t);
            if (j + warm <= m) e.fwd(base + j + warm, t);
        }
        e.update(true);
    }
}

// Continuous 1F1B across batch boundaries: 2BW (update every m backwards) and
// PipeDream weight stashing (update after every backward) (schedule.cpp:126-144).
void emit_continuous(Emitter& e, bool two_bw, int stage, int d, int m, int batches) {
    const int total = m * batches;
    const int warm = std::min(d - stage, total);
    auto ver = [&](int k) { return two_bw ? weight_version_2bw(k, m) : kLatestVersion; };
    for (int k = 1; k <= warm; ++k) e.fwd(k, ver(k));
    for (int k = 1; k <= total; ++k) {
        e.bwd(k, ver(k));
        if (!two_bw || k % m == 0) e.update(false);
        const int next = k + warm;
        if (next <= total) e.fwd(next, ver(next));
    }
}

}  // namespace

std::string to_string(PipelinePolicy policy) {
    for (const auto& [p, name] : kPolicyNames)
        if (p == policy) return name;
    throw Error("unknown policy");
}

PipelinePolicy parse_policy(const std::string& name) {
    for (const auto& [p, n] : kPolicyNames)
        if (name == n) return p;
    throw Error("unknown policy '" + name + "' (expected none|gpipe|1f1b|flush|2bw)");
}

std::string to_string(OpKind kind) {
    for (const auto& [k, name] : kOpNames)
        if (k == kind) return name;
    throw Error("unknown op kind");
}

// schedule.cpp:58-62
int weight_version_2bw(int k, int m) {
    if (k < 1) throw Error("microbatch index must be >= 1");
    if (m < 1) throw Error("microbatches per batch must be >= 1");
    const int batch_index = (k - 1) / m;  // 0-based batch of microbatch k
    return batch_index >= 1 ? batch_index - 1 : 0;
}

// schedule.cpp:64-78
int required_versions(PipelinePolicy policy, int d, int /*m*/) {
    switch (policy) {
        case PipelinePolicy::TwoBW: return 2;
        case PipelinePolicy::PipeDream1F1B: return d;
        case PipelinePolicy::NoPipelining:
        case PipelinePolicy::GPipe:
        case PipelinePolicy::PipeDreamFlush: return 1;
    }
    throw Error("unknown policy");
}

// schedule.cpp:148-175
std::vector<StageProgram> generate_schedule(PipelinePolicy policy, int d, int m,
                                            int num_batches) {
    if (d < 1) throw Error("depth must be >= 1");
    if (m < 1) throw Error("microbatches per batch must be >= 1");
    if (num_batches < 1) throw Error("num_batches must be >= 1");
    if (policy == PipelinePolicy::TwoBW && m < d)
        throw Error("2bw requires m >= d (m=" + std::to_string(m) + ", d=" + std::to_string(d) +
                    ")");
    std::vector<StageProgram> out(static_cast<size_t>(d));
    for (int s = 0; s < d; ++s) {
        out[s].stage = s;
        Emitter e{out[s].ops};
        switch (policy) {
            case PipelinePolicy::GPipe: emit_batched(e, true, m, num_batches); break;
            case PipelinePolicy::NoPipelining: emit_batched(e, false, m, num_batches); break;
            case PipelinePolicy::PipeDreamFlush: emit_flush(e, s, d, m, num_batches); break;
            case PipelinePolicy::TwoBW: emit_continuous(e, true, s, d, m, num_batches); break;
            case PipelinePolicy::PipeDream1F1B:
                emit_continuous(e, false, s, d, m, num_batches);
                break;
        }
    }
    return out;
}

// schedule.cpp:177-195
std::string serialize_programs(const std::vector<StageProgram>& programs) {
    std::string text;
    for (const StageProgram& p : programs) {
        for (const ScheduledOp& op : p.ops) {
            text += "stage=" + std::to_string(p.stage) + " op=" + to_string(op.kind);
            if (carries_microbatch(op.kind)) {
                text += " mb=" + std::to_string(op.microbatch) + " ver=" +
                        (op.weight_version == kLatestVersion ? std::string("latest")
                                                             : std::to_string(op.weight_version));
            }
            text += '\n';
        }
    }
    return text;
}

// schedule.cpp:197-242
std::vector<StageProgram> parse_programs(const std::string& text) {
    std::vector<StageProgram> programs;
    std::istringstream lines(text);
    std::string line;
    for (int lineno = 1; std::getline(lines, line); ++lineno) {
        if (line.empty()) continue;
        const std::string where = "program line " + std::to_string(lineno) + ": ";
        std::istringstream tokens(line);
        std::string tok;
        int stage = -1;
        bool got_kind = false;
        ScheduledOp op;
        while (tokens >> tok) {
            const size_t eq = tok.find('=');
            if (eq == std::string::npos) throw Error(where + "bad field '" + tok + "'");
            const std::string key = tok.substr(0, eq), val = tok.substr(eq + 1);
            if (key == "stage") {
                stage = std::stoi(val);
            } else if (key == "op") {
                bool found = false;
                for (const auto& [k, name] : kOpNames) {
                    if (val == name) {
                        op.kind = k;
                        found = true;
                    }
                }
                if (!found) throw Error("unknown op kind '" + val + "'");
                got_kind = true;
            } else if (key == "mb") {
                op.microbatch = std::stoi(val);
            } else if (key == "ver") {
                op.weight_version = val == "latest" ? kLatestVersion : std::stoi(val);
            } else {
                throw Error(where + "unknown key '" + key + "'");
            }
        }
        if (stage < 0 || !got_kind) throw Error(where + "missing stage or op");
        while (static_cast<int>(programs.size()) <= stage) {
            programs.push_back(StageProgram{static_cast<int>(programs.size()), {}});
        }
        programs[stage].ops.push_back(op);
    }
    return programs;
}

}  // namespace pipesim
