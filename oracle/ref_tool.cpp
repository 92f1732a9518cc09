// Command-line driver over the REFERENCE pipesim library (test infrastructure).
// Built by oracle/Makefile into oracle/_ref/ref_tool from /root/reference sources;
// used by tests/golden/make_golden.py (golden vectors) and by bench.py's
// reference / cpu_baseline arm (timing the reference's own pipelined_execute).
//   ref_tool schedule <policy> <d> <m> <T>
//   ref_tool version <k> <m>
//   ref_tool plan <model.json> <cluster.json> <max_batch> <policy> [text]
//   ref_tool toy <dim> <layers> <b> <seed> <lr> <beta> <m> <T> <policy> <depth> <out.bin>
//   ref_tool loop <dim> <layers> <b> <seed> <lr> <beta> <m> <T> <delayed> <out.bin>
//   ref_tool time <dim> <layers> <b> <m> <T> <depth> <seed>   (2BW pipelined_execute, seconds)
//   ref_tool simulate <model.json> <cluster.json> <policy> <w> <d> <b> <grad_accum> <recompute> <T>
//            (simulate_policy, simulator.cpp:140-339: throughput / steady batch time / bubble)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "pipesim/planner.hpp"
#include "pipesim/profile.hpp"
#include "pipesim/schedule.hpp"
#include "pipesim/semantics.hpp"
#include "pipesim/simulator.hpp"

using namespace pipesim;

namespace {

std::string slurp(const char* path) {
    std::ifstream in(path);
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

TrainerConfig trainer(double lr, double beta, int m, int T) {
    TrainerConfig c;
    c.learning_rate = lr;
    c.momentum = beta;
    c.microbatches_per_batch = m;
    c.num_batches = T;
    return c;
}

void write_traj(const Trajectory& traj, const char* path) {
    std::ofstream out(path, std::ios::binary);
    for (const auto& ws : traj)
        for (const auto& w : ws)
            out.write(reinterpret_cast<const char*>(w.data.data()),
                      static_cast<std::streamsize>(w.data.size() * sizeof(double)));
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_tool <command> ...\n");
        return 2;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "schedule" && argc == 6) {
            std::cout << serialize_programs(generate_schedule(
                static_cast<PipelinePolicy>(std::atoi(argv[2])), std::atoi(argv[3]),
                std::atoi(argv[4]), std::atoi(argv[5])));
        } else if (cmd == "version" && argc == 4) {
            std::cout << weight_version_2bw(std::atoi(argv[2]), std::atoi(argv[3])) << "\n";
        } else if (cmd == "plan" && argc >= 6) {
            const auto r = plan(load_model_profile(slurp(argv[2])), load_cluster_spec(slurp(argv[3])),
                                std::atoll(argv[4]), static_cast<PipelinePolicy>(std::atoi(argv[5])));
            std::cout << (argc > 6 ? plan_to_text(r) : plan_to_json(r));
        } else if (cmd == "toy" && argc == 13) {
            const auto model = ToyModel::make(std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]),
                                              std::atoi(argv[8]) * std::atoi(argv[9]),
                                              std::strtoull(argv[5], nullptr, 10));
            const auto r = pipelined_execute(
                model, trainer(std::atof(argv[6]), std::atof(argv[7]), std::atoi(argv[8]), std::atoi(argv[9])),
                static_cast<PipelinePolicy>(std::atoi(argv[10])), std::atoi(argv[11]));
            write_traj(r.trajectory, argv[12]);
            std::cout << "{\"version_consistent\": " << (r.version_consistent ? 1 : 0)
                      << ", \"max_versions_held\": " << r.max_versions_held << "}\n";
        } else if (cmd == "loop" && argc == 12) {
            const int m = std::atoi(argv[8]), T = std::atoi(argv[9]);
            const auto model = ToyModel::make(std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]),
                                              m * T, std::strtoull(argv[5], nullptr, 10));
            const auto cfg = trainer(std::atof(argv[6]), std::atof(argv[7]), m, T);
            write_traj(std::atoi(argv[10]) ? reference_2bw(model, cfg) : reference_vanilla(model, cfg),
                       argv[11]);
        } else if (cmd == "simulate" && argc == 11) {
            ParallelConfig cfg;
            cfg.width = std::atoi(argv[5]);
            cfg.depth = std::atoi(argv[6]);
            cfg.microbatch_size = std::atoi(argv[7]);
            cfg.grad_accum = std::atoi(argv[8]);
            cfg.recompute = std::atoi(argv[9]) != 0;
            const auto r = simulate_policy(static_cast<PipelinePolicy>(std::atoi(argv[4])),
                                           load_model_profile(slurp(argv[2])), load_cluster_spec(slurp(argv[3])),
                                           cfg, std::atoi(argv[10]));
            std::printf("{\"throughput\": %.17g, \"steady_batch_time\": %.17g, \"bubble_fraction\": %.17g}\n",
                        r.throughput, r.steady_batch_time, r.bubble_fraction);
        } else if (cmd == "time" && argc == 9) {
            const int dim = std::atoi(argv[2]), layers = std::atoi(argv[3]), b = std::atoi(argv[4]);
            const int m = std::atoi(argv[5]), T = std::atoi(argv[6]), depth = std::atoi(argv[7]);
            const auto model = ToyModel::make(dim, layers, b, m * T, std::strtoull(argv[8], nullptr, 10));
            const auto t0 = std::chrono::steady_clock::now();
            const auto r = pipelined_execute(model, trainer(0.01, 0.9, m, T), PipelinePolicy::TwoBW, depth);
            const double sec =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            std::cout << "{\"seconds\": " << sec << ", \"batches\": " << T
                      << ", \"max_versions_held\": " << r.max_versions_held << "}\n";
        } else {
            std::fprintf(stderr, "bad command line\n");
            return 2;
        }
    } catch (const std::exception& e) {
        std::cout << "ERROR: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
