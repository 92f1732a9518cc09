// validate_plan for the drop-in harness: the reference planner's validation
// step needs the reference's discrete-event simulator, which the B200 engine
// does not rebuild (out of scope).  Linked only into
// oracle/_ref/dropin_* next to the reference simulator objects.
#include <algorithm>
#include <cmath>

#include "pipesim/planner.hpp"
#include "pipesim/simulator.hpp"

namespace pipesim {

ValidationReport validate_plan(const PlanResult& plan, const ModelProfile& model,
                               const ClusterSpec& cluster, int num_batches, PipelinePolicy policy) {
    if (plan.ranked.empty()) throw Error("validate_plan requires a feasible plan");
    const SimReport sim = simulate_policy(policy, model, cluster, plan.best, num_batches);
    const std::vector<double> peaks = measure_high_water(sim);
    ValidationReport r;
    r.predicted_throughput = plan.predicted_throughput;
    r.predicted_memory = plan.predicted_memory;
    r.simulated_throughput = sim.throughput;
    r.simulated_memory = *std::max_element(peaks.begin(), peaks.end());
    r.throughput_rel_error = std::abs(r.predicted_throughput - r.simulated_throughput) / r.simulated_throughput;
    r.memory_rel_error = r.simulated_memory == 0.0
                             ? 0.0
                             : std::abs(r.predicted_memory - r.simulated_memory) / r.simulated_memory;
    return r;
}

}  // namespace pipesim
