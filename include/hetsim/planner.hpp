// hetsim::core drop-in — Eq.(6) exhaustive planner, prefetch fine-tuning, presets.
// Mirrors /root/reference/proj/core/include/hetsim/planner.hpp:17-74.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hetsim/costmodel.hpp"
#include "hetsim/workload.hpp"

namespace hetsim {

enum class TieBreak {
    least_offload,  // equal objective: smaller o_hat, then p_hat, then c_hat
};

struct PlanRequest {
    ModelProfile profile;
    HardwareSpec hardware;
    TieBreak tie_break = TieBreak::least_offload;
};

struct PlanResult {
    Strategy strategy;
    CostEstimate cost;
    std::int64_t feasible_count = 0;
    double solve_time = 0.0;
};

class InfeasibleError : public std::runtime_error {
public:
    InfeasibleError(std::int64_t gpu_shortfall, std::int64_t cpu_shortfall,
                    std::int64_t gpu_shortfall_at_cpu_cap);
    std::int64_t gpu_shortfall_bytes() const { return gpu_; }
    std::int64_t cpu_shortfall_bytes() const { return cpu_; }
    std::int64_t gpu_shortfall_at_cpu_cap_bytes() const { return gpu_cap_; }

private:
    std::int64_t gpu_;
    std::int64_t cpu_;
    std::int64_t gpu_cap_;
};

PlanResult solve(const PlanRequest& req);

Strategy fine_tune_prefetch(const ModelProfile& profile, const Strategy& s,
                            const HardwareSpec& hw);

std::vector<std::pair<std::string, Strategy>> baseline_presets(
    const ModelProfile& profile, const HardwareSpec& hw);

}  // namespace hetsim
