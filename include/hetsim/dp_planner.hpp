// hetsim::dp — data-parallel extension of the Eq.(6) planner (not in the reference: its
// SPEC.md:14 and :278 leave multi-GPU / ZeRO out of scope).
//
// With N data-parallel ranks each owning a 1/N shard of every block's fp32 master + moments
// (on the GPU or in pinned host DRAM per the plan) and gathering the full bf16 weights before
// use, the per-rank memory equations become
//   Eq.(1)_N = 2 m_a_in c + 2 m_a (L - c + 1) + 2 full (L - p + 1) + 12 shard (L - o) + m_gc
//   Eq.(2)_N = 14 shard o + m_cc
// with shard = round_up(ceil(m_p / N), 8) and full = N * shard (the padded gather buffer), and
// only the shard crosses the host link and is updated per rank: t_h2d = 2 shard / h2d_bw,
// t_d2h = 2 shard / d2h_bw, t_opt_{cpu,gpu} = shard / rate. The bf16 all-gather (before F / R / B)
// and reduce-scatter (after B) run on a side stream; with a collective bandwidth they bound the
// block times from below: t_fp >= t_ag, t_bp >= t_ag + t_rs, t_ag = t_rs = 2 full (N-1)/N / bw.
// Search space, scan order and the lexicographic (objective, o, p, c) tie break are the
// reference solve()'s (planner.cpp:37-108); at N = 1 every function here returns exactly what
// the reference counterpart returns.
#pragma once

#include <cstdint>

#include "hetsim/costmodel.hpp"
#include "hetsim/planner.hpp"
#include "hetsim/workload.hpp"

namespace hetsim {
namespace dp {

struct DpSpec {
    int dp_size = 1;
    double collective_bandwidth = 0.0;  // bytes/s of one rank's all-gather / reduce-scatter; <= 0: free
};

std::int64_t shard_params(std::int64_t m_p, int dp_size);  // per-rank optimizer elements of a block
std::int64_t gather_params(std::int64_t m_p, int dp_size);  // elements of the gathered bf16 buffer

// The per-rank block profile (durations of the shard's copies / optimizer steps, collective floor).
ModelProfile rank_profile(const ModelProfile& full, const HardwareSpec& hw, const DpSpec& dp);

std::int64_t peak_gpu_mem(const ModelProfile& full, const Strategy& s, const DpSpec& dp);
std::int64_t cpu_mem(const ModelProfile& full, const Strategy& s, const DpSpec& dp);
CostEstimate evaluate(const ModelProfile& full, const HardwareSpec& hw, const Strategy& s, const DpSpec& dp);

// Eq.(6) over the per-rank model. req.profile is the full (unsharded) profile.
PlanResult solve(const PlanRequest& req, const DpSpec& dp);

// GPU budget under which the reference simulator (whose memory model keeps 12 m_p per
// GPU-resident block) admits the same realised footprint as Eq.(1)_N for strategy s.
std::int64_t simulator_gpu_budget(const ModelProfile& full, const Strategy& s, std::int64_t gpu_budget,
                                  const DpSpec& dp);

}  // namespace dp
}  // namespace hetsim
