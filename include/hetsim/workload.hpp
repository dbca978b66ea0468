// hetsim::core drop-in — model / hardware description and the per-block profile.
//
// Public surface mirrors /root/reference/proj/core/include/hetsim/workload.hpp:13-118
// (same type names, field names, field order and function signatures) so code written
// against the reference links unchanged. Implementation: csrc/hetsim/workload.cpp.
#pragma once

#include <cstdint>
#include <optional>

namespace hetsim {

// Transformer being trained. Every block has the same shape; the embedding is
// accounted for in ModelProfile::m_gc, not per block.
struct ModelSpec {
    int num_blocks = 1;            // L
    std::int64_t hidden_size = 1;  // h
    std::int64_t seq_len = 1;      // s
    std::int64_t batch_size = 1;   // b
    std::int64_t vocab_size = 1;   // V
    double activation_coef = 16.0; // activation elements per token per block / h
    double bwd_fwd_ratio = 2.0;    // backward FLOPs / forward FLOPs

    void validate() const;  // std::invalid_argument on a bad field
};

// Platform capacities and rates. On B200 the runtime fills the rates from measurement
// (see paper_2503_01890_b200/runtime profiler); the planner only sees these numbers.
struct HardwareSpec {
    std::int64_t gpu_mem = 0;       // bytes
    std::int64_t cpu_mem = 0;       // bytes
    double gpu_compute_rate = 0.0;  // FLOP/s
    double h2d_bandwidth = 0.0;     // B/s
    double d2h_bandwidth = 0.0;     // B/s
    double cpu_optim_rate = 0.0;    // params/s (CPU Adam)
    double gpu_optim_rate = 0.0;    // params/s (GPU Adam)

    void validate() const;
};

// One block: element counts (m_a, m_a_in), parameter count (m_p) and the six stream
// durations in seconds.
struct BlockProfile {
    std::int64_t m_a = 0;
    std::int64_t m_a_in = 0;
    std::int64_t m_p = 0;
    double t_fp = 0.0;
    double t_bp = 0.0;
    double t_h2d = 0.0;
    double t_d2h = 0.0;
    double t_opt_cpu = 0.0;
    double t_opt_gpu = 0.0;
};

struct ModelProfile {
    BlockProfile block;
    int num_blocks = 0;
    std::int64_t m_gc = 0;          // bytes pinned on the GPU outside the blocks
    std::int64_t m_cc = 0;          // bytes pinned on the CPU outside the blocks
    std::int64_t total_params = 0;
    double flops_per_iter = 0.0;
};

// 12h^2 + 13h: GPT-2 block (QKV 3h^2+3h, out-proj h^2+h, fc 4h^2+4h, fc2 4h^2+h, 2 LN 4h).
std::int64_t block_param_count(std::int64_t hidden_size);

struct ActivationSizes {
    std::int64_t m_a;
    std::int64_t m_a_in;
};

ActivationSizes activation_sizes(const ModelSpec& spec);

struct BlockTimes {
    double t_fp, t_bp, t_h2d, t_d2h, t_opt_cpu, t_opt_gpu;
};

BlockTimes estimate_block_times(const ModelSpec& spec, const HardwareSpec& hw);

struct ProfileOverrides {
    std::optional<std::int64_t> m_gc;
    std::optional<std::int64_t> m_cc;
};

ModelProfile build_profile(const ModelSpec& spec, const HardwareSpec& hw,
                           const ProfileOverrides& overrides = {});

}  // namespace hetsim
