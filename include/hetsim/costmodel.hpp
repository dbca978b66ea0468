// hetsim::core drop-in — strategy triple and the paper's Eq.(1)-(5) cost model.
// Mirrors /root/reference/proj/core/include/hetsim/costmodel.hpp:22-84.
#pragma once

#include <cstdint>
#include <vector>

#include "hetsim/workload.hpp"

namespace hetsim {

// (c_hat, p_hat, o_hat): C = {1..c_hat} recompute, P = {1..p_hat} bf16-param offload,
// O = {L-o_hat+1..L} optimizer offload, with p_hat <= o_hat. prefetch_lookahead[i-1]
// is how many backward units ahead block i's backward prefetch is issued.
struct Strategy {
    int c_hat = 0;
    int p_hat = 0;
    int o_hat = 0;
    std::vector<int> prefetch_lookahead;

    static Strategy uniform(int c_hat, int p_hat, int o_hat, int num_blocks);
    void validate(int num_blocks) const;  // std::invalid_argument
};

struct CostEstimate {
    double t_fwd = 0.0;
    double t_bwd = 0.0;
    double t_sync = 0.0;
    int v_hat = 0;
    std::int64_t peak_gpu = 0;
    std::int64_t cpu_bytes = 0;
    double objective = 0.0;
};

std::int64_t peak_gpu_mem(const ModelProfile& profile, const Strategy& s);  // Eq.(1)
std::int64_t cpu_mem(const ModelProfile& profile, const Strategy& s);       // Eq.(2)
double t_fwd(const ModelProfile& profile, const Strategy& s);               // Eq.(3)
int v_hat(const Strategy& s);
double t_sync(const ModelProfile& profile, const Strategy& s);              // Eq.(4)
double t_bwd(const ModelProfile& profile, const Strategy& s);               // Eq.(5)
CostEstimate evaluate(const ModelProfile& profile, const Strategy& s);

}  // namespace hetsim
