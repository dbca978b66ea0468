// Data-parallel planner extension (include/hetsim/dp_planner.hpp). The scan and tie break are
// the reference solve()'s (proj/core/src/planner.cpp:37-108); only the per-rank memory and time
// terms change, and at dp_size == 1 they reduce to Eq.(1)-(5) bit for bit.
#include "hetsim/dp_planner.hpp"

#include <algorithm>
#include <chrono>

namespace hetsim {
namespace dp {

namespace {
int ranks(const DpSpec& dp) { return dp.dp_size < 1 ? 1 : dp.dp_size; }

bool beats(double obj_a, int o_a, int p_a, int c_a, const CostEstimate& cb, const Strategy& sb) {
    if (obj_a != cb.objective) return obj_a < cb.objective;
    if (o_a != sb.o_hat) return o_a < sb.o_hat;
    if (p_a != sb.p_hat) return p_a < sb.p_hat;
    return c_a < sb.c_hat;
}
}  // namespace

std::int64_t shard_params(std::int64_t m_p, int n) {
    if (n <= 1) return m_p;
    const std::int64_t per = (m_p + n - 1) / n;
    return (per + 7) / 8 * 8;
}

std::int64_t gather_params(std::int64_t m_p, int n) { return n <= 1 ? m_p : shard_params(m_p, n) * n; }

ModelProfile rank_profile(const ModelProfile& full, const HardwareSpec& hw, const DpSpec& dp) {
    const int n = ranks(dp);
    if (n == 1) return full;
    ModelProfile pr = full;
    BlockProfile& k = pr.block;
    const double shard = static_cast<double>(shard_params(k.m_p, n));
    k.t_h2d = 2.0 * shard / hw.h2d_bandwidth;
    k.t_d2h = 2.0 * shard / hw.d2h_bandwidth;
    k.t_opt_cpu = shard / hw.cpu_optim_rate;
    k.t_opt_gpu = shard / hw.gpu_optim_rate;
    if (dp.collective_bandwidth > 0.0) {
        const double bytes = 2.0 * static_cast<double>(gather_params(k.m_p, n)) * (n - 1) / n;
        const double t_coll = bytes / dp.collective_bandwidth;
        k.t_fp = std::max(k.t_fp, t_coll);
        k.t_bp = std::max(k.t_bp, 2.0 * t_coll);
    }
    return pr;
}

std::int64_t peak_gpu_mem(const ModelProfile& pr, const Strategy& s, const DpSpec& dp) {
    const int n = ranks(dp);
    if (n == 1) return hetsim::peak_gpu_mem(pr, s);
    const std::int64_t L = pr.num_blocks;
    const BlockProfile& k = pr.block;
    std::int64_t bytes = 2 * k.m_a_in * s.c_hat;
    bytes += 2 * k.m_a * (L - s.c_hat + 1);
    bytes += 2 * gather_params(k.m_p, n) * (L - s.p_hat + 1);
    bytes += 12 * shard_params(k.m_p, n) * (L - s.o_hat);
    return bytes + pr.m_gc;
}

std::int64_t cpu_mem(const ModelProfile& pr, const Strategy& s, const DpSpec& dp) {
    const int n = ranks(dp);
    if (n == 1) return hetsim::cpu_mem(pr, s);
    return 14 * shard_params(pr.block.m_p, n) * s.o_hat + pr.m_cc;
}

CostEstimate evaluate(const ModelProfile& full, const HardwareSpec& hw, const Strategy& s, const DpSpec& dp) {
    if (ranks(dp) == 1) return hetsim::evaluate(full, s);
    const ModelProfile pr = rank_profile(full, hw, dp);
    CostEstimate c = hetsim::evaluate(pr, s);
    c.peak_gpu = peak_gpu_mem(full, s, dp);
    c.cpu_bytes = cpu_mem(full, s, dp);
    return c;
}

PlanResult solve(const PlanRequest& req, const DpSpec& dp) {
    if (ranks(dp) == 1) return hetsim::solve(req);
    using clock = std::chrono::steady_clock;
    const clock::time_point begin = clock::now();
    req.hardware.validate();
    const ModelProfile& full = req.profile;
    const ModelProfile pr = rank_profile(full, req.hardware, dp);
    const int L = full.num_blocks;
    PlanResult out;
    bool have = false;
    std::int64_t n_feasible = 0;
    for (int o = 0; o <= L; ++o) {
        if (cpu_mem(full, Strategy::uniform(0, 0, o, L), dp) > req.hardware.cpu_mem) break;
        for (int p = 0; p <= o; ++p) {
            for (int c = 0; c <= L; ++c) {
                Strategy cand = Strategy::uniform(c, p, o, L);
                if (peak_gpu_mem(full, cand, dp) > req.hardware.gpu_mem) continue;
                ++n_feasible;
                CostEstimate est = hetsim::evaluate(pr, cand);
                est.peak_gpu = peak_gpu_mem(full, cand, dp);
                est.cpu_bytes = cpu_mem(full, cand, dp);
                if (!have || beats(est.objective, o, p, c, out.cost, out.strategy)) {
                    have = true;
                    out.strategy = std::move(cand);
                    out.cost = est;
                }
            }
        }
    }
    if (!have) {
        const std::int64_t gpu_short = std::max<std::int64_t>(
            0, peak_gpu_mem(full, Strategy::uniform(L, L, L, L), dp) - req.hardware.gpu_mem);
        const std::int64_t cpu_short = std::max<std::int64_t>(0, full.m_cc - req.hardware.cpu_mem);
        std::int64_t at_cap = gpu_short;
        for (int o = L; o >= 0; --o) {
            if (cpu_mem(full, Strategy::uniform(0, 0, o, L), dp) <= req.hardware.cpu_mem) {
                at_cap = std::max<std::int64_t>(
                    0, peak_gpu_mem(full, Strategy::uniform(L, o, o, L), dp) - req.hardware.gpu_mem);
                break;
            }
        }
        throw InfeasibleError(gpu_short, cpu_short, at_cap);
    }
    out.feasible_count = n_feasible;
    out.solve_time = std::chrono::duration<double>(clock::now() - begin).count();
    return out;
}

std::int64_t simulator_gpu_budget(const ModelProfile& full, const Strategy& s, std::int64_t gpu_budget,
                                  const DpSpec& dp) {
    const int n = ranks(dp);
    if (n == 1) return gpu_budget;
    // the simulator charges 12 m_p per GPU-resident block and 2 m_p per bf16 buffer; the realised
    // per-rank footprint is 12 shard and 2 full: credit the difference
    const std::int64_t L = full.num_blocks, m_p = full.block.m_p;
    const std::int64_t opt = 12 * (m_p - shard_params(m_p, n)) * (L - s.o_hat);
    const std::int64_t buf = 2 * (m_p - gather_params(m_p, n)) * (L - s.p_hat + 1);  // <= 0 (padding)
    return gpu_budget + opt + buf;
}

}  // namespace dp
}  // namespace hetsim
