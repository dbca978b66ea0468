// Eq.(6) exhaustive planner + greedy prefetch tuning + comparison presets.
// Decision semantics follow /root/reference/proj/core/src/planner.cpp:37-183:
//   * scan o ascending, stop at the first o whose CPU footprint exceeds the budget;
//   * p in [0,o], c in [0,L]; GPU filter by Eq.(1);
//   * keep the lexicographic minimum of (objective, o, p, c).
// Because every candidate is compared under a strict total order, the winner does not
// depend on scan order; we still scan in the reference order so feasible_count matches.
#include "hetsim/planner.hpp"

#include <algorithm>
#include <chrono>

#include "hetsim/simulator.hpp"

namespace hetsim {

namespace {

std::string infeasible_text(std::int64_t gpu, std::int64_t cpu, std::int64_t cap) {
    return "no (c_hat, p_hat, o_hat) satisfies the memory constraints; GPU shortfall "
           "at full offload (L,L,L): " + std::to_string(gpu) +
           " B; CPU shortfall for the constant residue alone: " + std::to_string(cpu) +
           " B; GPU shortfall at the largest CPU-feasible offload: " +
           std::to_string(cap) + " B";
}

// Strict "a beats incumbent b" under (objective, o_hat, p_hat, c_hat).
bool beats(double obj_a, int o_a, int p_a, int c_a, const CostEstimate& cb,
           const Strategy& sb) {
    if (obj_a != cb.objective) return obj_a < cb.objective;
    if (o_a != sb.o_hat) return o_a < sb.o_hat;
    if (p_a != sb.p_hat) return p_a < sb.p_hat;
    return c_a < sb.c_hat;
}

}  // namespace

InfeasibleError::InfeasibleError(std::int64_t gpu, std::int64_t cpu, std::int64_t cap)
    : std::runtime_error(infeasible_text(gpu, cpu, cap)), gpu_(gpu), cpu_(cpu), gpu_cap_(cap) {}

PlanResult solve(const PlanRequest& req) {
    using clock = std::chrono::steady_clock;
    const clock::time_point begin = clock::now();
    req.hardware.validate();
    const ModelProfile& pr = req.profile;
    const int L = pr.num_blocks;

    PlanResult out;
    bool have = false;
    std::int64_t n_feasible = 0;

    for (int o = 0; o <= L; ++o) {
        if (cpu_mem(pr, Strategy::uniform(0, 0, o, L)) > req.hardware.cpu_mem) break;
        for (int p = 0; p <= o; ++p) {
            for (int c = 0; c <= L; ++c) {
                Strategy cand = Strategy::uniform(c, p, o, L);
                if (peak_gpu_mem(pr, cand) > req.hardware.gpu_mem) continue;
                ++n_feasible;
                const CostEstimate est = evaluate(pr, cand);
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
            0, peak_gpu_mem(pr, Strategy::uniform(L, L, L, L)) - req.hardware.gpu_mem);
        const std::int64_t cpu_short = std::max<std::int64_t>(0, pr.m_cc - req.hardware.cpu_mem);
        std::int64_t at_cap = gpu_short;
        for (int o = L; o >= 0; --o) {
            if (cpu_mem(pr, Strategy::uniform(0, 0, o, L)) <= req.hardware.cpu_mem) {
                at_cap = std::max<std::int64_t>(
                    0, peak_gpu_mem(pr, Strategy::uniform(L, o, o, L)) - req.hardware.gpu_mem);
                break;
            }
        }
        throw InfeasibleError(gpu_short, cpu_short, at_cap);
    }

    out.feasible_count = n_feasible;
    out.solve_time = std::chrono::duration<double>(clock::now() - begin).count();
    return out;
}

// Greedy lookahead advancement (reference planner.cpp:110-153): walk P-blocks from the
// last to the first; bump one block's lookahead while both a FIFO and a PS dry run
// (2 iterations) stay in budget, neither gets slower and at least one gets faster.
Strategy fine_tune_prefetch(const ModelProfile& pr, const Strategy& s, const HardwareSpec& hw) {
    s.validate(pr.num_blocks);
    const int L = pr.num_blocks;

    struct Probe {
        bool ok;
        double steady;
    };
    const auto probe = [&](const Strategy& cand, bool ps) -> Probe {
        try {
            const SimResult r = run(pr, cand, hw, 2, ps);
            return {r.peak_gpu <= hw.gpu_mem, r.steady_state_time};
        } catch (const MemoryExceededError&) {
            return {false, 0.0};
        }
    };

    Strategy best = s;
    Probe fifo0 = probe(best, false);
    if (!fifo0.ok) return best;
    Probe ps0 = probe(best, true);
    if (!ps0.ok) return best;

    for (int blk = std::min(best.p_hat, L); blk >= 1; --blk) {
        int& la = best.prefetch_lookahead[static_cast<std::size_t>(blk - 1)];
        const int ceiling = std::max(1, L - blk + 1);
        while (la < ceiling) {
            Strategy cand = best;
            cand.prefetch_lookahead[static_cast<std::size_t>(blk - 1)] += 1;
            const Probe f = probe(cand, false);
            if (!f.ok) break;
            const Probe p = probe(cand, true);
            if (!p.ok) break;
            if (f.steady > fifo0.steady || p.steady > ps0.steady) break;
            if (f.steady == fifo0.steady && p.steady == ps0.steady) break;
            la += 1;
            fifo0.steady = f.steady;
            ps0.steady = p.steady;
        }
    }
    return best;
}

std::vector<std::pair<std::string, Strategy>> baseline_presets(const ModelProfile& pr,
                                                               const HardwareSpec& hw) {
    const int L = pr.num_blocks;
    const auto fits = [&](const Strategy& s) {
        return peak_gpu_mem(pr, s) <= hw.gpu_mem && cpu_mem(pr, s) <= hw.cpu_mem;
    };
    // ZeRO-Offload shape: params on GPU, every optimizer on the CPU; checkpoint all
    // blocks only if that is needed to fit, or if it is strictly faster.
    const Strategy plain = Strategy::uniform(0, 0, L, L);
    const Strategy ckpt = Strategy::uniform(L, 0, L, L);
    const bool plain_ok = fits(plain);
    const bool ckpt_ok = fits(ckpt);
    Strategy zero = plain;
    if (!plain_ok)
        zero = ckpt;
    else if (ckpt_ok && evaluate(pr, ckpt).objective < evaluate(pr, plain).objective)
        zero = ckpt;

    std::vector<std::pair<std::string, Strategy>> out;
    out.emplace_back("zero-offload", zero);
    out.emplace_back("full-offload", Strategy::uniform(L, L, L, L));
    out.emplace_back("all-gpu", Strategy::uniform(0, 0, 0, L));
    return out;
}

}  // namespace hetsim
