// extern "C" wrappers of the hetsim::core drop-in (include/hetsim_c.h).
#include "hetsim_c.h"

#include <cstring>
#include <sstream>
#include <string>

#include "hetsim/config.hpp"
#include "hetsim/plan_io.hpp"
#include "hetsim/planner.hpp"
#include "hetsim/dp_planner.hpp"
#include "hetsim/simulator.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int64_t guard(F&& f) {
    try {
        return f();
    } catch (const hetsim::ConfigError& e) {
        g_err = e.what();
        return HETSIM_ERR_CONFIG;
    } catch (const hetsim::InfeasibleError& e) {
        g_err = e.what();
        return HETSIM_ERR_INFEASIBLE;
    } catch (const hetsim::MemoryExceededError& e) {
        g_err = e.what();
        return HETSIM_ERR_MEMORY;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return HETSIM_ERR_INVALID;
    } catch (const std::exception& e) {
        g_err = e.what();
        return HETSIM_ERR_OTHER;
    }
}

int64_t emit(const std::string& s, char* out, size_t cap) {
    if (out && cap) {
        const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    }
    return static_cast<int64_t>(s.size()) + 1;
}
}  // namespace

extern "C" {

const char* ah_hetsim_last_error(void) { return g_err.c_str(); }

int64_t ah_hetsim_block_param_count(int64_t h) {
    return guard([&]() -> int64_t { return hetsim::block_param_count(h); });
}

int64_t ah_hetsim_plan_json(const char* text, char* out, size_t cap) {
    return guard([&]() -> int64_t {
        const hetsim::RunConfig cfg = hetsim::parse_config(text ? text : "", "<memory>");
        const hetsim::ModelProfile prof = hetsim::build_profile(cfg.model, cfg.hardware, cfg.overrides);
        hetsim::PlanRequest req;
        req.profile = prof;
        req.hardware = cfg.hardware;
        const hetsim::PlanResult r = hetsim::solve(req);
        hetsim::PlanDocument doc;
        doc.strategy = hetsim::fine_tune_prefetch(prof, r.strategy, cfg.hardware);
        doc.cost = r.cost;
        doc.gpu_margin = cfg.hardware.gpu_mem - r.cost.peak_gpu;
        doc.cpu_margin = cfg.hardware.cpu_mem - r.cost.cpu_bytes;
        doc.feasible_count = r.feasible_count;
        std::ostringstream s;
        hetsim::write_plan_json(s, doc);
        return emit(s.str(), out, cap);
    });
}

int64_t ah_hetsim_plan_dp_json(const char* text, int32_t dp_size, double collective_gbps, char* out, size_t cap) {
    return guard([&]() -> int64_t {
        const hetsim::RunConfig cfg = hetsim::parse_config(text ? text : "", "<memory>");
        const hetsim::ModelProfile prof = hetsim::build_profile(cfg.model, cfg.hardware, cfg.overrides);
        hetsim::PlanRequest req;
        req.profile = prof;
        req.hardware = cfg.hardware;
        hetsim::dp::DpSpec dp;
        dp.dp_size = dp_size;
        dp.collective_bandwidth = collective_gbps * 1e9;
        const hetsim::PlanResult r = hetsim::dp::solve(req, dp);
        hetsim::PlanDocument doc;
        hetsim::HardwareSpec hw_sim = cfg.hardware;
        hw_sim.gpu_mem = hetsim::dp::simulator_gpu_budget(prof, r.strategy, cfg.hardware.gpu_mem, dp);
        doc.strategy = hetsim::fine_tune_prefetch(hetsim::dp::rank_profile(prof, cfg.hardware, dp), r.strategy, hw_sim);
        doc.cost = r.cost;
        doc.gpu_margin = cfg.hardware.gpu_mem - r.cost.peak_gpu;
        doc.cpu_margin = cfg.hardware.cpu_mem - r.cost.cpu_bytes;
        doc.feasible_count = r.feasible_count;
        std::ostringstream s;
        hetsim::write_plan_json(s, doc);
        return emit(s.str(), out, cap);
    });
}

int64_t ah_hetsim_simulate_trace(const char* text, int32_t c, int32_t p, int32_t o, int32_t n_iters,
                                 int32_t priority, char* out, size_t cap) {
    return guard([&]() -> int64_t {
        const hetsim::RunConfig cfg = hetsim::parse_config(text ? text : "", "<memory>");
        const hetsim::ModelProfile prof = hetsim::build_profile(cfg.model, cfg.hardware, cfg.overrides);
        hetsim::Strategy s;
        if (c >= 0) {
            s = hetsim::Strategy::uniform(c, p, o, prof.num_blocks);
        } else {
            hetsim::PlanRequest req;
            req.profile = prof;
            req.hardware = cfg.hardware;
            s = hetsim::fine_tune_prefetch(prof, hetsim::solve(req).strategy, cfg.hardware);
        }
        const hetsim::SimResult r = hetsim::run(prof, s, cfg.hardware, n_iters, priority != 0);
        std::ostringstream os;
        hetsim::write_chrome_trace(os, r.trace);
        return emit(os.str(), out, cap);
    });
}

}  // extern "C"
