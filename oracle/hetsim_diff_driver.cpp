// ORACLE / TEST INFRASTRUCTURE — not product code.
//
// Differential driver for planner + scheduler parity. The same source is compiled twice:
//   * against the reference headers + the reference core built from
//     /root/reference/proj/core/src/*.cpp   (oracle/_ref/hetsim_diff_ref), and
//   * against include/hetsim + our libhetsim_core.so     (oracle/_ref/hetsim_diff_new).
// Both print a canonical text dump (every double as hexfloat) of
//   solve / InfeasibleError shortfalls        (ref planner.cpp:37-108)
//   fine_tune_prefetch lookaheads             (ref planner.cpp:110-153)
//   baseline_presets                          (ref planner.cpp:155-183)
//   build_iteration_ops                       (ref simulator.cpp:91-229)
//   run() traces, timelines, steady state for FIFO and PS (ref simulator.cpp:263-596)
//   write_chrome_trace / write_memory_csv / write_plan_json bytes
// over seeded random GPT-like cases plus random feasible strategies with random
// lookaheads. tests/test_hetsim_parity.py requires the two dumps to be identical, and
// compares against committed digests in tests/golden/ when /root/reference is absent.
//
// usage: hetsim_diff_<x> <n_cases> <seed>
#include <cstdint>
#include <cstdio>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "hetsim/costmodel.hpp"
#include "hetsim/plan_io.hpp"
#include "hetsim/planner.hpp"
#include "hetsim/simulator.hpp"
#include "hetsim/workload.hpp"

using namespace hetsim;

static void hexd(const char* tag, double x) { std::printf("%s=%a ", tag, x); }

static void dump_profile(const ModelProfile& p) {
    const BlockProfile& b = p.block;
    std::printf("profile L=%d m_a=%lld m_a_in=%lld m_p=%lld m_gc=%lld m_cc=%lld tot=%lld ",
                p.num_blocks, (long long)b.m_a, (long long)b.m_a_in, (long long)b.m_p,
                (long long)p.m_gc, (long long)p.m_cc, (long long)p.total_params);
    hexd("fp", b.t_fp); hexd("bp", b.t_bp); hexd("h2d", b.t_h2d); hexd("d2h", b.t_d2h);
    hexd("ocpu", b.t_opt_cpu); hexd("ogpu", b.t_opt_gpu); hexd("flops", p.flops_per_iter);
    std::printf("\n");
}

static void dump_cost(const CostEstimate& c) {
    hexd("fwd", c.t_fwd); hexd("bwd", c.t_bwd); hexd("sync", c.t_sync);
    std::printf("v=%d peak=%lld cpu=%lld ", c.v_hat, (long long)c.peak_gpu, (long long)c.cpu_bytes);
    hexd("obj", c.objective);
    std::printf("\n");
}

static void dump_strategy(const char* tag, const Strategy& s) {
    std::printf("%s c=%d p=%d o=%d la=", tag, s.c_hat, s.p_hat, s.o_hat);
    for (int x : s.prefetch_lookahead) std::printf("%d,", x);
    std::printf("\n");
}

static void dump_ops(const ModelProfile& p, const Strategy& s, int iter) {
    for (const StreamOp& op : build_iteration_ops(p, s, iter)) {
        std::printf("op %d/%d/%d/%d ", (int)op.kind, op.block, op.iter, (int)op.backward_copy);
        hexd("dur", op.duration);
        std::printf("a=%lld r=%lld deps=", (long long)op.alloc_at_start, (long long)op.release_at_end);
        for (const OpRef& d : op.deps)
            std::printf("%d/%d/%d/%d;", (int)d.kind, d.block, d.iter, (int)d.backward_copy);
        std::printf(" gates=");
        for (const OpRef& g : op.start_after_start_of)
            std::printf("%d/%d/%d/%d;", (int)g.kind, g.block, g.iter, (int)g.backward_copy);
        std::printf("\n");
    }
}

static void dump_run(const ModelProfile& p, const Strategy& s, const HardwareSpec& hw, int n,
                     bool ps) {
    std::printf("run n=%d ps=%d\n", n, (int)ps);
    try {
        const SimResult r = run(p, s, hw, n, ps);
        for (double t : r.iter_times) hexd("it", t);
        hexd("steady", r.steady_state_time);
        hexd("thr", r.throughput);
        std::printf("peak=%lld ntrace=%zu\n", (long long)r.peak_gpu, r.trace.size());
        for (const CompletedOp& op : r.trace) {
            std::printf("t %d/%d/%d/%d/%d ", (int)op.kind, op.block, op.iter,
                        (int)op.backward_copy, (int)op.stream);
            hexd("s", op.start); hexd("e", op.end);
            std::printf("\n");
        }
        for (const auto& m : r.mem_timeline) {
            hexd("m", m.first);
            std::printf("%lld\n", (long long)m.second);
        }
        std::ostringstream tr, csv;
        write_chrome_trace(tr, r.trace);
        write_memory_csv(csv, r.mem_timeline);
        std::printf("TRACE<<\n%sCSV<<\n%s>>\n", tr.str().c_str(), csv.str().c_str());
    } catch (const MemoryExceededError& e) {
        std::printf("MemoryExceeded what=%s op=%d/%d/%d/%d attempted=%lld budget=%lld ", e.what(),
                    (int)e.op().kind, e.op().block, e.op().iter, (int)e.op().backward_copy,
                    (long long)e.attempted_bytes(), (long long)e.budget_bytes());
        hexd("time", e.time());
        std::printf("\n");
    } catch (const std::exception& e) {
        std::printf("exception %s\n", e.what());
    }
}

int main(int argc, char** argv) {
    const int n_cases = argc > 1 ? std::atoi(argv[1]) : 200;
    const unsigned long long seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 424242ULL;
    std::mt19937_64 rng(seed);
    const std::int64_t hiddens[] = {512, 768, 1024, 2048, 4096, 6144, 8192};
    const std::int64_t seqs[] = {512, 1024, 2048};
    const std::int64_t batches[] = {1, 4, 8, 16};

    for (int cs = 0; cs < n_cases; ++cs) {
        ModelSpec m;
        m.num_blocks = 2 + (int)(rng() % 31);
        m.hidden_size = hiddens[rng() % 7];
        m.seq_len = seqs[rng() % 3];
        m.batch_size = batches[rng() % 4];
        m.vocab_size = 50257;
        if (rng() % 4 == 0) m.activation_coef = 8.0 + (double)(rng() % 1000) / 37.0;
        HardwareSpec hw;
        hw.gpu_compute_rate = (20.0 + (double)(rng() % 200000) / 100.0) * 1e12;
        hw.h2d_bandwidth = (8.0 + (double)(rng() % 6000) / 100.0) * 1e9;
        hw.d2h_bandwidth = (8.0 + (double)(rng() % 6000) / 100.0) * 1e9;
        hw.cpu_optim_rate = (50.0 + (double)(rng() % 400000) / 100.0) * 1e6;
        hw.gpu_optim_rate = (5.0 + (double)(rng() % 50000) / 100.0) * 1e9;
        hw.cpu_mem = (rng() % 5 == 0) ? ((std::int64_t)(rng() % 200) << 30)
                                      : ((std::int64_t)2048 << 30);
        const ModelProfile pr = build_profile(m, hw);
        const int L = pr.num_blocks;
        const std::int64_t lo = peak_gpu_mem(pr, Strategy::uniform(L, L, L, L));
        const std::int64_t hi = peak_gpu_mem(pr, Strategy::uniform(0, 0, 0, L));
        const double frac = (double)(rng() % 1200) / 1000.0;
        hw.gpu_mem = lo + (std::int64_t)(frac * (double)(hi - lo));
        if (rng() % 9 == 0) hw.gpu_mem /= 3;

        std::printf("=== case %d L=%d h=%lld s=%lld b=%lld coef=%a gpu_mem=%lld cpu_mem=%lld\n", cs,
                    L, (long long)m.hidden_size, (long long)m.seq_len, (long long)m.batch_size,
                    m.activation_coef, (long long)hw.gpu_mem, (long long)hw.cpu_mem);
        dump_profile(pr);

        PlanRequest req;
        req.profile = pr;
        req.hardware = hw;
        Strategy plan;
        bool feasible = true;
        try {
            const PlanResult r = solve(req);
            plan = r.strategy;
            dump_strategy("solve", r.strategy);
            dump_cost(r.cost);
            std::printf("feasible=%lld\n", (long long)r.feasible_count);
            PlanDocument doc;
            doc.strategy = r.strategy;
            doc.cost = r.cost;
            doc.gpu_margin = hw.gpu_mem - r.cost.peak_gpu;
            doc.cpu_margin = hw.cpu_mem - r.cost.cpu_bytes;
            doc.feasible_count = r.feasible_count;
            std::ostringstream pj;
            write_plan_json(pj, doc);
            std::printf("PLAN<<\n%s>>\n", pj.str().c_str());
        } catch (const InfeasibleError& e) {
            feasible = false;
            std::printf("infeasible gpu=%lld cpu=%lld cap=%lld what=%s\n",
                        (long long)e.gpu_shortfall_bytes(), (long long)e.cpu_shortfall_bytes(),
                        (long long)e.gpu_shortfall_at_cpu_cap_bytes(), e.what());
        }
        for (const auto& [name, s] : baseline_presets(pr, hw)) dump_strategy(name.c_str(), s);

        if (feasible) {
            Strategy tuned = plan;
            try {
                tuned = fine_tune_prefetch(pr, plan, hw);
            } catch (const std::exception& e) {
                std::printf("tuned exception %s\n", e.what());
            }
            dump_strategy("tuned", tuned);
            dump_ops(pr, tuned, 2);
            dump_run(pr, tuned, hw, 3, false);
            dump_run(pr, tuned, hw, 3, true);
        }
        // A random strategy (feasible or not) with random lookaheads: exercises P-block
        // gates, envelope / runahead guards and the MemoryExceeded path.
        Strategy r;
        r.o_hat = (int)(rng() % (unsigned)(L + 1));
        r.p_hat = (int)(rng() % (unsigned)(r.o_hat + 1));
        r.c_hat = (int)(rng() % (unsigned)(L + 1));
        r.prefetch_lookahead.assign((std::size_t)L, 1);
        for (int i = 0; i < L; ++i) r.prefetch_lookahead[(std::size_t)i] = 1 + (int)(rng() % 4);
        HardwareSpec hw2 = hw;
        hw2.gpu_mem = std::max<std::int64_t>(hw.gpu_mem, peak_gpu_mem(pr, r)) -
                      ((rng() % 3 == 0) ? (std::int64_t)(rng() % (std::uint64_t)(2 * pr.block.m_p + 1)) : 0);
        dump_strategy("random", r);
        dump_cost(evaluate(pr, r));
        dump_ops(pr, r, 1);
        dump_run(pr, r, hw2, 2 + (int)(rng() % 3), false);
        dump_run(pr, r, hw2, 2 + (int)(rng() % 3), true);
        try {
            const Strategy rt = fine_tune_prefetch(pr, r, hw2);
            dump_strategy("random_tuned", rt);
        } catch (const std::exception& e) {
            std::printf("random_tuned exception %s\n", e.what());
        }
    }
    return 0;
}
