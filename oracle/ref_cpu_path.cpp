// ORACLE / TEST INFRASTRUCTURE — the reference's CPU path for bench.py (cpu_baseline leg and
// `bench.py --impl reference`). Never linked into the product.
//
// Times, on the host cores of the box it runs on:
//   1. the UNMODIFIED reference planner/scheduler (oracle/_ref/libhetsim_ref.a, built from
//      /root/reference/proj/core/src): build_profile -> solve -> fine_tune_prefetch ->
//      run(..., 5, priority=true)  (the library entry of proj/README.md:182-192);
//   2. the CPU optimizer step the reference schedules as OpKind::CpuOptim (simulator.cpp:210-216)
//      for EVERY block of the iteration (offload everything): the reference has no arithmetic
//      for it, so the oracle restatement (adam_oracle.c, AVX-512 clone, OpenMP) runs over one
//      full block of m_p = 12h^2 + 13h parameters (workload.cpp:41-44) in the paper's 14 B/param
//      host layout, L times per iteration — the whole parameter set, timed, not extrapolated.
//
// usage:
//   ref_cpu_path iter L h s b V gpu_mem cpu_mem flops h2d d2h cpu_rate gpu_rate threads iters
//       -> one JSON line per iteration {"plan_s","adam_s","total_s"} then a summary line
//   ref_cpu_path planner reps            -> solve / fine_tune_prefetch wall time at L in
//       {12, 24, 25, 26, 128} on the request of proj/benchmarks/bench_planner.cpp:10-30
//   ref_cpu_path sweep threads n1 n2 ...  -> CPU AdamW params/s and GB/s per size (config C5)
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hetsim/costmodel.hpp"
#include "hetsim/planner.hpp"
#include "hetsim/simulator.hpp"
#include "hetsim/workload.hpp"

extern "C" {
typedef struct {
    float lr, beta1, beta2, eps, weight_decay;
    int32_t step;
} oracle_adam_hparams;
void oracle_adam_f32_mt(const oracle_adam_hparams* hp, float* p, float* m, float* v, const uint16_t* g,
                        uint16_t* out, size_t n, float inv_scale, int nthreads);
}

namespace {

using Clock = std::chrono::steady_clock;

double secs(Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); }

// One block's host state: fp32 master / m / v + the shared bf16 grad -> param buffer.
struct HostBlock {
    std::vector<float> p, m, v;
    std::vector<uint16_t> g;
    explicit HostBlock(size_t n) : p(n), m(n), v(n), g(n) {
#pragma omp parallel for schedule(static)
        for (long long i = 0; i < (long long)n; ++i) {  // first touch in parallel, small values
            p[(size_t)i] = 0.02f * (float)((int)(i % 2003) - 1001) / 1001.f;
            m[(size_t)i] = 0.f;
            v[(size_t)i] = 0.f;
            g[(size_t)i] = (uint16_t)(0x3c00u + (i % 97));
        }
    }
    void step(int t, int threads) {
        oracle_adam_hparams hp{1e-4f, 0.9f, 0.999f, 1e-8f, 0.01f, t};
        oracle_adam_f32_mt(&hp, p.data(), m.data(), v.data(), g.data(), g.data(), p.size(), 1.f, threads);
    }
};

int mode_iter(int argc, char** argv) {
    if (argc < 17) return 2;
    hetsim::ModelSpec m;
    m.num_blocks = std::atoi(argv[2]);
    m.hidden_size = std::atoll(argv[3]);
    m.seq_len = std::atoll(argv[4]);
    m.batch_size = std::atoll(argv[5]);
    m.vocab_size = std::atoll(argv[6]);
    hetsim::HardwareSpec hw;
    hw.gpu_mem = std::atoll(argv[7]);
    hw.cpu_mem = std::atoll(argv[8]);
    hw.gpu_compute_rate = std::atof(argv[9]);
    hw.h2d_bandwidth = std::atof(argv[10]);
    hw.d2h_bandwidth = std::atof(argv[11]);
    hw.cpu_optim_rate = std::atof(argv[12]);
    hw.gpu_optim_rate = std::atof(argv[13]);
    const int threads = std::atoi(argv[14]);
    const int iters = std::atoi(argv[15]);
    const int warm = std::atoi(argv[16]);
    const size_t mp = (size_t)hetsim::block_param_count(m.hidden_size);
    // distinct block buffers cycled over the L blocks: enough that one pass exceeds ~2 GB
    // (> the last-level cache) so small blocks are not timed cache-resident
    const size_t per = mp * 14, want = ((size_t)2 << 30) / (per ? per : 1) + 1;
    const int nbuf = (int)std::min<size_t>((size_t)m.num_blocks, want);
    std::vector<HostBlock*> blks;
    for (int b = 0; b < nbuf; ++b) blks.push_back(new HostBlock(mp));
    for (HostBlock* b : blks) b->step(1, threads);  // page-in / warm
    std::vector<double> totals;
    hetsim::Strategy s;
    double plan_s = 0.0;
    for (int it = 0; it < warm + iters; ++it) {
        const auto t0 = Clock::now();
        const hetsim::ModelProfile pr = hetsim::build_profile(m, hw);
        hetsim::PlanRequest req;
        req.profile = pr;
        req.hardware = hw;
        try {
            s = hetsim::fine_tune_prefetch(pr, hetsim::solve(req).strategy, hw);
            (void)hetsim::run(pr, s, hw, 5, true);
        } catch (const std::exception&) {
            // budgets infeasible for the reference model: the planner call is still timed
        }
        plan_s = secs(t0);
        const auto t1 = Clock::now();
        for (int b = 0; b < m.num_blocks; ++b) blks[(size_t)(b % nbuf)]->step(it + 2, threads);
        const double adam_s = secs(t1);
        if (it >= warm) {
            totals.push_back(plan_s + adam_s);
            std::printf("{\"iter\": %d, \"plan_s\": %.9g, \"adam_s\": %.9g, \"total_s\": %.9g}\n", it - warm, plan_s,
                        adam_s, plan_s + adam_s);
            std::fflush(stdout);
        }
    }
    for (HostBlock* b : blks) delete b;
    std::vector<double> srt = totals;
    std::sort(srt.begin(), srt.end());
    const double med = srt.empty() ? 0.0 : srt[srt.size() / 2];
    const double params = (double)mp * m.num_blocks;
    std::printf("{\"summary\": true, \"median_s\": %.9g, \"params_per_iter\": %.0f, \"block_params\": %zu, "
                "\"threads\": %d, \"adam_params_per_s\": %.9g, \"host_GBps\": %.6g, \"strategy\": [%d, %d, %d]}\n",
                med, params, mp, threads, params / (med - plan_s > 0 ? med - plan_s : med),
                28.0 * params / (med - plan_s > 0 ? med - plan_s : med) / 1e9, s.c_hat, s.p_hat, s.o_hat);
    return 0;
}

// proj/benchmarks/bench_planner.cpp:10-30 (request_for_depth), timed with steady_clock.
hetsim::PlanRequest request_for_depth(int num_blocks) {
    hetsim::ModelSpec m;
    m.num_blocks = num_blocks;
    m.hidden_size = 4096;
    m.seq_len = 1024;
    m.batch_size = 8;
    m.vocab_size = 50257;
    hetsim::HardwareSpec hw;
    hw.gpu_compute_rate = 120e12;
    hw.h2d_bandwidth = hw.d2h_bandwidth = 20e9;
    hw.cpu_optim_rate = 200e6;
    hw.gpu_optim_rate = 20e9;
    hw.cpu_mem = 4ll << 40;
    const hetsim::ModelProfile profile = hetsim::build_profile(m, hw);
    hw.gpu_mem = hetsim::peak_gpu_mem(profile, hetsim::Strategy::uniform(0, 0, num_blocks / 2, num_blocks));
    hetsim::PlanRequest req;
    req.profile = profile;
    req.hardware = hw;
    return req;
}

int mode_planner(int argc, char** argv) {
    const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
    for (int L : {12, 24, 25, 26, 128}) {
        const hetsim::PlanRequest req = request_for_depth(L);
        std::vector<double> ts, tf;
        hetsim::PlanResult r;
        for (int i = 0; i < reps; ++i) {
            auto t0 = Clock::now();
            r = hetsim::solve(req);
            ts.push_back(secs(t0));
            t0 = Clock::now();
            (void)hetsim::fine_tune_prefetch(req.profile, r.strategy, req.hardware);
            tf.push_back(secs(t0));
        }
        std::sort(ts.begin(), ts.end());
        std::sort(tf.begin(), tf.end());
        std::printf("{\"L\": %d, \"solve_s\": %.9g, \"fine_tune_s\": %.9g, \"feasible_count\": %lld, "
                    "\"strategy\": [%d, %d, %d]}\n",
                    L, ts[ts.size() / 2], tf[tf.size() / 2], (long long)r.feasible_count, r.strategy.c_hat,
                    r.strategy.p_hat, r.strategy.o_hat);
        std::fflush(stdout);
    }
    return 0;
}

int mode_sweep(int argc, char** argv) {
    const int threads = std::atoi(argv[2]);
    size_t nmax = 0;
    for (int a = 3; a < argc; ++a) nmax = std::max(nmax, (size_t)std::atoll(argv[a]));
    HostBlock blk(nmax);
    for (int a = 3; a < argc; ++a) {
        const size_t n = (size_t)std::atoll(argv[a]);
        oracle_adam_hparams hp{1e-4f, 0.9f, 0.999f, 1e-8f, 0.01f, 1};
        oracle_adam_f32_mt(&hp, blk.p.data(), blk.m.data(), blk.v.data(), blk.g.data(), blk.g.data(), n, 1.f, threads);
        std::vector<double> t;
        for (int r = 0; r < 5; ++r) {
            hp.step = r + 2;
            const auto t0 = Clock::now();
            oracle_adam_f32_mt(&hp, blk.p.data(), blk.m.data(), blk.v.data(), blk.g.data(), blk.g.data(), n, 1.f,
                               threads);
            t.push_back(secs(t0));
        }
        std::sort(t.begin(), t.end());
        const double med = t[t.size() / 2];
        std::printf("{\"params\": %zu, \"s\": %.9g, \"params_per_s\": %.9g, \"GBps\": %.6g}\n", n, med, n / med,
                    28.0 * n / med / 1e9);
        std::fflush(stdout);
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const char* mode = argc > 1 ? argv[1] : "";
    int rc = 2;
    if (!std::strcmp(mode, "iter")) rc = mode_iter(argc, argv);
    else if (!std::strcmp(mode, "planner")) rc = mode_planner(argc, argv);
    else if (!std::strcmp(mode, "sweep") && argc > 3) rc = mode_sweep(argc, argv);
    if (rc == 2)
        std::fprintf(stderr,
                     "usage: %s iter L h s b V gpu_mem cpu_mem flops h2d d2h cpu_rate gpu_rate threads iters warm\n"
                     "       %s planner reps\n       %s sweep threads n...\n",
                     argv[0], argv[0], argv[0]);
    return rc;
}
