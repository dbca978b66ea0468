// ORACLE / TEST INFRASTRUCTURE — the reference's CPU path for bench.py (cpu_baseline leg and
// `bench.py --impl reference`). Never linked into the product.
//
// Times, on the host cores of the box it runs on:
//   1. the UNMODIFIED reference planner/scheduler (oracle/_ref/libhetsim_ref.a, built from
//      /root/reference/proj/core/src): build_profile -> solve -> fine_tune_prefetch ->
//      run(..., 5, priority=true)  (the library entry of proj/README.md:182-192);
//   2. the CPU optimizer step the reference schedules as OpKind::CpuOptim (simulator.cpp:210-216):
//      the reference has no arithmetic for it, so the oracle restatement (adam_oracle.c,
//      OpenMP over nthreads) is timed on a bounded sample of parameters.
// usage: ref_cpu_path L h s b V gpu_mem cpu_mem flops h2d d2h cpu_rate gpu_rate sample_params threads reps
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

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

int main(int argc, char** argv) {
    if (argc < 16) {
        std::fprintf(stderr, "usage: %s L h s b V gpu_mem cpu_mem flops h2d d2h cpu_rate gpu_rate sample threads reps\n", argv[0]);
        return 2;
    }
    using Clock = std::chrono::steady_clock;
    hetsim::ModelSpec m;
    m.num_blocks = std::atoi(argv[1]);
    m.hidden_size = std::atoll(argv[2]);
    m.seq_len = std::atoll(argv[3]);
    m.batch_size = std::atoll(argv[4]);
    m.vocab_size = std::atoll(argv[5]);
    hetsim::HardwareSpec hw;
    hw.gpu_mem = std::atoll(argv[6]);
    hw.cpu_mem = std::atoll(argv[7]);
    hw.gpu_compute_rate = std::atof(argv[8]);
    hw.h2d_bandwidth = std::atof(argv[9]);
    hw.d2h_bandwidth = std::atof(argv[10]);
    hw.cpu_optim_rate = std::atof(argv[11]);
    hw.gpu_optim_rate = std::atof(argv[12]);
    const size_t sample = (size_t)std::atoll(argv[13]);
    const int threads = std::atoi(argv[14]);
    const int reps = std::atoi(argv[15]);

    // 1. planner + scheduler (reference library)
    double plan_s = 1e30;
    hetsim::Strategy s;
    double sim_steady = 0.0;
    std::int64_t total_params = 0;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = Clock::now();
        const hetsim::ModelProfile pr = hetsim::build_profile(m, hw);
        hetsim::PlanRequest req;
        req.profile = pr;
        req.hardware = hw;
        const hetsim::PlanResult plan = hetsim::solve(req);
        s = hetsim::fine_tune_prefetch(pr, plan.strategy, hw);
        const hetsim::SimResult sim = hetsim::run(pr, s, hw, 5, true);
        const double dt = std::chrono::duration<double>(Clock::now() - t0).count();
        if (dt < plan_s) plan_s = dt;
        sim_steady = sim.steady_state_time;
        total_params = pr.total_params;
    }
    // 2. CPU AdamW (oracle restatement) on a bounded sample, 14 B/param host layout
    std::vector<float> p(sample), mm(sample, 0.f), vv(sample, 0.f);
    std::vector<uint16_t> g(sample);
    for (size_t i = 0; i < sample; ++i) {
        p[i] = 0.02f * (float)((int)(i % 2003) - 1001) / 1001.f;
        g[i] = (uint16_t)(0x3c00u + (i % 97));  // small positive bf16 grads
    }
    oracle_adam_hparams hp{1e-4f, 0.9f, 0.999f, 1e-8f, 0.01f, 1};
    oracle_adam_f32_mt(&hp, p.data(), mm.data(), vv.data(), g.data(), g.data(), sample, 1.f, threads);  // warm
    double adam_s = 1e30;
    for (int r = 0; r < reps; ++r) {
        hp.step = r + 2;
        const auto t0 = Clock::now();
        oracle_adam_f32_mt(&hp, p.data(), mm.data(), vv.data(), g.data(), g.data(), sample, 1.f, threads);
        const double dt = std::chrono::duration<double>(Clock::now() - t0).count();
        if (dt < adam_s) adam_s = dt;
    }
    std::printf("{\"plan_s\": %.9g, \"adam_sample_params\": %zu, \"adam_sample_s\": %.9g, "
                "\"adam_params_per_s\": %.9g, \"total_params\": %lld, \"threads\": %d, "
                "\"strategy\": [%d, %d, %d], \"sim_steady_s\": %.9g}\n",
                plan_s, sample, adam_s, (double)sample / adam_s, (long long)total_params, threads, s.c_hat, s.p_hat,
                s.o_hat, sim_steady);
    return 0;
}
