// B200 executor of the planned AutoHete iteration (see executor.h).
#include "executor.h"
#include "hetsim/dp_planner.hpp"
#include "loopback_comm.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <sstream>
#include <stdexcept>

#include "../kernels/gemm.h"
#include "../kernels/gpt_kernels.h"
#include "../kernels/kernels.h"
#include "adam_scalars.h"
#include "hetsim/costmodel.hpp"
#include "hetsim/workload.hpp"

#include <nccl.h>
#include <cstdlib>

namespace ah {

void cpu_adam(const ah_adam_hparams& hp, float* p, float* m, float* v, const uint16_t* g, uint16_t* p_bf16,
              std::size_t n, float inv_scale, int nthreads);
void cpu_cast_f32_bf16(const float* src, uint16_t* dst, std::size_t n, int nthreads);

namespace {

using hetsim::OpKind;
using Clock = std::chrono::steady_clock;

int lane_of(OpKind k) { return static_cast<int>(hetsim::stream_of(k)) - 1; }

void host_zero(void* p, size_t bytes) {
    if (bytes == 0) return;
    char* c = static_cast<char*>(p);
    const size_t chunk = (size_t)1 << 24;
    const long long n = (long long)((bytes + chunk - 1) / chunk);
#pragma omp parallel for schedule(dynamic, 1)
    for (long long i = 0; i < n; ++i) {
        const size_t a = (size_t)i * chunk;
        std::memset(c + a, 0, std::min(chunk, bytes - a));
    }
}

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

AdamArgs adam_args(const ah_adam_hparams& hp, int step, float* p, float* m, float* v, const uint16_t* g,
                   uint16_t* out, size_t n) {
    ah_adam_hparams h = hp;
    h.step = step;
    const AdamConsts c = derive_adam_scalars(h);
    AdamArgs a;
    a.p = p;
    a.m = m;
    a.v = v;
    a.g = g;
    a.p_bf16 = out;
    a.n = n;
    a.decay = c.decay;
    a.beta1 = c.beta1;
    a.one_minus_beta1 = c.one_minus_beta1;
    a.beta2 = c.beta2;
    a.one_minus_beta2 = c.one_minus_beta2;
    a.step_size = c.step_size;
    a.inv_sqrt_bc2 = c.inv_sqrt_bc2;
    a.eps = c.eps;
    a.inv_scale = 1.f;
    return a;
}

}  // namespace

void Trainer::check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

cudaStream_t Trainer::stream_of(int lane) const {
    return lane == kCompute ? s_compute_ : (lane == kH2D ? s_h2d_ : s_d2h_);
}

Trainer::Trainer(const ah_trainer_config& cfg) {
    d_.L = cfg.num_blocks;
    d_.h = cfg.hidden;
    d_.nh = cfg.heads;
    d_.hd = cfg.heads > 0 ? cfg.hidden / cfg.heads : 0;
    d_.s = cfg.seq_len;
    d_.B = cfg.batch;
    d_.V = cfg.vocab;
    // padded vocabulary: a multiple of the 256-column GEMM tile, so the LM-head GEMMs take the
    // lean epilogue (N % 256 == 0); padding rows of wte are zero and masked out of the loss
    d_.Vp = (int)round_up((size_t)cfg.vocab, 256);
    if (d_.L < 1 || d_.h % 64 || d_.nh < 1 || d_.h % d_.nh || d_.hd % 64 || d_.s % 128 || d_.B < 1 || d_.V < 2 ||
        d_.T() > 16384)
        throw std::invalid_argument(
            "trainer: need h % 64 == 0, head_dim % 64 == 0, seq_len % 128 == 0, batch*seq <= 16384");
    adam_ = cfg.adam;
    seed_ = cfg.seed ? cfg.seed : 1234;
    cpu_threads_ = cfg.cpu_threads;
    ps_ = cfg.priority_sched != 0;
    dp_rank_ = cfg.dp_rank;
    dp_size_ = cfg.dp_size < 1 ? 1 : cfg.dp_size;
    dp_ = dp_size_ > 1 || cfg.force_collectives;
    if (dp_rank_ < 0 || dp_rank_ >= dp_size_) throw std::invalid_argument("trainer: dp_rank out of range");
    loop_ = static_cast<LoopbackComm*>(cfg.loopback_comm);
    if (loop_ && loop_->size() != dp_size_) throw std::invalid_argument("trainer: loopback comm size != dp_size");
    if (dp_) {
        shard_ = round_up((d_.m_p() + dp_size_ - 1) / dp_size_, 8);
        const size_t off = shard_ * (size_t)dp_rank_;
        my_len_ = off >= d_.m_p() ? 0 : std::min(shard_, d_.m_p() - off);
    }
    if (dp_ && !loop_) {
        ncclUniqueId id;
        static_assert(sizeof(id) == 128, "ncclUniqueId size");
        std::memcpy(&id, cfg.nccl_id, sizeof(id));
        ncclComm_t comm;
        const ncclResult_t r = ncclCommInitRank(&comm, dp_size_, id, dp_rank_);
        if (r != ncclSuccess) throw std::runtime_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        comm_ = comm;
    }
    int lo = 0, hi = 0;
    check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    check(cudaStreamCreateWithPriority(&s_compute_, cudaStreamNonBlocking, hi), "stream");
    check(cudaStreamCreateWithPriority(&s_h2d_, cudaStreamNonBlocking, lo), "stream");
    check(cudaStreamCreateWithPriority(&s_d2h_, cudaStreamNonBlocking, lo), "stream");
    check(cudaStreamCreateWithPriority(&s_side_, cudaStreamNonBlocking, hi), "stream");
    check(cudaStreamCreateWithFlags(&s_mark_, cudaStreamNonBlocking), "stream");
    check(cudaEventCreateWithFlags(&ev_c2s_, cudaEventDisableTiming), "event");
    check(cudaEventCreateWithFlags(&ev_s2c_, cudaEventDisableTiming), "event");
    check(cudaGetDevice(&device_), "get device");
    plan(cfg);
    allocate_and_init();
    for (int l = 0; l < 4; ++l) lanes_[l] = std::thread([this, l] { lane_main(l); });
}

Trainer::~Trainer() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : lanes_)
        if (t.joinable()) t.join();
    cudaDeviceSynchronize();
    if (comm_) ncclCommDestroy(static_cast<ncclComm_t>(comm_));
    for (Iter* it : iters_) {
        for (auto& kv : it->ops) {
            RtOp& o = kv.second;
            for (cudaEvent_t e : {o.done_ev, o.start_ev, o.t0, o.t1})
                if (e) cudaEventDestroy(e);
            for (cudaEvent_t e : o.ct) cudaEventDestroy(e);
        }
        delete it;
    }
    for (size_t i = 1; i < blocks_.size(); ++i) {
        BlockState& b = blocks_[i];
        if (b.o) {
            cudaFreeHost(b.master);
            cudaFreeHost(b.m1);
            cudaFreeHost(b.m2);
            cudaFreeHost(b.host_bf16);
        } else {
            cudaFree(b.master);
            cudaFree(b.m1);
            cudaFree(b.m2);
        }

    }
    for (uint16_t* x : x_) cudaFree(x);
    if (acts_arena_) cudaFree(acts_arena_);
    for (uint16_t* p : wslot_ptr_) cudaFree(p);
    for (cudaEvent_t e : wslot_ev_)
        if (e) cudaEventDestroy(e);
    for (void* p : {(void*)gx_[0], (void*)gx_[1], ws_mem_, (void*)wte_, (void*)wte_m_, (void*)wte_v_, (void*)wpe_,
                    (void*)wpe_m_, (void*)wpe_v_, (void*)lnf_, (void*)lnf_m_, (void*)lnf_v_, (void*)wte_b_,
                    (void*)wpe_b_, (void*)lnf_b_, (void*)dwte_, (void*)dwpe_, (void*)dwte_b_, (void*)dwpe_b_,
                    (void*)dlnf_b_, (void*)logits_, (void*)xf_, (void*)meanf_, (void*)rstdf_, (void*)losses_,
                    (void*)loss_dev_, (void*)tok_dev_, (void*)gstats_dev_})
        if (p) cudaFree(p);
    if (loss_host_) cudaFreeHost(loss_host_);
    if (gstats_host_) cudaFreeHost(gstats_host_);
    if (tok_host_) cudaFreeHost(tok_host_);
    cudaStreamDestroy(s_compute_);
    cudaStreamDestroy(s_h2d_);
    cudaStreamDestroy(s_side_);
    cudaEventDestroy(ev_c2s_);
    cudaEventDestroy(ev_s2c_);
    for (BlockState& b : blocks_) {
        if (b.mat_ev) cudaEventDestroy(b.mat_ev);
        for (cudaEvent_t e : b.go_ev) cudaEventDestroy(e);
    }
    cudaStreamDestroy(s_d2h_);
    cudaStreamDestroy(s_mark_);
}

// ---------------------------------------------------------------------------------------
// Planning: profile from the real block shape, then the reference planner API.
// ---------------------------------------------------------------------------------------
void Trainer::plan(const ah_trainer_config& cfg) {
    const size_t T = d_.T(), h = d_.h;
    dp_spec_.dp_size = dp_size_;
    dp_spec_.collective_bandwidth = cfg.collective_bw;
    hetsim::ModelSpec spec;
    spec.num_blocks = d_.L;
    spec.hidden_size = d_.h;
    spec.seq_len = d_.s;
    spec.batch_size = d_.B;
    spec.vocab_size = d_.V;
    // Real activation bytes of a block (input + saved set) over the 2*b*s*h unit.
    spec.activation_coef = (double)(BlockActs::bytes(d_) + T * h * 2) / (double)(2 * T * h);
    spec.bwd_fwd_ratio = cfg.bwd_fwd_ratio > 0 ? cfg.bwd_fwd_ratio : 2.0;
    hw_.gpu_mem = cfg.gpu_mem_budget;
    hw_.cpu_mem = cfg.cpu_mem_budget;
    hw_.gpu_compute_rate = cfg.gpu_flops;
    hw_.h2d_bandwidth = cfg.h2d_bw;
    hw_.d2h_bandwidth = cfg.d2h_bw;
    hw_.cpu_optim_rate = cfg.cpu_adam_rate;
    hw_.gpu_optim_rate = cfg.gpu_adam_rate;
    // Constant GPU residue of this runtime: embedding/positions/final-LN state (fp32 master,
    // m, v, bf16 copy, fp32 + bf16 grads), logits, head scratch, residual streams, workspace.
    const size_t emb = (size_t)d_.Vp * h + (size_t)d_.s * h + 2 * h;
    size_t m_gc = emb * (12 + 2 + 4 + 2) + T * (size_t)d_.Vp * 2 + T * h * 2 + T * 16;
    m_gc += (size_t)(d_.L + 1) * T * h * 2 + 2 * T * h * 2 + Workspace::bytes(d_);
    hetsim::ProfileOverrides ov;
    ov.m_gc = (std::int64_t)m_gc;
    spec_ = spec;
    ov_ = ov;
    hw_cfg_ = hw_;
    fine_tune_ = cfg.fine_tune != 0;
    profile_ = hetsim::build_profile(spec, hw_, ov);
    const int L = d_.L;
    if (cfg.c_hat >= 0 && cfg.p_hat >= 0 && cfg.o_hat >= 0) {
        strategy_ = hetsim::Strategy::uniform(cfg.c_hat, cfg.p_hat, cfg.o_hat, L);
        if (cfg.prefetch_lookahead)
            for (int i = 0; i < L; ++i) strategy_.prefetch_lookahead[(size_t)i] = cfg.prefetch_lookahead[i];
        strategy_.validate(L);
    } else if (dp_size_ > 1 && cfg.dp_aware_plan) {  // data-parallel extension (dp_planner.hpp)
        hetsim::PlanRequest req;
        req.profile = profile_;
        req.hardware = hw_;
        strategy_ = hetsim::dp::solve(req, dp_spec_).strategy;
    } else {
        hetsim::PlanRequest req;
        req.profile = profile_;
        req.hardware = hw_;
        strategy_ = hetsim::solve(req).strategy;
    }
    if (dp_size_ > 1 && cfg.dp_aware_plan) {
        // schedule on the per-rank durations; the simulator's (unsharded) memory model gets the
        // budget that admits the realised per-rank footprint
        const hetsim::ModelProfile full = profile_;
        profile_ = hetsim::dp::rank_profile(full, hw_, dp_spec_);
        hw_.gpu_mem = hetsim::dp::simulator_gpu_budget(full, strategy_, hw_.gpu_mem, dp_spec_);
    }
    if (cfg.fine_tune) strategy_ = hetsim::fine_tune_prefetch(profile_, strategy_, hw_);
    sim_ = hetsim::run(profile_, strategy_, hw_, 3, ps_);
    sim_steady_[ps_ ? 1 : 0] = sim_.steady_state_time;
    try {  // the other schedule of the same plan, for the PS-vs-FIFO comparison
        sim_steady_[ps_ ? 0 : 1] = hetsim::run(profile_, strategy_, hw_, 3, !ps_).steady_state_time;
    } catch (const std::exception&) {
        sim_steady_[ps_ ? 0 : 1] = std::nan("");
    }
    compile_order();
}

// Per-lane op order of iteration 1 and of the steady state (iteration 2) from the scheduler.
void Trainer::compile_order() {
    for (auto& it : order_)
        for (auto& lane : it) lane.clear();
    for (double& x : sim_lane_ms_) x = 0.0;
    for (const hetsim::CompletedOp& op : sim_.trace) {
        if (op.iter > 2) continue;
        order_[op.iter - 1][lane_of(op.kind)].push_back({(int)op.kind, op.block, op.backward_copy});
        if (op.iter == 2) sim_lane_ms_[lane_of(op.kind)] += (op.end - op.start) * 1e3;
    }
}

void Trainer::calibrate(ah_calibration* out) {
    drain();
    std::memset(out, 0, sizeof(*out));
    double sum[7] = {0}, cnt[7] = {0};  // F, B, R, H2D, D2H, CPU, GPU-opt
    {
        std::lock_guard<std::mutex> lk(mu_);
        // a trainer's first iteration runs an empty pipeline and pays one-time costs (lazy module
        // loading of every kernel, first tensor maps): it is left out when later ones are in the window
        const bool skip_first = iters_.size() > 1;
        for (Iter* it : iters_)
            for (auto& kv : it->ops) {
                if (skip_first && it->k == 1) continue;
                const RtOp& o = kv.second;
                int k = -1;
                switch (o.kind) {
                    case OpKind::Forward: k = 0; break;
                    case OpKind::Backward: k = 1; break;
                    case OpKind::Recompute: k = 2; break;
                    case OpKind::ParamPrefetch: k = blocks_[(size_t)o.block].o ? 3 : -1; break;  // PCIe copies only
                    case OpKind::GradOffload: k = 4; break;
                    case OpKind::CpuOptim: k = 5; break;
                    case OpKind::GpuOptim: k = 6; break;
                    default: break;
                }
                if (k < 0) continue;
                double ms = o.host_ms;
                if (o.lane != kCpu) {
                    ms = op_ms(o);
                    if (ms < 0) continue;
                }
                sum[k] += ms / 1e3;
                cnt[k] += 1;
            }
    }
    auto mean = [&](int k) { return cnt[k] > 0 ? sum[k] / cnt[k] : 0.0; };
    out->t_fwd_s = mean(0);
    out->t_bwd_s = mean(1);
    out->t_recompute_s = mean(2);
    out->t_h2d_s = mean(3);
    out->t_d2h_s = mean(4);
    out->t_opt_cpu_s = mean(5);
    out->t_opt_gpu_s = mean(6);
    // the running plan in the reference cost model with the measured durations
    hetsim::ModelProfile cal = profile_;
    hetsim::BlockProfile& b = cal.block;
    if (cnt[0] > 0) b.t_fp = out->t_fwd_s;
    if (cnt[1] > 0) b.t_bp = out->t_bwd_s;
    if (cnt[3] > 0) b.t_h2d = out->t_h2d_s;
    if (cnt[4] > 0) b.t_d2h = out->t_d2h_s;
    if (cnt[5] > 0) b.t_opt_cpu = out->t_opt_cpu_s;
    if (cnt[6] > 0) b.t_opt_gpu = out->t_opt_gpu_s;
    out->sim_steady_s = hetsim::run(cal, strategy_, hw_, 3, ps_).steady_state_time;
    try {
        out->sim_steady_other_s = hetsim::run(cal, strategy_, hw_, 3, !ps_).steady_state_time;
    } catch (const std::exception&) {
        out->sim_steady_other_s = std::nan("");
    }
    out->c_hat = out->p_hat = out->o_hat = -1;
    cal_valid_ = cal_plan_valid_ = false;
    if (dp_size_ > 1) return;
    // the plan the reference planner picks with these durations expressed as HardwareSpec rates
    // (the inverse of estimate_block_times, workload.cpp:55-73)
    hetsim::HardwareSpec hw = hw_cfg_;
    hetsim::ModelSpec spec = spec_;
    const double mp = (double)profile_.block.m_p;
    const double flops = 2.0 * mp * (double)d_.T() + 4.0 * d_.B * (double)d_.s * d_.s * d_.h;
    hw.gpu_compute_rate = flops / b.t_fp;
    spec.bwd_fwd_ratio = b.t_bp / b.t_fp;
    hw.h2d_bandwidth = 2.0 * mp / b.t_h2d;
    hw.d2h_bandwidth = 2.0 * mp / b.t_d2h;
    hw.cpu_optim_rate = mp / b.t_opt_cpu;
    hw.gpu_optim_rate = mp / b.t_opt_gpu;
    out->gpu_flops = hw.gpu_compute_rate;
    out->bwd_fwd_ratio = spec.bwd_fwd_ratio;
    out->h2d_bw = hw.h2d_bandwidth;
    out->d2h_bw = hw.d2h_bandwidth;
    out->cpu_adam_rate = hw.cpu_optim_rate;
    out->gpu_adam_rate = hw.gpu_optim_rate;
    cal_hw_ = hw;
    cal_spec_ = spec;
    cal_valid_ = true;
    try {
        const hetsim::ModelProfile pr = hetsim::build_profile(spec, hw, ov_);
        hetsim::PlanRequest req;
        req.profile = pr;
        req.hardware = hw;
        hetsim::Strategy st = hetsim::solve(req).strategy;
        if (fine_tune_) st = hetsim::fine_tune_prefetch(pr, st, hw);
        out->c_hat = st.c_hat;
        out->p_hat = st.p_hat;
        out->o_hat = st.o_hat;
        out->sim_steady_replan_s = hetsim::run(pr, st, hw, 3, ps_).steady_state_time;
        cal_strategy_ = st;
        cal_plan_valid_ = true;
    } catch (const std::exception&) {
        // infeasible with these rates: report no plan
    }
}

bool Trainer::apply_calibration(bool keep_strategy) {
    if (!cal_valid_ || dp_size_ > 1) return false;
    const bool same = cal_plan_valid_ && cal_strategy_.c_hat == strategy_.c_hat &&
                      cal_strategy_.p_hat == strategy_.p_hat && cal_strategy_.o_hat == strategy_.o_hat;
    if (!keep_strategy && !same) return false;
    drain();
    // build everything first (the scheduler may throw), then commit
    const hetsim::ModelProfile profile = hetsim::build_profile(cal_spec_, cal_hw_, ov_);
    const hetsim::Strategy strategy = keep_strategy ? strategy_ : cal_strategy_;  // same (c, p, o)
    hetsim::SimResult sim = hetsim::run(profile, strategy, cal_hw_, 3, ps_);
    double other = std::nan("");
    try {
        other = hetsim::run(profile, strategy, cal_hw_, 3, !ps_).steady_state_time;
    } catch (const std::exception&) {
    }
    hw_ = cal_hw_;
    spec_ = cal_spec_;
    profile_ = profile;
    strategy_ = strategy;
    sim_ = std::move(sim);
    sim_steady_[ps_ ? 1 : 0] = sim_.steady_state_time;
    sim_steady_[ps_ ? 0 : 1] = other;
    compile_order();
    return true;
}

void Trainer::set_schedule(bool priority) {
    drain();  // every lane idle: the next iteration starts on the new order
    if (priority == ps_) return;
    hetsim::SimResult sim = hetsim::run(profile_, strategy_, hw_, 3, priority);  // may throw: commit after
    ps_ = priority;
    sim_ = std::move(sim);
    compile_order();
}

// ---------------------------------------------------------------------------------------
void Trainer::allocate_and_init() {
    const size_t T = d_.T(), h = d_.h, mp = d_.m_p();
    const BlockLayout lay = BlockLayout::make(h);
    check(cudaDeviceGetDefaultMemPool(&pool_, device_), "mempool");  // this rank's GPU, not GPU 0
    uint64_t thr = UINT64_MAX;
    check(cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrReleaseThreshold, &thr), "mempool attr");
    size_t stat = 0;
    auto dalloc = [&](void** p, size_t bytes) {
        check(cudaMalloc(p, bytes), "cudaMalloc");
        stat += bytes;
    };
    x_.assign((size_t)d_.L + 1, nullptr);
    for (auto& x : x_) dalloc((void**)&x, T * h * 2);
    dalloc((void**)&gx_[0], T * h * 2);
    dalloc((void**)&gx_[1], T * h * 2);
    dalloc(&ws_mem_, Workspace::bytes(d_));
    ws_ = Workspace::carve(d_, ws_mem_);
    const size_t nwte = (size_t)d_.Vp * h, nwpe = (size_t)d_.s * h;
    for (float** p : {&wte_, &wte_m_, &wte_v_, &dwte_}) dalloc((void**)p, nwte * 4);
    for (float** p : {&wpe_, &wpe_m_, &wpe_v_, &dwpe_}) dalloc((void**)p, nwpe * 4);
    for (float** p : {&lnf_, &lnf_m_, &lnf_v_}) dalloc((void**)p, 2 * h * 4);
    dalloc((void**)&wte_b_, nwte * 2);
    dalloc((void**)&dwte_b_, nwte * 2);
    dalloc((void**)&wpe_b_, nwpe * 2);
    dalloc((void**)&dwpe_b_, nwpe * 2);
    dalloc((void**)&lnf_b_, 2 * h * 2);
    dalloc((void**)&dlnf_b_, 2 * h * 2);
    dalloc((void**)&logits_, T * (size_t)d_.Vp * 2);
    dalloc((void**)&xf_, T * h * 2);
    for (float** p : {&meanf_, &rstdf_, &losses_}) dalloc((void**)p, T * 4);
    dalloc((void**)&loss_dev_, 256);  // [0] mean loss, [1] (int) out-of-range id flag
    dalloc((void**)&gstats_dev_, (size_t)(d_.L + 1) * AH_STATS_FLOATS * 4);
    inv_words_ = 5 * T + 8;
    dalloc((void**)&tok_dev_, 2 * inv_words_ * 4);
    check(cudaHostAlloc((void**)&loss_host_, 64, cudaHostAllocPortable), "host alloc");
    check(cudaHostAlloc((void**)&gstats_host_, (size_t)(d_.L + 1) * 8, cudaHostAllocPortable), "host alloc");
    std::memset(gstats_host_, 0, (size_t)(d_.L + 1) * 8);
    check(cudaHostAlloc((void**)&tok_host_, 2 * 2 * T * 4, cudaHostAllocPortable), "host alloc");

    cudaStream_t st = s_compute_;
    const float std_res = 0.02f / std::sqrt(2.f * d_.L);
    float* tmp = nullptr;
    uint16_t* tmpb = nullptr;
    check(cudaMalloc(&tmp, mp * 4), "tmp");
    check(cudaMalloc(&tmpb, mp * 2), "tmp");
    blocks_.assign((size_t)d_.L + 1, BlockState{});
    const int L = d_.L;
    {   // sub-block streaming of the offload chain: ~16 MB bf16 chunks, at most 16 per block
        const size_t n = dp_ ? shard_ : mp;
        double mb = 16.0;
        if (const char* e = std::getenv("AH_STREAM_CHUNK_MB")) mb = std::atof(e);  // 0 = whole blocks
        nsub_ = mb > 0 ? (int)std::min<double>(16.0, std::max(1.0, std::floor(2.0 * (double)n / (mb * 1e6)))) : 1;
        if (n < 2 * 16384) nsub_ = 1;
    }
    for (int i = 1; i <= L; ++i) {
        BlockState& b = blocks_[(size_t)i];
        b.c = i <= strategy_.c_hat;
        b.p = i <= strategy_.p_hat;
        b.o = i > L - strategy_.o_hat;
        const unsigned long long s = seed_ * 1000003ull + (unsigned long long)i * 7919ull;
        check(gpt::init_normal(tmp + lay.w_qkv, 3 * h * h, s + 1, 0.f, 0.02f, st), "init");
        check(gpt::init_normal(tmp + lay.w_proj, h * h, s + 2, 0.f, std_res, st), "init");
        check(gpt::init_normal(tmp + lay.w_fc, 4 * h * h, s + 3, 0.f, 0.02f, st), "init");
        check(gpt::init_normal(tmp + lay.w_fc2, 4 * h * h, s + 4, 0.f, std_res, st), "init");
        check(gpt::fill_f32(tmp + lay.b_qkv, lay.ln1_g - lay.b_qkv, 0.f, st), "init");
        check(gpt::fill_f32(tmp + lay.ln1_g, h, 1.f, st), "init");
        check(gpt::fill_f32(tmp + lay.ln1_b, h, 0.f, st), "init");
        check(gpt::fill_f32(tmp + lay.ln2_g, h, 1.f, st), "init");
        check(gpt::fill_f32(tmp + lay.ln2_b, h, 0.f, st), "init");
        // this rank's part of the fp32 state: the whole block, or its DP shard (zero padded)
        const size_t n = dp_ ? shard_ : mp;
        const size_t off = dp_ ? shard_ * (size_t)dp_rank_ : 0;
        const size_t valid = dp_ ? my_len_ : mp;
        if (b.o && nsub_ > 1) {
            b.go_ev.assign((size_t)nsub_, nullptr);
            for (cudaEvent_t& e : b.go_ev) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        }
        if (b.o) {
            // optimizer state in pinned host DRAM: 12 B/param + shared 2 B param/grad buffer
            check(cudaHostAlloc((void**)&b.master, n * 4, cudaHostAllocPortable), "host alloc");
            check(cudaHostAlloc((void**)&b.m1, n * 4, cudaHostAllocPortable), "host alloc");
            check(cudaHostAlloc((void**)&b.m2, n * 4, cudaHostAllocPortable), "host alloc");
            check(cudaHostAlloc((void**)&b.host_bf16, n * 2, cudaHostAllocPortable), "host alloc");
            // the copies below fill [0, valid); zero the DP shard padding, and m / v, in parallel
            // (tens of GB of pinned host state at 10B-20B: single-threaded memsets took ~10 s)
            host_zero(b.master + valid, (n - valid) * 4);
            host_zero(b.host_bf16 + valid, (n - valid) * 2);
            host_zero(b.m1, n * 4);
            host_zero(b.m2, n * 4);
            check(launch_cast_f32_bf16(tmp, tmpb, mp, st), "cast");
            if (valid) {
                check(cudaMemcpyAsync(b.master, tmp + off, valid * 4, cudaMemcpyDeviceToHost, st), "copy");
                check(cudaMemcpyAsync(b.host_bf16, tmpb + off, valid * 2, cudaMemcpyDeviceToHost, st), "copy");
            }
            check(cudaStreamSynchronize(st), "sync");
        } else {
            dalloc((void**)&b.master, n * 4);
            dalloc((void**)&b.m1, n * 4);
            dalloc((void**)&b.m2, n * 4);
            check(cudaMemsetAsync(b.master, 0, n * 4, st), "memset");
            if (valid) check(cudaMemcpyAsync(b.master, tmp + off, valid * 4, cudaMemcpyDeviceToDevice, st), "copy");
            check(cudaMemsetAsync(b.m1, 0, n * 4, st), "memset");
            check(cudaMemsetAsync(b.m2, 0, n * 4, st), "memset");
        }
    }
    check(cudaMemsetAsync(loss_dev_, 0, 256, st), "memset");
    check(cudaMemsetAsync(gstats_dev_, 0, (size_t)(d_.L + 1) * AH_STATS_FLOATS * 4, st), "memset");
    check(cudaStreamSynchronize(st), "sync");
    cudaFree(tmp);
    cudaFree(tmpb);
    // embedding / positions / final LN
    check(gpt::init_normal(wte_, (size_t)d_.V * h, seed_ * 31 + 5, 0.f, 0.02f, st), "init");
    check(gpt::fill_f32(wte_ + (size_t)d_.V * h, (size_t)(d_.Vp - d_.V) * h, 0.f, st), "init");
    check(gpt::init_normal(wpe_, nwpe, seed_ * 31 + 6, 0.f, 0.01f, st), "init");
    check(gpt::fill_f32(lnf_, h, 1.f, st), "init");
    check(gpt::fill_f32(lnf_ + h, h, 0.f, st), "init");
    for (float* p : {wte_m_, wte_v_}) check(cudaMemsetAsync(p, 0, nwte * 4, st), "memset");
    for (float* p : {wpe_m_, wpe_v_}) check(cudaMemsetAsync(p, 0, nwpe * 4, st), "memset");
    for (float* p : {lnf_m_, lnf_v_}) check(cudaMemsetAsync(p, 0, 2 * h * 4, st), "memset");
    check(launch_cast_f32_bf16(wte_, wte_b_, nwte, st), "cast");
    check(launch_cast_f32_bf16(wpe_, wpe_b_, nwpe, st), "cast");
    check(launch_cast_f32_bf16(lnf_, lnf_b_, 2 * h, st), "cast");
    check(cudaStreamSynchronize(st), "sync");
    static_bytes_ = stat;
    // Activation arena: the L - c_hat + 1 activation sets Eq.(1) counts (2 m_a (L - c_hat + 1)),
    // allocated once. Activations are the largest transient buffers; taking them from the
    // stream-ordered pool let cudaMallocAsync block the compute lane thread for up to ~2 s while
    // the pool waited on frees pending on the copy streams (measured inside the 10B step).
    // Slots are taken and returned on the compute stream only, so stream order makes reuse safe;
    // the memory timeline still counts a slot from its op's start to its release.
    {
        const size_t sets = (size_t)std::max(1, d_.L - strategy_.c_hat + 1);
        acts_slot_ = round_up(BlockActs::bytes(d_), 4096);
        check(cudaMalloc(&acts_arena_, sets * acts_slot_), "activation arena");
        for (size_t k = sets; k-- > 0;) acts_free_.push_back(static_cast<char*>(acts_arena_) + k * acts_slot_);
    }
    // Weight / gradient buffers (materialised, prefetched, gathered bf16 block vectors) come from a
    // fixed set of slots: Eq.(1)'s L - p_hat + 1 resident block buffers plus the prefetch lookahead
    // and two in-flight gradients (at least the simulated transient peak). They are taken and
    // released on different streams (compute, side, H2D; compute, D2H), so a release records an
    // event on its stream and the next taker's stream waits on it (GPU-side; the host never
    // blocks). The stream-ordered pool did the same reuse with host-blocking allocations and grew
    // by up to 10 GiB inside the timed region at 10B. Should every slot be live, one more is added
    // with cudaMalloc (warm-up only in practice; counted in stats.buffer_overflows).
    {
        const int64_t arena = (int64_t)(acts_free_.size() * acts_slot_);
        const int64_t transient = std::max<int64_t>(0, sim_.peak_gpu - (int64_t)static_bytes_ - arena);
        wslot_bytes_ = round_up(full_len() * 2, 4096);
        int la = 1;
        for (int x : strategy_.prefetch_lookahead) la = std::max(la, x);
        const size_t by_sim = (size_t)((transient + (int64_t)wslot_bytes_ - 1) / (int64_t)wslot_bytes_);
        const size_t by_eq1 = (size_t)std::max(0, d_.L - strategy_.p_hat + 1) + (size_t)la + 2;
        // within the GPU budget (the rest, if the schedule ever needs it, is added in warm-up)
        const int64_t room = hw_.gpu_mem - (int64_t)static_bytes_ - arena;
        const size_t cap = room > 0 ? (size_t)(room / (int64_t)wslot_bytes_) : 0;
        size_t n = std::min(by_eq1, std::max(by_sim, cap));
        if (const char* e = std::getenv("AH_BUFFER_SLOTS")) n = (size_t)std::max(1, std::atoi(e));  // tests
        for (size_t k = 0; k < n; ++k) wslot_add();
    }
}


uint16_t* Trainer::wslot_alloc(cudaStream_t st) {
    std::lock_guard<std::mutex> lk(wslot_mu_);
    if (wslot_free_.empty()) {  // every slot live: one more (cudaMalloc synchronises the device)
        wslot_add();
        ++wslot_overflow_;
    }
    const int k = wslot_free_.front();  // the longest-released slot
    wslot_free_.pop_front();
    if (wslot_recorded_[(size_t)k]) check(cudaStreamWaitEvent(st, wslot_ev_[(size_t)k], 0), "slot reuse wait");
    return wslot_ptr_[(size_t)k];
}

void Trainer::wslot_add() {
    void* p = nullptr;
    check(cudaMalloc(&p, wslot_bytes_), "block buffer slot");
    cudaEvent_t e = nullptr;
    check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    wslot_index_[p] = (int)wslot_ptr_.size();
    wslot_ptr_.push_back(static_cast<uint16_t*>(p));
    wslot_ev_.push_back(e);
    wslot_recorded_.push_back(0);
    wslot_free_.push_back((int)wslot_ptr_.size() - 1);
}

void Trainer::wslot_free(uint16_t* p, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(wslot_mu_);
    const auto f = wslot_index_.find(p);
    if (f == wslot_index_.end()) throw std::logic_error("executor: release of an unknown block buffer");
    const int k = f->second;
    check(cudaEventRecord(wslot_ev_[(size_t)k], st), "slot release");
    wslot_recorded_[(size_t)k] = 1;
    wslot_free_.push_back(k);
}

// ---------------------------------------------------------------------------------------
// Iteration construction: the reference op DAG + executor-only physical dependencies.
// ---------------------------------------------------------------------------------------
void Trainer::build_iteration(Iter& it) {
    const int ksim = it.k <= 1 ? 1 : 2;
    const std::vector<hetsim::StreamOp> ops = hetsim::build_iteration_ops(profile_, strategy_, ksim);
    for (const hetsim::StreamOp& so : ops) {
        RtOp r;
        r.kind = so.kind;
        r.block = so.block;
        r.bwd = so.backward_copy;
        r.iter = it.k;
        r.lane = lane_of(so.kind);
        for (const hetsim::OpRef& d : so.deps)
            r.deps.push_back({it.k - (ksim - d.iter), OpKey{(int)d.kind, d.block, d.backward_copy}});
        for (const hetsim::OpRef& g : so.start_after_start_of)
            r.gates.push_back({it.k, OpKey{(int)g.kind, g.block, g.backward_copy}});
        // Physical requirement not in the timing model: a recompute needs the block's bf16
        // weights, which for P-blocks arrive with the backward prefetch.
        if (so.kind == OpKind::Recompute && so.block <= strategy_.p_hat)
            r.deps.push_back({it.k, OpKey{(int)OpKind::ParamPrefetch, so.block, true}});
        if (nsub_ > 1 && so.kind == OpKind::ParamPrefetch && !so.backward_copy)
            for (const auto& d : r.deps)
                if (d.second.kind == (int)OpKind::CpuOptim && d.second.block == so.block) {
                    r.streamed = true;
                    r.stream_src = d;
                    r.ct.assign(2 * (size_t)nsub_, nullptr);
                    for (cudaEvent_t& e : r.ct) check(cudaEventCreate(&e), "event");
                }
        check(cudaEventCreateWithFlags(&r.done_ev, cudaEventDisableTiming), "event");
        check(cudaEventCreateWithFlags(&r.start_ev, cudaEventDisableTiming), "event");
        // GPU lanes: timing events on the op's stream; CPU lane: on the idle marker stream, where a
        // record completes at once, so the host AdamW ops land on the same timeline (trace)
        check(cudaEventCreate(&r.t0), "event");
        check(cudaEventCreate(&r.t1), "event");
        it.ops.emplace(OpKey{(int)so.kind, so.block, so.backward_copy}, std::move(r));
    }
    for (int l = 0; l < 4; ++l) it.lane_order[l] = order_[ksim - 1][l];
}

Trainer::RtOp* Trainer::find(long long iter, const OpKey& key) {
    for (Iter* it : iters_)
        if (it->k == iter) {
            auto f = it->ops.find(key);
            return f == it->ops.end() ? nullptr : &f->second;
        }
    return nullptr;
}

void Trainer::wait_dep(int lane, long long iter, const OpKey& key, bool gate, bool needs_side, int state_only) {
    if (iter < 1) return;
    cudaEvent_t ev = nullptr;
    int dep_lane = 0;
    bool on_side = false;
    {
        std::unique_lock<std::mutex> lk(mu_);
        RtOp* d = find(iter, key);
        if (!d) return;  // retired => long complete
        dep_lane = d->lane;
        const int need = state_only > 0 ? state_only : gate ? 1 : (d->lane == kCpu ? 3 : 2);
        cv_.wait(lk, [&] { return d->state >= need || stop_; });
        if (stop_ || state_only > 0) return;
        if (d->lane == kCpu) return;  // host ordering already established
        ev = gate ? d->start_ev : d->done_ev;
        on_side = d->done_on_side;
    }
    // same in-order stream, unless the consumer needs the dependency's side-stream tail
    // (GpuOptim reads the reduce-scattered gradient of its backward)
    if (dep_lane == lane && !gate && !(needs_side && on_side)) return;
    if (lane == kCpu)
        check(cudaEventSynchronize(ev), "event sync");
    else
        check(cudaStreamWaitEvent(stream_of(lane), ev, 0), "stream wait");
}

void Trainer::lane_main(int lane) {
    try {
        // A new host thread starts on device 0: bind it to this trainer's device (one rank per
        // GPU under DP), or its launches / stream-ordered allocations would target GPU 0.
        check(cudaSetDevice(device_), "lane set device");
        long long next = 1;
        while (true) {
            Iter* it = nullptr;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || submitted_ >= next; });
                if (stop_) return;
                for (Iter* x : iters_)
                    if (x->k == next) it = x;
            }
            if (!it) throw std::logic_error("executor: iteration window lost");
            for (size_t idx = 0; idx < it->lane_order[lane].size(); ++idx) {
                const OpKey& key = it->lane_order[lane][idx];
                RtOp& op = it->ops.at(key);
                const bool needs_side = op.kind == OpKind::GpuOptim;
                for (const auto& dp : op.deps) {
                    // sub-block streaming: CpuOptim follows its GradOffload chunk by chunk (the
                    // copies are issued), a forward prefetch follows the previous iteration's
                    // CpuOptim chunk by chunk (it started)
                    int state_only = 0;
                    if (nsub_ > 1 && op.kind == OpKind::CpuOptim && dp.second.kind == (int)OpKind::GradOffload)
                        state_only = 2;
                    if (op.streamed && dp.second.kind == (int)OpKind::CpuOptim) state_only = 1;
                    wait_dep(lane, dp.first, dp.second, false, needs_side, state_only);
                }
                for (const auto& gt : op.gates) wait_dep(lane, gt.first, gt.second, true);
                if (lane == kCpu) {
                    {
                        std::lock_guard<std::mutex> lk(mu_);
                        op.state = 1;
                    }
                    cv_.notify_all();
                    check(cudaEventRecord(op.t0, s_mark_), "record");
                    run_cpu(*it, op);
                    check(cudaEventRecord(op.t1, s_mark_), "record");
                    {
                        std::lock_guard<std::mutex> lk(mu_);
                        op.state = 3;
                        lane_stats_[lane].busy_ms += op.host_ms;
                        lane_stats_[lane].ops += 1;
                    }
                    cv_.notify_all();
                    continue;
                }
                cudaStream_t st = stream_of(lane);
                check(cudaEventRecord(op.start_ev, st), "record");
                check(cudaEventRecord(op.t0, st), "record");
                {
                    std::lock_guard<std::mutex> lk(mu_);
                    op.state = 1;
                }
                cv_.notify_all();
                if (lane == kCompute) {
                    const auto h0 = Clock::now();
                    prefetch_weights(*it, idx, op);  // the next op's weights, overlapping this op
                    run_compute(*it, op);
                    const double hm = std::chrono::duration<double, std::milli>(Clock::now() - h0).count();
                    std::lock_guard<std::mutex> lk(mu_);
                    enqueue_ms_ += hm;
                    enqueue_max_ms_ = std::max(enqueue_max_ms_, hm);
                }
                else if (lane == kH2D)
                    run_h2d(*it, op);
                else
                    run_d2h(*it, op);
                check(cudaEventRecord(op.t1, st), "record");
                check(cudaEventRecord(op.done_ev, op.done_on_side ? s_side_ : st), "record");
                {
                    std::lock_guard<std::mutex> lk(mu_);
                    op.state = 2;
                }
                cv_.notify_all();
            }
            {
                std::lock_guard<std::mutex> lk(mu_);
                it->finished_lanes += 1;
                if (it->finished_lanes == 4) completed_ = std::max(completed_, it->k);
            }
            cv_.notify_all();
            ++next;
        }
    } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(mu_);
        if (error_.empty()) error_ = std::string("lane ") + std::to_string(lane) + ": " + e.what();
        stop_ = true;
        cv_.notify_all();
    }
}

// ---------------------------------------------------------------------------------------
// Lane work
// ---------------------------------------------------------------------------------------
void Trainer::upload_inputs(Iter& it) {
    const size_t T = d_.T();
    const int slot = (int)(it.k & 1);
    int32_t* dtok = tok_dev_ + slot * inv_words_;
    int32_t* dtgt = dtok + T;
    if (it.on_device) {
        check(cudaMemcpyAsync(dtok, it.tokens, T * 4, cudaMemcpyDeviceToDevice, s_compute_), "tokens");
        check(cudaMemcpyAsync(dtgt, it.targets, T * 4, cudaMemcpyDeviceToDevice, s_compute_), "targets");
        // device inputs were not seen by the host check in submit(): ids outside [0, V) are
        // replaced by 0 (no out-of-bounds embedding / logits access) and reported by drain()
        int* flag = reinterpret_cast<int*>(loss_dev_ + 1);
        check(gpt::sanitize_ids(dtok, 2 * (int)T, d_.V, flag, s_compute_), "sanitize ids");
    } else {
        check(cudaMemcpyAsync(dtok, it.tokens, T * 4, cudaMemcpyHostToDevice, s_compute_), "tokens");
        check(cudaMemcpyAsync(dtgt, it.targets, T * 4, cudaMemcpyHostToDevice, s_compute_), "targets");
    }
    int32_t* uniq = dtgt + T;
    int32_t* offs = uniq + T;
    int32_t* pos = offs + T + 1;
    int32_t* nuniq = pos + T;
    check(gpt::token_index(dtok, (int)T, uniq, offs, pos, nuniq, s_compute_), "token index");
}

void Trainer::embed_forward(Iter& it) {
    upload_inputs(it);
    const int32_t* dtok = tok_dev_ + (it.k & 1) * inv_words_;
    check(gpt::embed_fwd(dtok, wte_b_, wpe_b_, x_[0], d_.T(), d_.s, d_.h, s_compute_), "embed");
}

void Trainer::head_forward_backward(Iter& it) {
    const int T = d_.T(), h = d_.h;
    const int32_t* dtgt = tok_dev_ + (it.k & 1) * inv_words_ + T;
    cudaStream_t st = s_compute_;
    check(gpt::ln_fwd(x_[(size_t)d_.L], lnf_b_, lnf_b_ + h, xf_, meanf_, rstdf_, T, h, st), "lnf");
    gemm::GemmArgs g;
    g.M = T; g.N = d_.Vp; g.K = h;
    g.A = xf_; g.lda = h; g.B = wte_b_; g.ldb = h; g.C = logits_; g.ldc = d_.Vp;
    check(gemm::run(g, st), "logits");
    check(gpt::cross_entropy(logits_, dtgt, losses_, T, d_.V, d_.Vp, 1.f / T, st), "ce");
    check(gpt::mean_loss(losses_, T, loss_dev_, st), "loss");
    check(cudaMemcpyAsync(loss_host_, loss_dev_, 8, cudaMemcpyDeviceToHost, st), "loss d2h");  // loss + id flag
    gemm::GemmArgs dg;  // dxf = dlogits . wte
    dg.M = T; dg.N = h; dg.K = d_.Vp;
    dg.A = logits_; dg.lda = d_.Vp; dg.B = wte_b_; dg.b_mn_major = 1; dg.ldb = h; dg.C = ws_.dln; dg.ldc = h;
    check(gemm::run(dg, st), "head dgrad");
    gemm::GemmArgs wg;  // dwte (fp32) = dlogits^T . xf
    wg.M = d_.Vp; wg.N = h; wg.K = T;
    wg.A = logits_; wg.a_mn_major = 1; wg.lda = d_.Vp; wg.B = xf_; wg.b_mn_major = 1; wg.ldb = h;
    wg.C = dwte_; wg.c_f32 = 1; wg.ldc = h;
    check(gemm::run(wg, st), "head wgrad");
    check(gpt::ln_bwd2(ws_.dln, x_[(size_t)d_.L], meanf_, rstdf_, lnf_b_, nullptr, gx_[d_.L & 1], dlnf_b_, ws_.part,
                      T, h, st),
          "lnf bwd");
}

void Trainer::embed_backward_and_update(Iter& it) {
    const int T = d_.T(), h = d_.h;
    cudaStream_t st = s_compute_;
    int32_t* base = tok_dev_ + (it.k & 1) * inv_words_;
    int32_t* uniq = base + 2 * T;
    int32_t* offs = uniq + T;
    int32_t* pos = offs + T + 1;
    int32_t* nuniq = pos + T;
    const uint16_t* dx0 = gx_[0];
    check(gpt::embed_bwd_tok_dev(dx0, uniq, offs, pos, nuniq, T, dwte_, h, st), "embed bwd");
    check(gpt::embed_bwd_pos(dx0, dwpe_, d_.B, d_.s, h, st), "pos bwd");
    const size_t nwte = (size_t)d_.Vp * h, nwpe = (size_t)d_.s * h;
    if (dp_) {  // replicated embedding / positions / final LN: sum gradients over ranks
        side_after_compute();
        dp_allreduce_f32(dwte_, nwte, s_side_);
        dp_allreduce_f32(dwpe_, nwpe, s_side_);
        dp_allreduce_bf16(dlnf_b_, 2 * (size_t)h, s_side_);
        compute_after_side();
    }
    check(gpt::f32_to_bf16(dwte_, dwte_b_, nwte, st), "cvt");
    check(gpt::f32_to_bf16(dwpe_, dwpe_b_, nwpe, st), "cvt");
    const int step = (step_base_ + (int)it.k);
    const float inv = 1.f / (float)dp_size_;
    // overflow check of the replicated group (slot 0): one skip flag for all three updates
    grad_stats_pass(0, dwte_b_, nwte, st);
    check(launch_grad_stats(dwpe_b_, nwpe, inv, gstats(0), st), "grad stats");
    check(launch_grad_stats(dlnf_b_, 2 * (size_t)h, inv, gstats(0), st), "grad stats");
    AdamArgs a1 = adam_args(adam_, step, wte_, wte_m_, wte_v_, dwte_b_, wte_b_, nwte);
    AdamArgs a2 = adam_args(adam_, step, wpe_, wpe_m_, wpe_v_, dwpe_b_, wpe_b_, nwpe);
    AdamArgs a3 = adam_args(adam_, step, lnf_, lnf_m_, lnf_v_, dlnf_b_, lnf_b_, 2 * (size_t)h);
    a1.inv_scale = a2.inv_scale = a3.inv_scale = inv;
    a1.skip = a2.skip = a3.skip = reinterpret_cast<const int*>(gstats(0) + 1);
    check(launch_adam(a1, st), "adam wte");
    check(launch_adam(a2, st), "adam wpe");
    check(launch_adam(a3, st), "adam lnf");
}

void Trainer::run_compute(Iter& it, RtOp& op) {
    const int i = op.block;
    BlockState& b = blocks_[(size_t)i];
    cudaStream_t st = s_compute_;
    const size_t mp = d_.m_p();
    const size_t off = shard_ * (size_t)dp_rank_;
    auto materialize = [&]() {  // bf16 weights from the on-GPU fp32 master (footnote 2)
        b.wbuf = wslot_alloc(st);
        op.alloc_b += (int64_t)full_len() * 2;
        if (dp_) {  // own shard, then all-gather the others over NVLink (side stream)
            check(launch_cast_f32_bf16(b.master, b.wbuf + off, shard_, st), "cast");
            side_after_compute();
            dp_gather(b.wbuf, s_side_);
            compute_after_side();
        } else {
            check(launch_cast_f32_bf16(b.master, b.wbuf, mp, st), "cast");
        }
    };
    if (b.mat_pending) {  // materialised ahead on the side stream (prefetch_weights)
        check(cudaStreamWaitEvent(st, b.mat_ev, 0), "wait materialised weights");
        b.mat_pending = false;
    }
    if (b.needs_gather && op.kind != OpKind::GpuOptim) {  // prefetched shard -> full weights
        side_after_compute();
        dp_gather(b.wbuf, s_side_);
        compute_after_side();
        b.needs_gather = false;
    }
    auto alloc_acts = [&]() {  // a slot of the activation arena (allocated and freed on this stream only)
        if (acts_free_.empty()) throw std::logic_error("executor: more live activation sets than L - c_hat + 1");
        b.acts = acts_free_.back();
        acts_free_.pop_back();
        op.alloc_b += (int64_t)BlockActs::bytes(d_);
    };
    auto free_acts = [&]() {
        acts_free_.push_back(b.acts);
        b.acts = nullptr;
        op.free_b += (int64_t)BlockActs::bytes(d_);
    };
    auto free_wbuf = [&]() {
        wslot_free(b.wbuf, st);
        b.wbuf = nullptr;
        op.free_b += (int64_t)full_len() * 2;
    };
    switch (op.kind) {
        case OpKind::Forward: {
            if (i == 1) embed_forward(it);
            if (!b.o && !b.wbuf) materialize();
            if (!b.wbuf) throw std::logic_error("forward without resident weights");
            alloc_acts();
            const BlockActs a = BlockActs::carve(d_, b.acts);
            check(block_forward(d_, b.wbuf, x_[(size_t)i - 1], x_[(size_t)i], a, ws_, st), "block fwd");
            if (i == d_.L) head_forward_backward(it);
            if (b.c) free_acts();
            // P blocks re-fetch their weights for the backward; every other block keeps its bf16
            // weights live from F to R / B, as Eq. 1 models them (2 m_p (L - p_hat + 1) resident,
            // costmodel.cpp:36-41): no second cast from the master (and, under DP, no second
            // all-gather) per iteration
            if (b.p) free_wbuf();
            break;
        }
        case OpKind::Recompute: {
            if (!b.wbuf) materialize();  // plain C-block: B's materialisation moves up to R
            alloc_acts();
            const BlockActs a = BlockActs::carve(d_, b.acts);
            check(block_forward(d_, b.wbuf, x_[(size_t)i - 1], nullptr, a, ws_, st), "recompute");
            break;
        }
        case OpKind::Backward: {
            if (!b.wbuf) materialize();
            const BlockActs a = BlockActs::carve(d_, b.acts);
            check(block_backward(d_, b.wbuf, x_[(size_t)i - 1], a, gx_[i & 1], gx_[(i - 1) & 1], ws_, st),
                  "block bwd");
            free_acts();
            if (dp_) {  // full local grads -> this rank's reduced shard (in place), on the side
                // stream: the next block's backward overlaps it; GpuOptim / GradOffload wait on
                // this op's done_ev, which is recorded behind the reduce-scatter
                side_after_compute();
                if (full_len() > mp) check(cudaMemsetAsync(b.wbuf + mp, 0, (full_len() - mp) * 2, s_side_), "pad");
                dp_reduce_grads(b.wbuf, s_side_);
                grad_stats_pass(i, b.wbuf + off, shard_, s_side_);  // the reduced shard this rank updates
                op.done_on_side = true;
            } else {
                grad_stats_pass(i, b.wbuf, mp, st);
            }
            if (i == 1) embed_backward_and_update(it);
            break;
        }
        case OpKind::GpuOptim: {
            AdamArgs aa = dp_ ? adam_args(adam_, (step_base_ + (int)it.k), b.master, b.m1, b.m2, b.wbuf + off, nullptr, shard_)
                              : adam_args(adam_, (step_base_ + (int)it.k), b.master, b.m1, b.m2, b.wbuf, nullptr, mp);
            aa.inv_scale = 1.f / (float)dp_size_;
            aa.skip = reinterpret_cast<const int*>(gstats(i) + 1);  // no-op if a grad of block i is inf / nan
            check(launch_adam(aa, st), "adam");
            free_wbuf();
            break;
        }
        default:
            throw std::logic_error("compute lane got a non-compute op");
    }
}

void Trainer::run_h2d(Iter& it, RtOp& op) {
    (void)it;
    BlockState& b = blocks_[(size_t)op.block];
    const size_t mp = d_.m_p();
    const size_t n = dp_ ? shard_ : mp;  // DP: only this rank's shard crosses the host link
    uint16_t* dst = nullptr;
    dst = wslot_alloc(s_h2d_);
    op.alloc_b += (int64_t)full_len() * 2;
    uint16_t* mine = dp_ ? dst + shard_ * (size_t)dp_rank_ : dst;
    if (b.o && op.streamed) {  // chunk c goes up as soon as the host AdamW finished it
        for (int c = 0; c < nsub_; ++c) {
            size_t a = 0, len = 0;
            sub_range(c, n, a, len);
            wait_progress(op.stream_src.first, op.stream_src.second, c + 1);
            check(cudaEventRecord(op.ct[2 * (size_t)c], s_h2d_), "record");
            check(cudaMemcpyAsync(mine + a, b.host_bf16 + a, len * 2, cudaMemcpyHostToDevice, s_h2d_), "prefetch");
            check(cudaEventRecord(op.ct[2 * (size_t)c + 1], s_h2d_), "record");
        }
    } else if (b.o)
        check(cudaMemcpyAsync(mine, b.host_bf16, n * 2, cudaMemcpyHostToDevice, s_h2d_), "prefetch");
    else  // P\O backward prefetch: the fp32 master is on the GPU; materialise without PCIe
        check(launch_cast_f32_bf16(b.master, mine, n, s_h2d_), "prefetch cast");
    std::lock_guard<std::mutex> lk(mu_);
    b.wbuf = dst;
    b.needs_gather = dp_;  // the compute lane all-gathers before first use (deterministic order)
}

void Trainer::run_d2h(Iter& it, RtOp& op) {
    (void)it;
    BlockState& b = blocks_[(size_t)op.block];
    const size_t n = dp_ ? shard_ : d_.m_p();
    const uint16_t* src = dp_ ? b.wbuf + shard_ * (size_t)dp_rank_ : b.wbuf;
    // the block's overflow check rides along (first, so it has landed with chunk 0)
    check(cudaMemcpyAsync(gstats_host_ + 2 * op.block, gstats(op.block), 8, cudaMemcpyDeviceToHost, s_d2h_),
          "offload stats");
    if (nsub_ > 1) {
        for (int c = 0; c < nsub_; ++c) {
            size_t a = 0, len = 0;
            sub_range(c, n, a, len);
            check(cudaMemcpyAsync(b.host_bf16 + a, src + a, len * 2, cudaMemcpyDeviceToHost, s_d2h_), "offload");
            check(cudaEventRecord(b.go_ev[(size_t)c], s_d2h_), "record");
        }
    } else {
        check(cudaMemcpyAsync(b.host_bf16, src, n * 2, cudaMemcpyDeviceToHost, s_d2h_), "offload");
    }
    wslot_free(b.wbuf, s_d2h_);
    b.wbuf = nullptr;
    op.free_b += (int64_t)full_len() * 2;
}

void Trainer::run_cpu(Iter& it, RtOp& op) {
    BlockState& b = blocks_[(size_t)op.block];
    ah_adam_hparams hp = adam_;
    hp.step = (step_base_ + (int)it.k);
    const size_t n = dp_ ? shard_ : d_.m_p();
    double busy = 0.0;  // host AdamW time only (not the waits for gradient chunks)
    uint32_t bad = 0;
    for (int c = 0; c < nsub_; ++c) {
        size_t a = 0, len = 0;
        sub_range(c, n, a, len);
        if (nsub_ > 1) check(cudaEventSynchronize(b.go_ev[(size_t)c]), "offload chunk sync");
        if (c == 0) std::memcpy(&bad, gstats_host_ + 2 * op.block + 1, 4);
        const auto t0 = Clock::now();
        if (bad == 0) {
            cpu_adam(hp, b.master + a, b.m1 + a, b.m2 + a, b.host_bf16 + a, b.host_bf16 + a, len,
                     1.f / (float)dp_size_, cpu_threads_);
        } else {  // overflow skip: state untouched; the shared buffer holds grads -> restore bf16(master)
            cpu_cast_f32_bf16(b.master + a, b.host_bf16 + a, len, cpu_threads_);
        }
        busy += std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
        if (nsub_ > 1) {
            {
                std::lock_guard<std::mutex> lk(mu_);
                op.progress = c + 1;
            }
            cv_.notify_all();
        }
    }
    op.host_ms = busy;
}

// Chunk c of nsub_ over n elements, boundaries on 16384-element (64 KiB fp32) multiples.
void Trainer::sub_range(int c, size_t n, size_t& a, size_t& len) const {
    if (nsub_ <= 1) {
        a = 0;
        len = n;
        return;
    }
    const size_t q = 16384;
    const size_t per = round_up((n + (size_t)nsub_ - 1) / (size_t)nsub_, q);
    a = std::min(n, per * (size_t)c);
    len = std::min(n, a + per) - a;
}

void Trainer::wait_progress(long long iter, const OpKey& key, int chunks) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] {
        if (stop_) return true;
        const RtOp* d = find(iter, key);
        return !d || d->state >= 3 || d->progress >= chunks;  // retired => complete
    });
}

double Trainer::op_ms(const RtOp& o) const {
    float x = 0.f;
    if (o.ct.empty()) return cudaEventElapsedTime(&x, o.t0, o.t1) == cudaSuccess ? x : -1.0;
    double sum = 0.0;
    for (size_t c = 0; c + 1 < o.ct.size(); c += 2) {
        if (cudaEventElapsedTime(&x, o.ct[c], o.ct[c + 1]) != cudaSuccess) return -1.0;
        sum += x;
    }
    return sum;
}

float* Trainer::gstats(int slot) const { return gstats_dev_ + (size_t)slot * AH_STATS_FLOATS; }

// Zero the slot's accumulators and run the overflow / norm pre-pass (2 B/param read) on the
// group's gradients; the slot's non-finite count then gates the group's update.
void Trainer::grad_stats_pass(int slot, const uint16_t* g, size_t n, cudaStream_t st) {
    check(cudaMemsetAsync(gstats(slot), 0, 8, st), "stats reset");
    check(launch_grad_stats(g, n, 1.f / (float)dp_size_, gstats(slot), st), "grad stats");
}

// After a drain: norm / non-finite count / skipped groups of the last iteration (fixed slot
// order; this rank's gradients — under DP its reduced shards plus the replicated group).
void Trainer::collect_grad_stats() {
    std::vector<float> h((size_t)(d_.L + 1) * 2);
    check(cudaMemcpy2D(h.data(), 8, gstats_dev_, AH_STATS_FLOATS * 4, 8, (size_t)(d_.L + 1), cudaMemcpyDeviceToHost),
          "grad stats d2h");
    double ss = 0.0;
    long long bad = 0;
    int skipped = 0;
    for (int i = 0; i <= d_.L; ++i) {
        uint32_t nb = 0;
        std::memcpy(&nb, &h[(size_t)i * 2 + 1], 4);
        ss += (double)h[(size_t)i * 2];
        bad += nb;
        skipped += nb ? 1 : 0;
    }
    grad_norm_ = std::sqrt(ss);
    nonfinite_ = bad;
    skipped_ = skipped;
}

void Trainer::side_after_compute() {
    check(cudaEventRecord(ev_c2s_, s_compute_), "record");
    check(cudaStreamWaitEvent(s_side_, ev_c2s_, 0), "side wait");
}

void Trainer::compute_after_side() {
    check(cudaEventRecord(ev_s2c_, s_side_), "record");
    check(cudaStreamWaitEvent(s_compute_, ev_s2c_, 0), "compute wait");
}

// If the compute op after lane_order[idx] will materialise a GPU-resident block's bf16 weights
// (F, R or B of a non-O, non-P block whose buffer is not live), do it now on the side stream —
// cast from the fp32 master (+ DP all-gather) — so it overlaps op idx instead of preceding the
// next op on the compute stream. Only the compute lane thread touches these blocks' buffers.
void Trainer::prefetch_weights(const Iter& it, size_t idx, RtOp& cur) {
    const std::vector<OpKey>& order = it.lane_order[kCompute];
    if (idx + 1 >= order.size()) return;
    const OpKey& x = order[idx];
    const OpKey& y = order[idx + 1];
    const bool uses_weights = y.kind == (int)OpKind::Forward || y.kind == (int)OpKind::Recompute ||
                              y.kind == (int)OpKind::Backward;
    if (!uses_weights || y.block == x.block || y.block < 1 || y.block > d_.L) return;
    BlockState& b = blocks_[(size_t)y.block];
    if (b.o || b.p || b.wbuf || b.mat_pending) return;
    side_after_compute();  // the master is final: every compute op enqueued so far precedes the cast
    b.wbuf = wslot_alloc(s_side_);
    cur.alloc_b += (int64_t)full_len() * 2;  // lives from the current op on
    if (dp_) {
        check(launch_cast_f32_bf16(b.master, b.wbuf + shard_ * (size_t)dp_rank_, shard_, s_side_), "cast");
        dp_gather(b.wbuf, s_side_);
    } else {
        check(launch_cast_f32_bf16(b.master, b.wbuf, d_.m_p(), s_side_), "cast");
    }
    if (!b.mat_ev) check(cudaEventCreateWithFlags(&b.mat_ev, cudaEventDisableTiming), "event");
    check(cudaEventRecord(b.mat_ev, s_side_), "record");
    b.mat_pending = true;
}

void Trainer::dp_gather(uint16_t* wbuf, cudaStream_t st) {
    if (loop_) return check(loop_->call(dp_rank_, LoopbackComm::kAllGatherBf16, wbuf, shard_, st), "loopback all-gather");
    const ncclResult_t r = ncclAllGather(wbuf + shard_ * (size_t)dp_rank_, wbuf, shard_, ncclBfloat16,
                                         static_cast<ncclComm_t>(comm_), st);
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclAllGather: ") + ncclGetErrorString(r));
}

void Trainer::dp_reduce_grads(uint16_t* wbuf, cudaStream_t st) {
    if (loop_)
        return check(loop_->call(dp_rank_, LoopbackComm::kReduceScatterBf16, wbuf, shard_, st), "loopback reduce-scatter");
    const ncclResult_t r = ncclReduceScatter(wbuf, wbuf + shard_ * (size_t)dp_rank_, shard_, ncclBfloat16, ncclSum,
                                             static_cast<ncclComm_t>(comm_), st);
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclReduceScatter: ") + ncclGetErrorString(r));
}

void Trainer::dp_allreduce_f32(float* p, size_t n, cudaStream_t st) {
    if (loop_) return check(loop_->call(dp_rank_, LoopbackComm::kAllReduceF32, p, n, st), "loopback all-reduce");
    const ncclResult_t r = ncclAllReduce(p, p, n, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm_), st);
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclAllReduce: ") + ncclGetErrorString(r));
}

void Trainer::dp_allreduce_bf16(uint16_t* p, size_t n, cudaStream_t st) {
    if (loop_) return check(loop_->call(dp_rank_, LoopbackComm::kAllReduceBf16, p, n, st), "loopback all-reduce");
    const ncclResult_t r = ncclAllReduce(p, p, n, ncclBfloat16, ncclSum, static_cast<ncclComm_t>(comm_), st);
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclAllReduce: ") + ncclGetErrorString(r));
}

// ---------------------------------------------------------------------------------------
// Public
// ---------------------------------------------------------------------------------------
void Trainer::submit(const int32_t* tokens, const int32_t* targets, bool on_device) {
    if (!on_device) {  // host ids index wte / dwte / the logits rows: reject any outside [0, V)
        const size_t T = d_.T();
        for (size_t t = 0; t < T; ++t)
            if (tokens[t] < 0 || tokens[t] >= d_.V || targets[t] < 0 || targets[t] >= d_.V)
                throw std::invalid_argument("trainer: token / target id outside [0, vocab) at position " +
                                            std::to_string(t));
    }
    Iter* it = new Iter;
    {
        std::lock_guard<std::mutex> lk(mu_);
        if (!error_.empty()) {
            delete it;
            throw std::runtime_error(error_);
        }
        it->k = submitted_ + 1;
    }
    it->on_device = on_device;
    if (on_device) {
        it->tokens = tokens;
        it->targets = targets;
    } else {  // stage into pinned memory so the H2D copy is truly asynchronous
        const size_t T = d_.T();
        int32_t* stage = tok_host_ + (it->k & 1) * 2 * T;
        // the previous user of this staging slot (iteration k-2) must have consumed it
        {
            std::unique_lock<std::mutex> lk(mu_);
            for (Iter* x : iters_)
                if (x->k == it->k - 2) {
                    RtOp* f1 = nullptr;
                    auto f = x->ops.find(OpKey{(int)OpKind::Forward, 1, false});
                    if (f != x->ops.end()) f1 = &f->second;
                    if (f1) {
                        cv_.wait(lk, [&] { return f1->state >= 2 || stop_; });
                        cudaEvent_t e = f1->done_ev;
                        lk.unlock();
                        check(cudaEventSynchronize(e), "staging reuse");
                        lk.lock();
                    }
                }
        }
        std::memcpy(stage, tokens, T * 4);
        std::memcpy(stage + T, targets, T * 4);
        it->tokens = stage;
        it->targets = stage + T;
    }
    build_iteration(*it);
    {
        std::lock_guard<std::mutex> lk(mu_);
        iters_.push_back(it);
        submitted_ = it->k;
        // retire iterations that no live op can reference any more
        while (iters_.size() > 4 && iters_.front()->k + 3 <= completed_) {
            Iter* old = iters_.front();
            retired_.push_back(old);
            iters_.pop_front();
        }
    }
    cv_.notify_all();
    for (Iter* old : retired_) {
        int64_t net = 0;
        for (auto& kv : old->ops) net += kv.second.alloc_b - kv.second.free_b;
        {
            std::lock_guard<std::mutex> lk(mu_);
            retired_bytes_ += net;
        }
        for (auto& kv : old->ops) {
            RtOp& o = kv.second;
            if (o.lane != kCpu && o.host_ms >= 0) {  // account GPU lane time before the events go
                double ms = -1.0;
                if (cudaEventSynchronize(o.t1) == cudaSuccess) ms = op_ms(o);
                if (ms >= 0) {
                    std::lock_guard<std::mutex> lk(mu_);
                    lane_stats_[o.lane].busy_ms += ms;
                    lane_stats_[o.lane].ops += 1;
                }
            }
            for (cudaEvent_t e : {o.done_ev, o.start_ev, o.t0, o.t1})
                if (e) cudaEventDestroy(e);
            for (cudaEvent_t e : o.ct) cudaEventDestroy(e);
        }
        delete old;
    }
    retired_.clear();
}

float Trainer::drain() {
    {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || completed_ >= submitted_; });
        if (!error_.empty()) throw std::runtime_error(error_);
    }
    check(cudaStreamSynchronize(s_compute_), "sync");
    check(cudaStreamSynchronize(s_h2d_), "sync");
    check(cudaStreamSynchronize(s_d2h_), "sync");
    check(cudaStreamSynchronize(s_side_), "sync");
    // accumulate GPU lane busy time of finished iterations
    {
        std::lock_guard<std::mutex> lk(mu_);
        for (Iter* it : iters_)
            for (auto& kv : it->ops) {
                RtOp& o = kv.second;
                if (o.lane == kCpu || o.host_ms < 0) continue;
                const double ms = op_ms(o);
                if (ms >= 0) {
                    lane_stats_[o.lane].busy_ms += ms;
                    lane_stats_[o.lane].ops += 1;
                }
                o.host_ms = -1.0;  // counted
            }
    }
    account_window();
    collect_grad_stats();
    last_loss_ = *loss_host_;
    int bad = 0;
    std::memcpy(&bad, loss_host_ + 1, 4);
    if (bad) {  // an on-device batch carried ids outside [0, V): they were trained as id 0
        check(cudaMemsetAsync(loss_dev_ + 1, 0, 4, s_compute_), "clear id flag");
        check(cudaStreamSynchronize(s_compute_), "sync");
        std::memset(loss_host_ + 1, 0, 4);
        throw std::invalid_argument("trainer: token / target id outside [0, vocab) in an on-device batch "
                                    "(replaced by 0 in that iteration)");
    }
    return last_loss_;
}

float Trainer::step(const int32_t* tokens, const int32_t* targets) {
    submit(tokens, targets, false);
    return drain();
}

size_t Trainer::master_size(int block) const {
    if (block >= 1 && block <= d_.L) return dp_ ? shard_ : d_.m_p();  // DP: this rank's shard
    if (block == 0) return (size_t)d_.Vp * d_.h;
    if (block == -1) return (size_t)d_.s * d_.h;
    if (block == -2) return 2 * (size_t)d_.h;
    return 0;
}

void Trainer::read_master(int block, float* out, size_t n) {
    const size_t want = master_size(block);
    if (want == 0 || n < want) throw std::invalid_argument("read_master: bad block or buffer too small");
    const float* src = nullptr;
    bool host = false;
    if (block >= 1) {
        src = blocks_[(size_t)block].master;
        host = blocks_[(size_t)block].o;
    } else {
        src = block == 0 ? wte_ : (block == -1 ? wpe_ : lnf_);
    }
    if (host)
        std::memcpy(out, src, want * 4);
    else
        check(cudaMemcpy(out, src, want * 4, cudaMemcpyDeviceToHost), "read master");
}

void Trainer::stats(ah_trainer_stats* s) {
    std::memset(s, 0, sizeof(*s));
    s->c_hat = strategy_.c_hat;
    s->p_hat = strategy_.p_hat;
    s->o_hat = strategy_.o_hat;
    s->activation_coef = (double)profile_.block.m_a / (double)profile_.block.m_a_in;
    s->m_p = profile_.block.m_p;
    s->m_gc = profile_.m_gc;
    s->modeled_peak_bytes = hetsim::dp::peak_gpu_mem(profile_, strategy_, dp_spec_);  // Eq.(1), per rank under DP
    s->simulated_peak_bytes = sim_.peak_gpu;
    uint64_t hw = 0;
    cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrUsedMemHigh, &hw);
    s->pool_peak_bytes = (int64_t)hw;
    uint64_t rsv = 0;
    cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrReservedMemCurrent, &rsv);
    s->pool_reserved_bytes = (int64_t)rsv;
    s->static_bytes = (int64_t)static_bytes_;
    s->sim_steady_s = sim_.steady_state_time;
    std::lock_guard<std::mutex> lk(mu_);
    for (int l = 0; l < 4; ++l) {
        s->lane_busy_ms[l] = lane_stats_[l].busy_ms;
        s->lane_ops[l] = lane_stats_[l].ops;
    }
    s->compute_enqueue_ms = enqueue_ms_;
    {
        std::lock_guard<std::mutex> lk2(wslot_mu_);
        s->buffer_overflows = wslot_overflow_;
    }
    s->compute_enqueue_max_ms = enqueue_max_ms_;
    const int64_t per_block = dp_ ? (int64_t)shard_ : profile_.block.m_p;  // host-link elements
    // host-link bytes: every O block's forward prefetch, plus the backward re-fetch of the P blocks
    // that are also O (a P block outside O re-materialises from its GPU master, no PCIe)
    const int p_and_o = std::max(0, strategy_.p_hat + strategy_.o_hat - d_.L);
    s->h2d_bytes = 2 * per_block * (strategy_.o_hat + p_and_o);
    s->d2h_bytes = 2 * per_block * strategy_.o_hat;
    s->window_iters = win_iters_;
    s->compute_busy_ms = win_compute_ms_;
    s->h2d_busy_ms = win_h2d_ms_;
    s->d2h_busy_ms = win_d2h_ms_;
    s->offload_blocked_ms = win_blocked_ms_;
    s->h2d_gbps = win_h2d_link_ms_ > 0 ? win_h2d_bytes_ / (win_h2d_link_ms_ * 1e6) : 0.0;
    s->d2h_gbps = win_d2h_ms_ > 0 ? win_d2h_bytes_ / (win_d2h_ms_ * 1e6) : 0.0;
    s->copy_blocked_ms = win_copy_blocked_ms_;
    s->upstream_blocked_ms = win_upstream_blocked_ms_;
    s->cpu_busy_ms = win_cpu_ms_;
    s->window_ms = win_span_ms_;
    s->sim_steady_fifo_s = sim_steady_[0];
    s->sim_steady_ps_s = sim_steady_[1];
    s->priority_sched = ps_ ? 1 : 0;
    s->grad_norm = grad_norm_;
    s->nonfinite_grads = nonfinite_;
    s->skipped_updates = skipped_;
    for (int l = 0; l < 4; ++l) s->sim_lane_busy_ms[l] = sim_lane_ms_[l];
    s->stream_chunks = nsub_;
}

std::string Trainer::trace_json() {
    std::ostringstream out;
    std::vector<hetsim::CompletedOp> ops;
    std::lock_guard<std::mutex> lk(mu_);
    if (iters_.empty()) return "[]\n";
    // time origin: first op of the oldest iteration still in the window
    cudaEvent_t origin = nullptr;
    for (auto& kv : iters_.front()->ops)
        if (kv.second.lane == kCompute && kv.second.kind == OpKind::Forward && kv.second.block == 1)
            origin = kv.second.t0;
    for (Iter* it : iters_)
        for (auto& kv : it->ops) {
            RtOp& o = kv.second;
            if (!origin) continue;
            float a = 0, b = 0;
            if (cudaEventElapsedTime(&a, origin, o.t0) != cudaSuccess) continue;
            if (cudaEventElapsedTime(&b, origin, o.t1) != cudaSuccess) continue;
            ops.push_back({o.kind, o.block, (int)o.iter, o.bwd, hetsim::stream_of(o.kind), a / 1e3, b / 1e3});
        }
    std::sort(ops.begin(), ops.end(), [](const hetsim::CompletedOp& x, const hetsim::CompletedOp& y) {
        return x.start < y.start;
    });
    hetsim::write_chrome_trace(out, ops);
    return out.str();
}

std::string Trainer::memory_csv(int64_t* peak_bytes) {
    std::lock_guard<std::mutex> lk(mu_);
    std::vector<std::pair<double, int64_t>> ev;  // (time s, delta bytes)
    cudaEvent_t origin = nullptr;
    float first = 0.f;
    for (Iter* it : iters_)
        for (auto& kv : it->ops) {
            RtOp& o = kv.second;
            if (o.lane == kCpu || (!o.alloc_b && !o.free_b)) continue;
            if (!origin) origin = o.t0;
            float a = 0.f, b = 0.f;
            if (cudaEventElapsedTime(&a, origin, o.t0) != cudaSuccess) continue;
            if (cudaEventElapsedTime(&b, origin, o.t1) != cudaSuccess) continue;
            first = std::min(first, a);
            if (o.alloc_b) ev.push_back({a / 1e3, o.alloc_b});
            if (o.free_b) ev.push_back({b / 1e3, -o.free_b});
        }
    std::sort(ev.begin(), ev.end(), [](const auto& x, const auto& y) {
        return x.first != y.first ? x.first < y.first : x.second < y.second;  // frees first on ties
    });
    std::vector<std::pair<double, int64_t>> tl;
    int64_t cur = (int64_t)static_bytes_ + retired_bytes_, peak = cur;
    tl.push_back({0.0, cur});
    for (const auto& e : ev) {
        cur += e.second;
        peak = std::max(peak, cur);
        tl.push_back({e.first - first / 1e3, cur});
    }
    if (peak_bytes) *peak_bytes = peak;
    std::ostringstream out;
    hetsim::write_memory_csv(out, tl);
    return out.str();
}

}  // namespace ah

// ---------------------------------------------------------------------------------------
// Runtime profiler (paper §3.1): one block measured on this box.
// ---------------------------------------------------------------------------------------
namespace ah {

ah_hw_profile profile_block(const ah_trainer_config& cfg) {
    GptDims d;
    d.L = 1;
    d.h = cfg.hidden;
    d.nh = cfg.heads;
    d.hd = cfg.hidden / cfg.heads;
    d.s = cfg.seq_len;
    d.B = cfg.batch;
    d.V = cfg.vocab;
    d.Vp = (int)round_up((size_t)cfg.vocab, 256);
    const int L_model = cfg.num_blocks > 0 ? cfg.num_blocks : 1;
    const size_t mp = d.m_p(), T = d.T(), h = d.h;
    auto ok = [](cudaError_t e, const char* w) {
        if (e != cudaSuccess) throw std::runtime_error(std::string(w) + ": " + cudaGetErrorString(e));
    };
    cudaStream_t st;
    ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    std::vector<void*> dev;  // everything allocated here, freed at the end
    auto dmalloc = [&](size_t bytes) {
        void* p = nullptr;
        ok(cudaMalloc(&p, bytes), "profile alloc");
        dev.push_back(p);
        return p;
    };
    float* master = (float*)dmalloc(mp * 4);
    float* m1 = (float*)dmalloc(mp * 4);
    float* m2 = (float*)dmalloc(mp * 4);
    uint16_t* w = (uint16_t*)dmalloc(mp * 2);
    uint16_t *x0 = (uint16_t*)dmalloc(T * h * 2), *x1 = (uint16_t*)dmalloc(T * h * 2);
    uint16_t *gx0 = (uint16_t*)dmalloc(T * h * 2), *gx1 = (uint16_t*)dmalloc(T * h * 2);
    void* acts = dmalloc(BlockActs::bytes(d));
    void* wsm = dmalloc(Workspace::bytes(d));
    const Workspace ws = Workspace::carve(d, wsm);
    const BlockActs a = BlockActs::carve(d, acts);
    ok(gpt::init_normal(master, mp, 99, 0.f, 0.02f, st), "init");
    ok(cudaMemsetAsync(m1, 0, mp * 4, st), "memset");
    ok(cudaMemsetAsync(m2, 0, mp * 4, st), "memset");
    ok(launch_cast_f32_bf16(master, w, mp, st), "cast");
    ok(cudaMemsetAsync(x0, 0, T * h * 2, st), "memset");
    ok(cudaMemsetAsync(gx0, 0, T * h * 2, st), "memset");
    cudaEvent_t e0, e1;
    ok(cudaEventCreate(&e0), "event");
    ok(cudaEventCreate(&e1), "event");
    auto timed = [&](int reps, auto&& body) {
        body();  // warm-up
        ok(cudaStreamSynchronize(st), "sync");
        ok(cudaEventRecord(e0, st), "record");
        for (int r = 0; r < reps; ++r) body();
        ok(cudaEventRecord(e1, st), "record");
        ok(cudaEventSynchronize(e1), "sync");
        float ms = 0.f;
        ok(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
        return (double)ms / 1e3 / reps;
    };
    // the backward consumes the weight slots as gradient storage: re-materialise each rep
    auto fwd = [&] { ok(block_forward(d, w, x0, x1, a, ws, st), "fwd"); };
    auto cast = [&] { ok(launch_cast_f32_bf16(master, w, mp, st), "cast"); };
    auto bwd = [&] {
        cast();
        ok(block_backward(d, w, x0, a, gx0, gx1, ws, st), "bwd");
    };
    // sustained clock: >= 1 s of back-to-back forward + backward before anything is timed
    {
        const double one = timed(1, [&] { fwd(); bwd(); });
        const int n = (int)std::min(100000.0, std::ceil(1.0 / std::max(one, 1e-6)));
        (void)timed(n, [&] { fwd(); bwd(); });
    }
    ah_hw_profile out{};
    out.t_block_fwd_s = timed(10, fwd);
    out.t_block_bwd_s = timed(10, bwd) - timed(10, cast);

    // per-iteration work outside the blocks, on the real shapes (executor.cpp embed_forward,
    // head_forward_backward, embed_backward_and_update)
    {
        const size_t nwte = (size_t)d.Vp * h, nwpe = (size_t)d.s * h;
        uint16_t* wte_b = (uint16_t*)dmalloc(nwte * 2);
        uint16_t* wpe_b = (uint16_t*)dmalloc(nwpe * 2);
        uint16_t* lnf_b = (uint16_t*)dmalloc(2 * h * 2);
        uint16_t* dlnf_b = (uint16_t*)dmalloc(2 * h * 2);
        uint16_t* xf = (uint16_t*)dmalloc(T * h * 2);
        uint16_t* logits = (uint16_t*)dmalloc(T * (size_t)d.Vp * 2);
        float* stats = (float*)dmalloc((3 * T + 8 + AH_STATS_FLOATS) * 4);  // mean | rstd | losses | loss | grad stats
        float* lnf = (float*)dmalloc(2 * h * 4);
        float* wte = (float*)dmalloc(nwte * 4 * 4);  // master | m | v | fp32 grad
        float* wpe = (float*)dmalloc(nwpe * 4 * 4);
        uint16_t* dwte_b = (uint16_t*)dmalloc(nwte * 2);
        uint16_t* dwpe_b = (uint16_t*)dmalloc(nwpe * 2);
        int32_t* tok = (int32_t*)dmalloc((5 * T + 8) * 4);
        ok(gpt::init_normal(wte, nwte * 4, 7, 0.f, 0.02f, st), "init");
        ok(gpt::init_normal(wpe, nwpe * 4, 8, 0.f, 0.02f, st), "init");
        ok(launch_cast_f32_bf16(wte, wte_b, nwte, st), "cast");
        ok(launch_cast_f32_bf16(wpe, wpe_b, nwpe, st), "cast");
        ok(gpt::fill_f32(lnf, 2 * h, 1.f, st), "init");
        ok(launch_cast_f32_bf16(lnf, lnf_b, 2 * h, st), "cast");
        std::vector<int32_t> ids(2 * T);
        for (size_t i = 0; i < 2 * T; ++i) ids[i] = (int32_t)((i * 2654435761ull) % (uint64_t)d.V);
        ok(cudaMemcpy(tok, ids.data(), 2 * T * 4, cudaMemcpyHostToDevice), "ids");
        int32_t *tgt = tok + T, *uniq = tok + 2 * T, *offs = uniq + T, *pos = offs + T + 1, *nuniq = pos + T;
        float *meanf = stats, *rstdf = stats + T, *losses = stats + 2 * T, *loss = stats + 3 * T;
        ah_adam_hparams hp = cfg.adam;
        hp.step = 1;
        auto nb_fwd = [&] {
            ok(gpt::token_index(tok, (int)T, uniq, offs, pos, nuniq, st), "token index");
            ok(gpt::embed_fwd(tok, wte_b, wpe_b, x0, (int)T, d.s, (int)h, st), "embed");
            ok(gpt::ln_fwd(x1, lnf_b, lnf_b + h, xf, meanf, rstdf, (int)T, (int)h, st), "lnf");
            gemm::GemmArgs g;
            g.M = T; g.N = d.Vp; g.K = h;
            g.A = xf; g.lda = h; g.B = wte_b; g.ldb = h; g.C = logits; g.ldc = d.Vp;
            ok(gemm::run(g, st), "logits");
            ok(gpt::cross_entropy(logits, tgt, losses, (int)T, d.V, d.Vp, 1.f / T, st), "ce");
            ok(gpt::mean_loss(losses, (int)T, loss, st), "loss");
        };
        auto nb_bwd = [&] {
            gemm::GemmArgs dg;
            dg.M = T; dg.N = h; dg.K = d.Vp;
            dg.A = logits; dg.lda = d.Vp; dg.B = wte_b; dg.b_mn_major = 1; dg.ldb = h; dg.C = ws.dln; dg.ldc = h;
            ok(gemm::run(dg, st), "head dgrad");
            gemm::GemmArgs wg;
            wg.M = d.Vp; wg.N = h; wg.K = T;
            wg.A = logits; wg.a_mn_major = 1; wg.lda = d.Vp; wg.B = xf; wg.b_mn_major = 1; wg.ldb = h;
            wg.C = wte + 3 * nwte; wg.c_f32 = 1; wg.ldc = h;
            ok(gemm::run(wg, st), "head wgrad");
            ok(gpt::ln_bwd2(ws.dln, x1, meanf, rstdf, lnf_b, nullptr, gx0, dlnf_b, ws.part, (int)T, (int)h, st), "lnf bwd");
            ok(gpt::embed_bwd_tok_dev(gx0, uniq, offs, pos, nuniq, (int)T, wte + 3 * nwte, (int)h, st), "embed bwd");
            ok(gpt::embed_bwd_pos(gx0, wpe + 3 * nwpe, d.B, d.s, (int)h, st), "pos bwd");
            ok(gpt::f32_to_bf16(wte + 3 * nwte, dwte_b, nwte, st), "cvt");
            ok(gpt::f32_to_bf16(wpe + 3 * nwpe, dwpe_b, nwpe, st), "cvt");
            ok(launch_grad_stats(dwte_b, nwte, 1.f, stats + 3 * T + 8, st), "stats");
            ok(launch_adam(adam_args(hp, 1, wte, wte + nwte, wte + 2 * nwte, dwte_b, wte_b, nwte), st), "adam wte");
            ok(launch_adam(adam_args(hp, 1, wpe, wpe + nwpe, wpe + 2 * nwpe, dwpe_b, wpe_b, nwpe), st), "adam wpe");
        };
        ok(cudaMemsetAsync(stats + 3 * T, 0, (8 + AH_STATS_FLOATS) * 4, st), "memset");
        out.t_nonblock_fwd_s = timed(5, nb_fwd);
        out.t_nonblock_bwd_s = timed(5, nb_bwd);
    }
    out.t_fwd_s = out.t_block_fwd_s + out.t_nonblock_fwd_s / L_model;
    out.t_bwd_s = out.t_block_bwd_s + out.t_nonblock_bwd_s / L_model;
    const double flops = 2.0 * (double)mp * (double)T + 4.0 * d.B * (double)d.s * d.s * h;
    out.gpu_flops = flops / out.t_fwd_s;
    out.bwd_fwd_ratio = out.t_bwd_s / out.t_fwd_s;
    ah_adam_hparams hp = cfg.adam;
    hp.step = 1;
    const double t_adam = timed(5, [&] { ok(launch_adam(adam_args(hp, 1, master, m1, m2, w, nullptr, mp), st), "adam"); });
    out.gpu_adam_rate = (double)mp / t_adam;
    uint16_t* hbuf;
    ok(cudaHostAlloc((void**)&hbuf, mp * 2, cudaHostAllocPortable), "host alloc");
    std::memset(hbuf, 0, mp * 2);
    out.h2d_bw = (double)mp * 2 / timed(5, [&] { ok(cudaMemcpyAsync(w, hbuf, mp * 2, cudaMemcpyHostToDevice, st), "h2d"); });
    out.d2h_bw = (double)mp * 2 / timed(5, [&] { ok(cudaMemcpyAsync(hbuf, w, mp * 2, cudaMemcpyDeviceToHost, st), "d2h"); });
    cudaFreeHost(hbuf);
    // CPU Adam on pinned host block states, cycled so one pass covers >= 2 GB (DRAM-resident as
    // in the step, where L different blocks stream through; a single small block would be timed
    // partly from the last-level cache)
    {
        const size_t per = mp * 14;
        const int nbuf = (int)std::min<size_t>(64, ((size_t)2 << 30) / per + 1);
        struct HB {
            float *p, *m, *v;
            uint16_t* g;
        };
        std::vector<HB> hb((size_t)nbuf);
        for (HB& b : hb) {
            ok(cudaHostAlloc((void**)&b.p, mp * 4, cudaHostAllocPortable), "host alloc");
            ok(cudaHostAlloc((void**)&b.m, mp * 4, cudaHostAllocPortable), "host alloc");
            ok(cudaHostAlloc((void**)&b.v, mp * 4, cudaHostAllocPortable), "host alloc");
            ok(cudaHostAlloc((void**)&b.g, mp * 2, cudaHostAllocPortable), "host alloc");
            std::memset(b.p, 0, mp * 4);
            std::memset(b.m, 0, mp * 4);
            std::memset(b.v, 0, mp * 4);
            std::memset(b.g, 0, mp * 2);
        }
        auto pass = [&] {
            for (HB& b : hb) cpu_adam(hp, b.p, b.m, b.v, b.g, b.g, mp, 1.f, cfg.cpu_threads);
        };
        pass();  // page-in / warm
        std::vector<double> t;
        for (int r = 0; r < 3; ++r) {
            const auto c0 = Clock::now();
            pass();
            t.push_back(std::chrono::duration<double>(Clock::now() - c0).count());
        }
        std::sort(t.begin(), t.end());
        out.cpu_adam_rate = (double)mp * nbuf / t[1];
        for (HB& b : hb)
            for (void* q : {(void*)b.p, (void*)b.m, (void*)b.v, (void*)b.g}) cudaFreeHost(q);
    }
    for (void* p : dev) cudaFree(p);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
    return out;
}

float Trainer::timer(bool stop) {
    drain();
    if (!timer_ev_[0]) {
        check(cudaEventCreate(&timer_ev_[0]), "event");
        check(cudaEventCreate(&timer_ev_[1]), "event");
    }
    if (!stop) {
        check(cudaEventRecord(timer_ev_[0], s_compute_), "record");
        return 0.f;
    }
    check(cudaEventRecord(timer_ev_[1], s_compute_), "record");
    check(cudaEventSynchronize(timer_ev_[1]), "sync");
    float ms = 0.f;
    check(cudaEventElapsedTime(&ms, timer_ev_[0], timer_ev_[1]), "elapsed");
    return ms;
}

void Trainer::reset_stats() {
    std::lock_guard<std::mutex> lk(mu_);
    for (LaneStats& l : lane_stats_) l = LaneStats{};
    enqueue_ms_ = enqueue_max_ms_ = 0.0;
    win_iters_ = win_compute_ms_ = win_h2d_ms_ = win_d2h_ms_ = win_blocked_ms_ = 0;
    win_h2d_bytes_ = win_d2h_bytes_ = win_h2d_link_ms_ = 0;
    win_copy_blocked_ms_ = win_upstream_blocked_ms_ = win_cpu_ms_ = win_span_ms_ = 0;
}

}  // namespace ah

namespace ah {

// Offload overlap of the drained window: for every compute op that depends on a copy-lane or
// CPU op, the idle gap before it on the compute stream (previous compute op end -> its start)
// is time the compute lane was blocked by offloading. The gap is split at the start of the
// copy it waited for: the part while that copy ran is copy-blocked (the host link did not keep
// up), the part before it is upstream-blocked (the copy itself waited for the CPU optimizer or
// for the copy lane's in-order queue).
void Trainer::account_window() {
    std::lock_guard<std::mutex> lk(mu_);
    if (iters_.empty()) return;
    cudaEvent_t origin = nullptr;
    for (auto& kv : iters_.front()->ops)
        if (kv.second.kind == OpKind::Forward && kv.second.block == 1) origin = kv.second.t0;
    if (!origin) return;
    auto span = [&](const RtOp& o, double& a, double& b) {
        float x = 0, y = 0;
        if (cudaEventElapsedTime(&x, origin, o.t0) != cudaSuccess) return false;
        if (cudaEventElapsedTime(&y, origin, o.t1) != cudaSuccess) return false;
        a = x;
        b = y;
        return true;
    };
    struct Span {
        double a, b;
        bool waits;
        double ca, cb;  // the awaited copy's span (latest-finishing offload dependency)
    };
    std::vector<Span> comp;
    double h2d = 0, d2h = 0, hb = 0, db = 0, cpu = 0, h2d_link = 0;
    const double wbytes = 2.0 * (double)(dp_ ? shard_ : d_.m_p());
    for (Iter* it : iters_)
        for (auto& kv : it->ops) {
            RtOp& o = kv.second;
            if (o.lane == kCpu) {
                cpu += o.host_ms;
                continue;
            }
            double a = 0, b = 0;
            if (!span(o, a, b)) continue;
            if (o.lane == kCompute) {
                Span sp{a, b, false, 0, 0};
                for (const auto& dp : o.deps) {
                    const int k = dp.second.kind;
                    if (k != (int)OpKind::ParamPrefetch && k != (int)OpKind::GradOffload && k != (int)OpKind::CpuOptim)
                        continue;
                    sp.waits = true;
                    const RtOp* d = find(dp.first, dp.second);
                    double ca = 0, cb = 0;
                    if (d && d->lane != kCpu && span(*d, ca, cb) && cb >= sp.cb) {
                        // a streamed prefetch waits for the host AdamW between chunks: only its
                        // last chunk's copy is time the link kept the compute lane waiting
                        float x = 0.f;
                        if (!d->ct.empty() && cudaEventElapsedTime(&x, origin, d->ct[d->ct.size() - 2]) == cudaSuccess)
                            ca = x;
                        sp.ca = ca;
                        sp.cb = cb;
                    }
                }
                comp.push_back(sp);
            } else if (o.lane == kH2D) {
                const double ms = op_ms(o);
                h2d += ms;
                if (blocks_[(size_t)o.block].o) {  // a PCIe copy (a P block outside O is a GPU cast)
                    hb += wbytes;
                    h2d_link += ms;
                }
            } else {
                d2h += b - a;
                db += wbytes;
            }
        }
    std::sort(comp.begin(), comp.end(), [](const Span& x, const Span& y) { return x.a < y.a; });
    double busy = 0, copy_blocked = 0, upstream = 0;
    for (size_t i = 0; i < comp.size(); ++i) {
        busy += comp[i].b - comp[i].a;
        if (i == 0 || !comp[i].waits) continue;
        const double g0 = comp[i - 1].b, g1 = comp[i].a;
        if (g1 <= g0) continue;
        const double c = std::max(0.0, std::min(g1, comp[i].cb) - std::max(g0, comp[i].ca));
        copy_blocked += c;
        upstream += (g1 - g0) - c;
    }
    win_iters_ = (double)iters_.size();
    win_compute_ms_ = busy;
    win_h2d_ms_ = h2d;
    win_d2h_ms_ = d2h;
    win_blocked_ms_ = copy_blocked + upstream;
    win_copy_blocked_ms_ = copy_blocked;
    win_upstream_blocked_ms_ = upstream;
    win_cpu_ms_ = cpu;
    win_span_ms_ = comp.empty() ? 0.0 : comp.back().b - comp.front().a;
    win_h2d_bytes_ = hb;
    win_h2d_link_ms_ = h2d_link;
    win_d2h_bytes_ = db;
}

}  // namespace ah
