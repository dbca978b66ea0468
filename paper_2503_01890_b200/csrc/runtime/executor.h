// B200 executor for the AutoHete iteration: realises the hetsim op DAG
// (build_iteration_ops, reference proj/core/src/simulator.cpp:91-229) on four lanes —
// a high-priority compute stream, an H2D copy stream, a D2H copy stream and a host CPU
// worker — in the per-lane order produced by the reference scheduler (priority-based or
// FIFO, simulator.cpp:413-450). Each lane is driven by its own host thread; cross-lane
// dependencies become cudaStreamWaitEvent (GPU -> GPU), cudaEventSynchronize (GPU -> CPU)
// or a host condition variable (CPU -> GPU); start-after-start launch gates become events
// recorded on the compute stream immediately before the gated op.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "autohete.h"
#include "gpt_model.h"
#include "hetsim/dp_planner.hpp"
#include "hetsim/planner.hpp"
#include "hetsim/simulator.hpp"

namespace ah {

struct LaneStats {
    double busy_ms = 0.0;  // host-observed for the CPU lane; event-timed for GPU lanes
    int ops = 0;
};

class Trainer {
public:
    explicit Trainer(const ah_trainer_config& cfg);
    ~Trainer();

    // Enqueue one training iteration. tokens/targets: B*s int32, host (pinned or pageable)
    // unless on_device. Returns immediately; lanes run asynchronously.
    void submit(const int32_t* tokens, const int32_t* targets, bool on_device);
    // Block until every submitted iteration finished; returns the last iteration's loss.
    float drain();
    // One synchronous iteration (H2D of inputs, full step, D2H of the loss).
    float step(const int32_t* tokens, const int32_t* targets);

    const hetsim::Strategy& strategy() const { return strategy_; }
    const hetsim::ModelProfile& profile() const { return profile_; }
    const GptDims& dims() const { return d_; }
    const hetsim::SimResult& simulated() const { return sim_; }
    // Switch the per-lane order of subsequent iterations between the priority-based (paper §3.3)
    // and the FIFO schedule of the reference scheduler (drains first; weights / state kept).
    void set_schedule(bool priority);
    // In-step calibration of the block durations from the drained window (ah_calibration).
    void calibrate(ah_calibration* out);
    bool apply_calibration(bool keep_strategy);
    void stats(ah_trainer_stats* out);
    void reset_stats();  // zero the lane busy-time counters and the offload window
    // fp32 master of block b (1-based; 0 = embedding wte, -1 = wpe, -2 = final LN) -> host.
    void read_master(int block, float* out, size_t n);
    size_t master_size(int block) const;
    // Chrome trace of the last drained iterations in the reference schema (simulator.cpp:598).
    std::string trace_json();
    // Measured GPU-memory timeline of the drained window in the reference CSV schema
    // (write_memory_csv, simulator.cpp:615-622): persistent allocations + the executor's
    // stream-ordered transient buffers, taken at each op's start and returned at its end
    // (CUDA-event times, µs from the window's first op).
    std::string memory_csv(int64_t* peak_bytes = nullptr);
    // drain + record start (stop=false) / drain + record stop and return elapsed ms (stop=true)
    float timer(bool stop);
    // Optimizer-state checkpoint (fp32 master, m, v of this rank's part of every block + the
    // replicated embedding state + the step counter). Plan-independent: a checkpoint taken
    // under one (c, p, o) plan loads under another (GPU- or host-resident state alike).
    void save(const std::string& path);
    void load(const std::string& path);

private:
    cudaEvent_t timer_ev_[2] = {nullptr, nullptr};
    int step_base_ = 0;  // optimizer steps completed before this trainer (checkpoint resume)
    friend struct CheckpointIO;
    // data parallel
    int dp_rank_ = 0, dp_size_ = 1;
    int device_ = 0;  // the caller's current device at construction; every lane thread binds to it
    bool dp_ = false;      // collectives on
    void* comm_ = nullptr; // ncclComm_t
    class LoopbackComm* loop_ = nullptr;  // in-process ranks on one GPU instead of NCCL (not owned)
    size_t shard_ = 0;     // per-rank shard length of a block vector (elements, padded)
    size_t my_len_ = 0;    // valid elements of this rank's shard
    size_t full_len() const { return dp_ ? shard_ * (size_t)dp_size_ : d_.m_p(); }
    void dp_gather(uint16_t* wbuf, cudaStream_t st);     // shard -> full bf16 weights
    void dp_reduce_grads(uint16_t* wbuf, cudaStream_t st);  // full grads -> my shard (sum)
    void dp_allreduce_f32(float* p, size_t n, cudaStream_t st);
    void dp_allreduce_bf16(uint16_t* p, size_t n, cudaStream_t st);
    enum Lane { kCompute = 0, kH2D = 1, kD2H = 2, kCpu = 3 };
    struct OpKey {
        int kind, block;
        bool bwd;
        bool operator<(const OpKey& o) const {
            if (kind != o.kind) return kind < o.kind;
            if (block != o.block) return block < o.block;
            return bwd < o.bwd;
        }
    };
    struct RtOp {
        hetsim::OpKind kind;
        int block = 0;
        bool bwd = false;
        long long iter = 0;  // global iteration number (1-based)
        int lane = 0;
        std::vector<std::pair<long long, OpKey>> deps;   // (iteration, op)
        std::vector<std::pair<long long, OpKey>> gates;  // start-after-start (compute ops)
        cudaEvent_t done_ev = nullptr, start_ev = nullptr, t0 = nullptr, t1 = nullptr;
        int state = 0;  // 0 pending, 1 started (start_ev recorded), 2 issued (done_ev recorded), 3 done (host)
        double host_ms = 0.0;
        bool done_on_side = false;  // DP backward: done_ev follows the gradient reduce-scatter on s_side_
        int64_t alloc_b = 0, free_b = 0;  // transient bytes (arena slots) taken at its start / returned at its end
        // Sub-block streaming (nsub_ > 1). CpuOptim: chunks of the block updated so far (the
        // next iteration's forward ParamPrefetch copies chunk c up as soon as progress > c).
        // Streamed ParamPrefetch: the CpuOptim it follows, and per-chunk copy timing events
        // (start, end) so its busy time excludes the waits for the CPU between chunks.
        int progress = 0;
        bool streamed = false;
        std::pair<long long, OpKey> stream_src{0, OpKey{0, 0, false}};
        std::vector<cudaEvent_t> ct;
    };
    struct Iter {
        long long k = 0;
        std::map<OpKey, RtOp> ops;
        std::vector<OpKey> lane_order[4];
        const int32_t* tokens = nullptr;
        const int32_t* targets = nullptr;
        bool on_device = false;
        int finished_lanes = 0;
    };
    struct BlockState {
        bool o = false, p = false, c = false;
        float* master = nullptr;  // device (non-O) or pinned host (O)
        float* m1 = nullptr;
        float* m2 = nullptr;
        uint16_t* host_bf16 = nullptr;  // O blocks: shared param/grad buffer
        uint16_t* wbuf = nullptr;       // device bf16 weights / grads while resident
        void* acts = nullptr;           // device activation set while live
        bool needs_gather = false;      // DP: wbuf holds only this rank's shard so far
        cudaEvent_t mat_ev = nullptr;   // side-stream materialisation (cast [+ all-gather]) done
        bool mat_pending = false;       // wbuf was materialised ahead on s_side_; compute must wait mat_ev
        std::vector<cudaEvent_t> go_ev; // O blocks, nsub_ > 1: GradOffload chunk c landed in host_bf16
    };

    void plan(const ah_trainer_config& cfg);
    void allocate_and_init();
    void build_iteration(Iter& it);
    void lane_main(int lane);
    // state_only > 0: wait until the dependency reached that state (1 started, 2 issued) and
    // leave the data dependency to the caller (sub-block streaming)
    void wait_dep(int lane, long long iter, const OpKey& key, bool gate, bool needs_side = false, int state_only = 0);
    // Side stream: materialisation of the next compute op's weights (overlapping the current
    // op) and every NCCL collective, issued by the compute lane thread in op order.
    void prefetch_weights(const Iter& it, size_t idx, RtOp& cur);
    void side_after_compute();
    void compute_after_side();
    RtOp* find(long long iter, const OpKey& key);
    void run_compute(Iter& it, RtOp& op);
    void run_h2d(Iter& it, RtOp& op);
    void run_d2h(Iter& it, RtOp& op);
    void run_cpu(Iter& it, RtOp& op);
    // Sub-block streaming of the offload chain GradOffload -> CpuOptim -> next forward
    // ParamPrefetch of an O block: the block vector is cut into nsub_ contiguous chunks; the
    // host AdamW starts on chunk 0 as soon as its D2H copy landed, and the prefetch sends chunk
    // c up as soon as the host AdamW finished it. Per-lane op order and every dependency of the
    // reference DAG are kept; only the tail of one op overlaps the head of the next.
    int nsub_ = 1;
    void sub_range(int c, size_t n, size_t& a, size_t& len) const;
    void wait_progress(long long iter, const OpKey& key, int chunks);
    double op_ms(const RtOp& o) const;  // lane busy time of a GPU-lane op (chunk sum when streamed)
    void embed_forward(Iter& it);
    void head_forward_backward(Iter& it);
    void embed_backward_and_update(Iter& it);
    void upload_inputs(Iter& it);
    void check(cudaError_t e, const char* what);
    cudaStream_t stream_of(int lane) const;

    GptDims d_;
    hetsim::ModelProfile profile_;
    hetsim::HardwareSpec hw_;
    hetsim::Strategy strategy_;
    hetsim::dp::DpSpec dp_spec_;
    hetsim::ModelSpec spec_;            // model as given to build_profile
    hetsim::ProfileOverrides ov_;       // m_gc of this runtime
    hetsim::HardwareSpec hw_cfg_;       // rates / budgets as configured (before DP adjustments)
    bool fine_tune_ = false;
    // last calibrate(): the rates it derived and the plan the reference planner picks with them
    bool cal_valid_ = false, cal_plan_valid_ = false;
    hetsim::HardwareSpec cal_hw_;
    hetsim::ModelSpec cal_spec_;
    hetsim::Strategy cal_strategy_;
    hetsim::SimResult sim_;
    double sim_steady_[2] = {0.0, 0.0};  // reference scheduler steady state: [0] FIFO, [1] PS
    double sim_lane_ms_[4] = {0, 0, 0, 0};  // simulated busy time per lane, steady iteration
    void compile_order();                // order_ from sim_
    bool ps_ = true;
    ah_adam_hparams adam_{};
    unsigned long long seed_ = 1234;
    int cpu_threads_ = 0;
    // per-lane compiled order of iteration 1 and of the steady state (iteration 2)
    std::vector<OpKey> order_[2][4];

    cudaStream_t s_compute_ = nullptr, s_h2d_ = nullptr, s_d2h_ = nullptr;
    cudaStream_t s_side_ = nullptr;
    cudaStream_t s_mark_ = nullptr;  // idle: timestamps of host (CpuOptim) ops on the GPU timeline
    cudaEvent_t ev_c2s_ = nullptr, ev_s2c_ = nullptr;  // reused: a wait binds to the latest record
    std::vector<BlockState> blocks_;  // index 1..L
    std::vector<uint16_t*> x_;        // residual stream x[0..L] (x[0] = embedding output)
    uint16_t* gx_[2] = {nullptr, nullptr};  // residual-gradient ping-pong
    void* ws_mem_ = nullptr;
    void* acts_arena_ = nullptr;      // L - c_hat + 1 activation sets (see allocate_and_init)
    size_t acts_slot_ = 0;
    std::vector<void*> acts_free_;    // free slots, LIFO; compute lane only
    // block weight / gradient buffer slots (see allocate_and_init)
    size_t wslot_bytes_ = 0;
    std::vector<uint16_t*> wslot_ptr_;
    std::map<const void*, int> wslot_index_;
    std::vector<cudaEvent_t> wslot_ev_;   // recorded on the releasing stream
    std::vector<uint8_t> wslot_recorded_;
    std::deque<int> wslot_free_;
    std::mutex wslot_mu_;
    int wslot_overflow_ = 0;
    uint16_t* wslot_alloc(cudaStream_t st);
    void wslot_add();  // caller holds wslot_mu_ (or is the constructor)
    void wslot_free(uint16_t* p, cudaStream_t st);
    Workspace ws_;
    // head / embedding (GPU-resident, m_gc)
    float *wte_ = nullptr, *wte_m_ = nullptr, *wte_v_ = nullptr;
    float *wpe_ = nullptr, *wpe_m_ = nullptr, *wpe_v_ = nullptr;
    float *lnf_ = nullptr, *lnf_m_ = nullptr, *lnf_v_ = nullptr;
    uint16_t *wte_b_ = nullptr, *wpe_b_ = nullptr, *lnf_b_ = nullptr;
    float *dwte_ = nullptr, *dwpe_ = nullptr;
    uint16_t *dwte_b_ = nullptr, *dwpe_b_ = nullptr, *dlnf_b_ = nullptr;
    uint16_t* logits_ = nullptr;
    uint16_t* xf_ = nullptr;
    float *meanf_ = nullptr, *rstdf_ = nullptr, *losses_ = nullptr, *loss_dev_ = nullptr;
    float* loss_host_ = nullptr;  // pinned
    int32_t* tok_dev_ = nullptr;  // [2][T] tokens, [2][T] targets, inverse index
    int32_t* tok_host_ = nullptr; // pinned staging for inputs + inverse index
    size_t inv_words_ = 0;
    int n_uniq_[2] = {0, 0};
    cudaMemPool_t pool_ = nullptr;
    size_t static_bytes_ = 0;
    int gpu_adam_steps_ = 0;

    // iteration window
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Iter*> iters_;
    std::vector<Iter*> retired_;
    long long submitted_ = 0, completed_ = 0;
    bool stop_ = false;
    std::string error_;
    std::thread lanes_[4];
    size_t lane_pos_[4] = {0, 0, 0, 0};  // index into iters_ window per lane
    LaneStats lane_stats_[4];
    double enqueue_ms_ = 0.0, enqueue_max_ms_ = 0.0;  // compute lane: host time per compute op enqueue
    float last_loss_ = 0.f;
    // offload-overlap accounting of the last drain (see ah_trainer_stats)
    double win_iters_ = 0, win_compute_ms_ = 0, win_h2d_ms_ = 0, win_d2h_ms_ = 0, win_blocked_ms_ = 0;
    double win_h2d_bytes_ = 0, win_d2h_bytes_ = 0, win_h2d_link_ms_ = 0;
    double win_copy_blocked_ms_ = 0, win_upstream_blocked_ms_ = 0, win_cpu_ms_ = 0, win_span_ms_ = 0;
    // Gradient statistics (overflow check + norm), one AH_STATS_FLOATS slot per block group:
    // slot 0 = embedding / positions / final LN, slot i = block i. Each slot is zeroed and filled
    // by the grad_stats pre-pass right after the group's backward; its non-finite count is the
    // skip flag of that group's update (GPU: device flag; CPU: read from gstats_host_).
    float* gstats_dev_ = nullptr;
    float* gstats_host_ = nullptr;  // pinned: [2 * slot] = {sum g^2, (uint32) non-finite}
    double grad_norm_ = 0.0;
    long long nonfinite_ = 0;
    int skipped_ = 0;
    float* gstats(int slot) const;
    void grad_stats_pass(int slot, const uint16_t* g, size_t n, cudaStream_t st);
    void collect_grad_stats();
    void account_window();
    int64_t retired_bytes_ = 0;  // net transient bytes of ops in iterations already retired
};

}  // namespace ah
