/* autohete.h — C-ABI data plane of the B200-native AutoHete hot path.
 *
 * The reference (arXiv 2503.01890, /root/reference/proj) plans and SIMULATES one training
 * iteration: its hetsim::core API (include/hetsim/ headers here, drop-in) decides
 * (c_hat, p_hat, o_hat, prefetch_lookahead) and the per-lane op order, and models every op
 * only as a duration. This header is the layer beneath it that EXECUTES those ops on B200.
 * Each entry point names the reference op / interface it realises (file:line in
 * /root/reference/proj). Rules for every function:
 *   - plain pointers + sizes, no C++/torch types; caller owns all buffers;
 *   - return 0 (AH_OK) or a negative AH_ERR_* code; ah_last_error() gives a thread-local
 *     message; no exceptions cross this boundary;
 *   - "stream" is a cudaStream_t passed as void* (NULL = legacy default stream); device
 *     work is asynchronous on it and safe on distinct streams concurrently;
 *   - no allocation on the hot path (ah_*_create / ah_host_alloc are setup calls).
 */
#ifndef AUTOHETE_H
#define AUTOHETE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AH_OK 0
#define AH_ERR_INVALID -1   /* bad argument (std::invalid_argument in the C++ API) */
#define AH_ERR_CUDA -2      /* CUDA runtime / driver error */
#define AH_ERR_INFEASIBLE -3 /* hetsim::InfeasibleError (planner.hpp) */
#define AH_ERR_MEMORY -4    /* hetsim::MemoryExceededError (simulator.hpp) */
#define AH_ERR_NCCL -5      /* NCCL error */
#define AH_ERR_INTERNAL -6  /* std::logic_error / anything else */

const char* ah_last_error(void);
int ah_abi_version(void); /* bumps on any signature or struct layout change; 5: ah_trainer_stats gained
                           * stream_chunks, pool_reserved_bytes, compute_enqueue_ms / _max_ms,
                           * buffer_overflows (appended) */

/* ---------------------------------------------------------------------------------------
 * Optimizer (OpKind::GpuOptim / OpKind::CpuOptim).
 * Reference interface replaced: HardwareSpec::{gpu_optim_rate,cpu_optim_rate}
 * (proj/core/include/hetsim/workload.hpp:39-40) -> BlockProfile::{t_opt_gpu,t_opt_cpu}
 * (workload.hpp:58-59, workload.cpp:70-71) -> ops emitted at simulator.cpp:210-226.
 * --------------------------------------------------------------------------------------- */
typedef struct ah_adam_hparams {
    float lr;
    float beta1;
    float beta2;
    float eps;
    float weight_decay; /* decoupled (AdamW) */
    int32_t step;       /* 1-based step used for bias correction */
} ah_adam_hparams;

/* Gradient statistics buffer: device float[AH_STATS_FLOATS], zeroed once by the caller.
 * [0] = sum of squared unscaled grads, [1] = (uint32) count of non-finite grads, both
 * ACCUMULATED over the launches that use the buffer, in stream order; the rest is scratch for
 * the fixed-order cross-CTA reduction (bitwise reproducible: no float atomics). One buffer
 * must not be used by two launches running concurrently. Zero [0] and [1] to restart. */
#define AH_STATS_FLOATS 520

/* Fused AdamW on one parameter span (one block = m_p params, workload.cpp:41-44):
 * fp32 master p / moments m, v updated in place from bf16 grads g scaled by inv_scale;
 * optional bf16 copy of the updated params into p_bf16 (may alias nothing else).
 * skip_flag: optional device int32; non-zero => no-op (overflow skip). Pointing it at
 * stats + 1 of a preceding ah_grad_stats skips the update iff a grad was inf / nan.
 * stats: optional AH_STATS_FLOATS buffer (above) accumulating the grads this launch reads.
 * 28 HBM bytes/param with p_bf16, 26 without. */
int ah_adam_step(const ah_adam_hparams* hp, float* p, float* m, float* v, const uint16_t* g,
                 uint16_t* p_bf16, size_t n, float inv_scale, const int32_t* skip_flag,
                 float* stats, void* stream);

/* Grad norm / overflow pre-pass (2 B/param read; warp-shuffle + fixed-order cross-CTA
 * reductions) accumulated into an AH_STATS_FLOATS buffer as above. */
int ah_grad_stats(const uint16_t* g, size_t n, float inv_scale, float* stats, void* stream);

/* bf16 materialisation of a GPU-resident fp32 master (paper footnote 2, PAPER.md:205-207;
 * modelled as the transient 2*m_p alloc of F_i/B_i at simulator.cpp:131-136, 192-196). */
int ah_cast_f32_bf16(const float* src, uint16_t* dst, size_t n, void* stream);

/* Host AdamW over the 14 B/param host layout (costmodel.cpp:44-46): same arithmetic as
 * ah_adam_step, bit-identical results. g and p_bf16 may alias (the shared host buffer).
 * nthreads <= 0 => all host cores. Synchronous. */
int ah_cpu_adam(const ah_adam_hparams* hp, float* p, float* m, float* v, const uint16_t* g,
                uint16_t* p_bf16, size_t n, float inv_scale, int nthreads);

/* ---------------------------------------------------------------------------------------
 * Host link (OpKind::ParamPrefetch = H2D lane, OpKind::GradOffload = D2H lane).
 * Reference interface replaced: HardwareSpec::{h2d_bandwidth,d2h_bandwidth}
 * (workload.hpp:37-38) -> t_h2d/t_d2h = 2*m_p/BW (workload.cpp:68-69) -> ops at
 * simulator.cpp:113-123, 147-167, 200-208.
 * --------------------------------------------------------------------------------------- */
int ah_host_alloc(void** ptr, size_t bytes); /* pinned, portable */
int ah_host_free(void* ptr);
int ah_host_register(void* ptr, size_t bytes);
int ah_host_unregister(void* ptr);
int ah_copy_h2d(void* dst_dev, const void* src_host, size_t bytes, void* stream);
int ah_copy_d2h(void* dst_host, const void* src_dev, size_t bytes, void* stream);
/* Priority-ordered stream pair for the copy lanes (greatest priority). */
int ah_stream_create(void** stream, int high_priority);
int ah_stream_destroy(void* stream);

/* ---------------------------------------------------------------------------------------
 * Dense contractions of OpKind::Forward / Backward / Recompute on tcgen05 tensor cores.
 * Reference interface replaced: HardwareSpec::gpu_compute_rate (workload.hpp:36) ->
 * t_fp = (2*m_p*b*s + 4*b*s^2*h)/rate, t_bp = bwd_fwd_ratio*t_fp (workload.cpp:55-73).
 *
 *   C[z](m,n) = epi(alpha * sum_k A[z](m,k) * B[z](n,k) + beta * C[z](m,n))
 *   z = z1 + batch1*z2 ; element (m,k) of a K-major A is A[z1*a_s1 + z2*a_s2 + m*lda + k],
 *   of an MN-major A is A[... + k*lda + m]; likewise B with n. All strides in elements.
 * A, B bf16 (16-byte aligned, lda/ldb multiples of 8); C bf16 or fp32.
 * --------------------------------------------------------------------------------------- */
#define AH_EPI_BIAS 1
#define AH_EPI_GELU 2
#define AH_EPI_RESIDUAL 4
#define AH_EPI_AUX 16
#define AH_EPI_GELU_BWD 32 /* multiply by GELU'(aux): fused GELU backward */
#define AH_CAUSAL_NONE 0
#define AH_CAUSAL_SKIP_UPPER 1
#define AH_CAUSAL_K_UPTO_M 2
#define AH_CAUSAL_K_FROM_M 3

typedef struct ah_gemm_desc {
    int64_t M, N, K;
    int32_t batch1, batch2;
    const void* A;
    int32_t a_mn_major;
    int64_t lda, a_s1, a_s2;
    const void* B;
    int32_t b_mn_major;
    int64_t ldb, b_s1, b_s2;
    void* C;
    int32_t c_f32;
    int64_t ldc, c_s1, c_s2;
    const void* bias; /* per-n vector, bf16 or fp32 (bias_f32) */
    int32_t bias_f32;
    const void* residual; /* bf16, same indexing as C with ld_res / res_s1 / res_s2 */
    int64_t ld_res, res_s1, res_s2;
    void* aux; /* bf16 pre-GELU output (AH_EPI_AUX) */
    int64_t ld_aux, aux_s1, aux_s2;
    float alpha, beta;
    int32_t epilogue; /* AH_EPI_* bitmask */
    int32_t causal;   /* AH_CAUSAL_* */
    int32_t block_n;  /* 0 = auto, else 64 / 128 / 256 */
} ah_gemm_desc;

int ah_gemm_bf16(const ah_gemm_desc* desc, void* stream);

/* Fused causal attention of one block (part of OpKind::Forward / Recompute / Backward; the
 * reference's 4*b*s^2*h attention term of t_fp, workload.cpp:63). head_dim must be 128.
 * Flash attention forward: qkv [B, s, 3h] bf16 -> O [B, s, h] bf16 and
 * lse2 [B, heads, s] fp32, the per-row log2-domain log-sum-exp of the scaled scores. */
int ah_attention_flash_fwd(const uint16_t* qkv, uint16_t* O, float* lse2, int32_t batch, int32_t seq_len,
                           int32_t heads, int32_t head_dim, void* stream);

/* Flash attention backward: from qkv, O, dO [B, s, h] and lse2 -> dqkv [B, s, 3h] bf16 (dQ, dK,
 * dV of every head; P recomputed). workspace: caller-owned device scratch of at least
 * ah_attention_flash_bwd_workspace(batch, seq_len, heads) bytes (16-byte aligned). */
size_t ah_attention_flash_bwd_workspace(int32_t batch, int32_t seq_len, int32_t heads);
int ah_attention_flash_bwd(const uint16_t* qkv, const uint16_t* O, const uint16_t* dO, const float* lse2,
                           uint16_t* dqkv, int32_t batch, int32_t seq_len, int32_t heads, int32_t head_dim,
                           void* workspace, size_t workspace_bytes, void* stream);

/* LayerNorm of the block step (part of OpKind::Forward / Backward / Recompute; no reference
 * kernel — the reference times the whole block as t_fp / t_bp, workload.cpp:55-67).
 * x, y [rows, h] bf16; gamma, beta [h] bf16; mean, rstd [rows] fp32 (eps 1e-5). */
int ah_layernorm_fwd(const uint16_t* x, const uint16_t* gamma, const uint16_t* beta, uint16_t* y,
                     float* mean, float* rstd, int32_t rows, int32_t h, void* stream);
/* dx = LN'(dy) (+ dres if non-null); dgamma_dbeta [2h] = [sum dy*xhat | sum dy] (bf16).
 * Optional fused bias gradients (h % 256 == 0): dres_colsum [h] = column sums of dres,
 * dx_colsum [h] = column sums of bf16(dx). Deterministic (fixed-order reductions). */
/* workspace: caller-owned device scratch of ah_layernorm_bwd_workspace(rows, h) bytes (the
 * fixed-order column-reduction partials). */
size_t ah_layernorm_bwd_workspace(int32_t rows, int32_t h);
int ah_layernorm_bwd(const uint16_t* dy, const uint16_t* x, const float* mean, const float* rstd,
                     const uint16_t* gamma, const uint16_t* dres, uint16_t* dx, uint16_t* dgamma_dbeta,
                     uint16_t* dres_colsum, uint16_t* dx_colsum, int32_t rows, int32_t h, void* workspace,
                     size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------
 * Training executor: one GPT iteration = hetsim::build_iteration_ops(profile, strategy, k)
 * (proj/core/src/simulator.cpp:91-229) executed on B200 in the per-lane order of
 * hetsim::run(..., priority_sched) (simulator.cpp:263-596). The planner step is
 * hetsim::solve + fine_tune_prefetch (proj/core/src/planner.cpp:37-153) on a profile built
 * from the real block shape and the rates given here (measured on the box by the caller).
 * --------------------------------------------------------------------------------------- */
typedef struct ah_trainer_config {
    int32_t num_blocks, hidden, heads, seq_len, batch, vocab;
    /* strategy: c_hat/p_hat/o_hat >= 0 forces it; any < 0 => planner decides */
    int32_t c_hat, p_hat, o_hat;
    const int32_t* prefetch_lookahead; /* nullable; L entries when forcing a strategy */
    int32_t priority_sched;            /* 1: PS order (paper §3.3), 0: FIFO */
    int32_t fine_tune;                 /* run fine_tune_prefetch after solve */
    int64_t gpu_mem_budget, cpu_mem_budget; /* planner budgets, bytes */
    double gpu_flops, h2d_bw, d2h_bw, cpu_adam_rate, gpu_adam_rate; /* HardwareSpec rates */
    double bwd_fwd_ratio; /* ModelSpec::bwd_fwd_ratio (<= 0 => 2.0) */
    ah_adam_hparams adam;
    uint64_t seed;
    int32_t cpu_threads; /* CPU Adam threads, <= 0 = all */
    /* Data parallel (north_star (d)): dp_size ranks, one per GPU; each rank owns a 1/dp_size
     * shard of every block's fp32 master + moments (GPU or pinned host per the plan).
     * Parameters are all-gathered (bf16) before each use, gradients reduce-scattered
     * (bf16 sum, 1/dp_size folded into the optimizer) after each block's backward — NCCL over
     * NVLink, issued in the compute lane's deterministic order. dp_size <= 1 and
     * !force_collectives => no NCCL. nccl_id: ncclUniqueId from ah_dp_unique_id on rank 0. */
    int32_t dp_rank, dp_size, force_collectives;
    uint8_t nccl_id[128];
    /* dp_size > 1 and dp_aware_plan: plan with the data-parallel extension hetsim::dp::solve
     * (include/hetsim/dp_planner.hpp: per-rank sharded optimizer memory and shard copy /
     * optimizer times; collective_bw bytes/s bounds the block times, <= 0 = not modelled)
     * instead of the single-GPU reference solve. */
    int32_t dp_aware_plan;
    double collective_bw;
    /* non-null: exchange with these in-process ranks through an ah_dp_loopback_create
     * communicator instead of NCCL (all ranks on one GPU; validation of the DP path). */
    void* loopback_comm;
} ah_trainer_config;

/* ncclGetUniqueId into out[128] (rank 0; broadcast it to the other ranks). */
int ah_dp_unique_id(uint8_t* out);
/* Shard of a flat block vector of n elements owned by `rank` (16-byte aligned shards):
 * elements [*offset, *offset + *len) of the padded vector of dp_size * (*shard) elements. */
/* In-process loopback communicator for nranks trainers sharing one GPU (same in-place
 * collective semantics as the NCCL path; device copies + a fixed-order sum kernel). */
int ah_dp_loopback_create(int32_t nranks, void** comm);
int ah_dp_loopback_destroy(void* comm);
/* One rank's side of a loopback collective (blocks until every rank has posted it): op 0 =
 * all-gather bf16 (count = shard), 1 = reduce-scatter bf16 sum (count = shard), 2 = all-reduce
 * fp32, 3 = all-reduce bf16 (count = elements). buf = this rank's full buffer, in place. */
int ah_dp_loopback_call(void* comm, int32_t rank, int32_t op, void* buf, size_t count, void* stream);
int ah_dp_shard(int64_t n, int32_t rank, int32_t dp_size, int64_t* offset, int64_t* len, int64_t* shard);

/* ---------------------------------------------------------------------------------------
 * Data-parallel collectives of north_star (d) as standalone entry points (the executor issues
 * the same calls internally). The reference has no multi-GPU path; these realise
 * the per-block exchange around its ops: the all-gather before a block's first use in F / R / B
 * (bf16 params, after ParamPrefetch / materialisation, simulator.hpp:16-32) and the
 * reduce-scatter after its Backward (bf16 grads, before GradOffload / GpuOptim). NCCL over
 * NVLink / NVSwitch; one communicator per rank (device = the caller's current device).
 * --------------------------------------------------------------------------------------- */
/* nccl_id: 128 bytes from ah_dp_unique_id on rank 0, broadcast by the caller. Setup call. */
int ah_nccl_comm_create(const uint8_t* nccl_id, int32_t nranks, int32_t rank, void** comm);
int ah_nccl_comm_destroy(void* comm);
/* bf16 SUM over ranks of send [nranks * count] -> recv [count] = this rank's shard (the grads of
 * elements [rank*count, (rank+1)*count)); in place when recv == send + rank * count. */
int ah_nccl_reduce_scatter_bf16(const uint16_t* send, uint16_t* recv, size_t count, void* comm, void* stream);
/* send [count] (this rank's shard) -> recv [nranks * count]; in place when send == recv + rank * count. */
int ah_nccl_all_gather_bf16(const uint16_t* send, uint16_t* recv, size_t count, void* comm, void* stream);
/* In-place SUM all-reduce of the replicated groups' grads; dtype 0 = fp32, 1 = bf16. */
int ah_nccl_all_reduce(void* buf, size_t count, int32_t dtype, void* comm, void* stream);

typedef struct ah_trainer_stats {
    int32_t c_hat, p_hat, o_hat;
    double activation_coef;       /* real bytes of a block's activations / (2*b*s*h) */
    int64_t m_p, m_gc;            /* per-block params, constant GPU residue (bytes) */
    int64_t modeled_peak_bytes;   /* Eq.(1) for the chosen strategy */
    int64_t simulated_peak_bytes; /* hetsim::run peak */
    int64_t pool_peak_bytes;      /* measured: default stream-ordered pool high watermark (the executor's
                                   * transient buffers come from its fixed arenas: ~0) */
    int64_t static_bytes;         /* measured: persistent device allocations */
    double sim_steady_s;          /* hetsim::run steady-state iteration time */
    double lane_busy_ms[4];       /* compute, h2d, d2h, cpu: summed op time since reset */
    int32_t lane_ops[4];
    int64_t h2d_bytes, d2h_bytes; /* host-link bytes per iteration: parameter prefetch / grad offload */
    int32_t kernels_per_iter;     /* our kernel launches per iteration */
    /* Offload overlap over the last drained window (CUDA-event timestamps): compute-lane time
     * spent waiting for a ParamPrefetch / GradOffload / CpuOptim dependency, and the busy time
     * of the copy lanes. hidden = 1 - blocked / (h2d + d2h busy). */
    double window_iters, compute_busy_ms, h2d_busy_ms, d2h_busy_ms, offload_blocked_ms;
    double h2d_gbps, d2h_gbps; /* achieved host-link bandwidth of the copy ops */
    /* offload_blocked_ms split: time the compute lane waited while the needed copy was running
     * (copy_blocked_ms) vs before it had started — held up upstream by the CPU optimizer or the
     * copy lane's own order (upstream_blocked_ms). hidden = 1 - copy_blocked / (h2d + d2h busy). */
    double copy_blocked_ms, upstream_blocked_ms;
    double cpu_busy_ms; /* CpuOptim host time of the window's iterations */
    double window_ms;   /* compute-stream span of the window (first op start -> last op end) */
    double sim_steady_fifo_s, sim_steady_ps_s; /* reference scheduler, both orders of this plan */
    int32_t priority_sched;                    /* order the executor currently runs */
    /* Gradient statistics of the last drained iteration (this rank's gradients): global norm,
     * non-finite count, and block groups whose update was skipped because a gradient was
     * inf / nan (per-block overflow check: the pipelined schedule updates block L before block
     * 1's gradients exist, so the skip is per block group, not per step). */
    double grad_norm;
    int64_t nonfinite_grads;
    int32_t skipped_updates;
    /* the reference scheduler's per-lane busy time of one steady-state iteration (compute, h2d,
     * d2h, cpu; ms) for the plan and order in use — the simulated counterpart of lane_busy_ms */
    double sim_lane_busy_ms[4];
    /* sub-block streaming of the offload chain GradOffload -> CpuOptim -> ParamPrefetch: chunks
     * per block vector (1 = whole-block ops; env AH_STREAM_CHUNK_MB sets the chunk size, 16 MB
     * of bf16 by default, 0 = off) */
    int32_t stream_chunks;
    /* the stream-ordered pool's physically reserved bytes now (it grows when a transient
     * allocation pattern outruns the reservation made at create) */
    int64_t pool_reserved_bytes;
    /* host time the compute lane thread spent enqueueing compute ops since the last reset (sum,
     * max over ops): a stalled enqueue (CPU starvation, a pool growth in cudaMallocAsync) leaves
     * the GPU idle inside an op */
    double compute_enqueue_ms, compute_enqueue_max_ms;
    /* block weight / gradient buffers served by the stream-ordered pool because every slot of the
     * fixed buffer arena (sized by the simulated transient peak) was live (expected 0) */
    int32_t buffer_overflows;
} ah_trainer_stats;

int ah_trainer_create(const ah_trainer_config* cfg, void** trainer);
int ah_trainer_destroy(void* trainer);
/* Async: enqueue one iteration; inputs are B*s int32 on host (or device if on_device). */
int ah_trainer_submit(void* trainer, const int32_t* tokens, const int32_t* targets, int32_t on_device);
/* Wait for all submitted iterations; *loss = mean loss of the last one. */
int ah_trainer_drain(void* trainer, float* loss);
/* Synchronous e2e step: H2D inputs, iteration, D2H loss. */
int ah_trainer_step(void* trainer, const int32_t* tokens, const int32_t* targets, float* loss);
int ah_trainer_stats_get(void* trainer, ah_trainer_stats* out);
int ah_trainer_reset_stats(void* trainer);
/* Run subsequent iterations in the priority-based (1, paper §3.3) or FIFO (0) per-lane order of
 * the reference scheduler (simulator.cpp:413-450) for the same plan; drains first. */
int ah_trainer_set_schedule(void* trainer, int32_t priority_sched);
/* Per-lane op order of one steady-state iteration as "LANE:OP_block" tokens. */
int ah_trainer_schedule(void* trainer, char* buf, size_t cap);
/* fp32 master parameters of block b (1..L), 0 = token embedding, -1 = positions,
 * -2 = final LayerNorm; n = element count written to out (host). */
int ah_trainer_read_master(void* trainer, int32_t block, float* out, size_t n);
int64_t ah_trainer_master_size(void* trainer, int32_t block);
/* Optimizer-state checkpoint (fp32 master / m / v of every block and of the embedding state,
 * plus the step counter), independent of the plan: load under a different (c, p, o) works.
 * Load only into a freshly created trainer with the same model shape and dp layout. */
int ah_trainer_save(void* trainer, const char* path);
int ah_trainer_load(void* trainer, const char* path);
int ah_trainer_trace(void* trainer, char* buf, size_t cap); /* Chrome trace JSON, measured */
/* Measured GPU-memory timeline of the last drained iterations in the reference's CSV schema
 * ("time_us,gpu_bytes", simulator.cpp:615-622): persistent allocations + the executor's
 * transient buffers taken at each op's start / returned at its end (CUDA-event times).
 * Returns the bytes needed (incl. NUL) like ah_trainer_trace; *peak_bytes (nullable) = max. */
int ah_trainer_memory_csv(void* trainer, char* buf, size_t cap, int64_t* peak_bytes);
/* Device-timed region on the executor's compute stream: stop=0 drains then records the
 * start event; stop=1 drains all lanes, records the stop event and returns elapsed ms. */
int ah_trainer_timer(void* trainer, int32_t stop, float* ms);

/* ---------------------------------------------------------------------------------------
 * Runtime profiler (paper §3.1): measures one block on this box and
 * returns the HardwareSpec rates the planner consumes. Reference counterpart: the analytic
 * estimate_block_times (proj/core/src/workload.cpp:55-73), which this replaces.
 * --------------------------------------------------------------------------------------- */
/* GPU times are taken after >= 1 s of back-to-back block forward + backward (the power-capped
 * sustained clock a training step runs at, not the idle-GPU boost clock). The reference model
 * has per-block times only (workload.cpp:55-73), so the per-iteration work outside the blocks —
 * embedding forward / backward, final LayerNorm, LM-head GEMMs, cross-entropy, the embedding
 * group's AdamW — is measured on the real shapes and folded into every block's time as a 1/L
 * share: L * t_fwd_s + L * t_bwd_s is the whole compute-lane iteration. */
typedef struct ah_hw_profile {
    double t_fwd_s, t_bwd_s;  /* per block incl. the 1/L share of non-block work (what the planner uses) */
    double gpu_flops;         /* (2*m_p*b*s + 4*b*s^2*h) / t_fwd_s, workload.cpp:63 */
    double bwd_fwd_ratio;     /* t_bwd_s / t_fwd_s -> ModelSpec::bwd_fwd_ratio */
    double h2d_bw, d2h_bw;    /* pinned 2*m_p-byte copies, B/s */
    double gpu_adam_rate;     /* params/s, fused sm_100a AdamW */
    double cpu_adam_rate;     /* params/s, host AdamW with cfg->cpu_threads over >= 2 GB of distinct
                               * block states (DRAM-resident, as in the step), median of 3 passes */
    double t_block_fwd_s, t_block_bwd_s;        /* the block alone (sustained clock) */
    double t_nonblock_fwd_s, t_nonblock_bwd_s;  /* per iteration, outside the blocks */
} ah_hw_profile;
int ah_profile_block(const ah_trainer_config* cfg, ah_hw_profile* out);

/* In-step calibration (profiler fidelity): the per-block durations the running trainer actually
 * achieved over its last drained iterations — means over the window of F, B, GpuOptim ops
 * (CUDA events; F / B include the 1/L share of embedding / head work the blocks carry),
 * ParamPrefetch / GradOffload copies of optimizer-offloaded blocks, and CpuOptim (host clock) —
 * put into the reference cost model: sim_steady_s = hetsim::run of the running plan with them;
 * (c_hat, p_hat, o_hat) = the plan hetsim::solve (+ fine_tune_prefetch) picks with them
 * (single-GPU trainers; -1 under DP) and sim_steady_replan_s its simulated iteration. */
typedef struct ah_calibration {
    double t_fwd_s, t_bwd_s, t_recompute_s;   /* per block (0 if no op of that kind ran) */
    double t_h2d_s, t_d2h_s, t_opt_cpu_s, t_opt_gpu_s;
    double sim_steady_s;
    int32_t c_hat, p_hat, o_hat;
    double sim_steady_replan_s;
    double sim_steady_other_s; /* the running plan in the OTHER order (FIFO if PS runs, PS if FIFO) */
    /* the durations as HardwareSpec / ModelSpec rates (inverse of estimate_block_times) */
    double gpu_flops, bwd_fwd_ratio, h2d_bw, d2h_bw, cpu_adam_rate, gpu_adam_rate;
} ah_calibration;
int ah_trainer_calibrate(void* trainer, ah_calibration* out);
/* Plan on the last calibration (the paper's profiler measures by executing):
 * if the reference planner keeps the running (c_hat, p_hat, o_hat) with the calibrated rates — or
 * keep_strategy != 0 — the trainer adopts the calibrated profile, lookaheads and per-lane order in
 * place (drains first; memory layout unchanged) and *applied = 1; otherwise nothing changes and
 * *applied = 0 (a different plan needs a new trainer built from the calibrated rates).
 * Single-GPU trainers only. */
int ah_trainer_apply_calibration(void* trainer, int32_t keep_strategy, int32_t* applied);

/* Host side of the profiler: the CpuOptim lane's roofline on this host. n params of pinned
 * 14 B/param state (allocated and freed inside: a setup call); stream_gbps = best in-place pass
 * over p/m/v (fp32) and g (bf16) with trivial arithmetic (the 28 B/param pattern of the host
 * AdamW), adam_gbps / adam_params_per_s = ah_cpu_adam on the same buffers. */
typedef struct ah_host_profile {
    double stream_gbps, adam_gbps, adam_params_per_s;
    int32_t threads;
} ah_host_profile;
int ah_profile_host(size_t n, int32_t nthreads, ah_host_profile* out);

/* Instrumentation for the bench: kernels launched by this library so far, and live GEMM
 * timing (enable=1 starts recording; enable=0 stops and returns totals since enabling). */
int64_t ah_kernel_launches(void);
int ah_gemm_timing(int32_t enable, double* total_ms, double* total_flops, int64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* AUTOHETE_H */
