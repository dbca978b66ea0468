// hetsim::core drop-in — op DAG of one iteration and the four-lane discrete-event
// scheduler (FIFO or priority-based). Mirrors
// /root/reference/proj/core/include/hetsim/simulator.hpp:16-178. The B200 executor
// (paper_2503_01890_b200/csrc/runtime) realises exactly these ops on CUDA streams and a
// host worker, in the per-lane order this scheduler produces.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <queue>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hetsim/costmodel.hpp"
#include "hetsim/workload.hpp"

namespace hetsim {

enum class OpKind {
    Forward,
    Backward,
    Recompute,
    GpuOptim,
    ParamPrefetch,
    GradOffload,
    CpuOptim,
};

enum class StreamId : int {
    Compute = 1,
    H2D = 2,
    D2H = 3,
    Cpu = 4,
};

StreamId stream_of(OpKind kind);
const char* op_code(OpKind kind);
const char* stream_name(StreamId id);

struct OpRef {
    OpKind kind;
    int block = 0;
    int iter = 0;
    bool backward_copy = false;

    friend bool operator==(const OpRef&, const OpRef&) = default;
};

struct StreamOp {
    OpKind kind;
    int block = 0;
    int iter = 0;
    bool backward_copy = false;
    double duration = 0.0;
    std::vector<OpRef> deps;                  // finish-before-start
    std::vector<OpRef> start_after_start_of;  // start-before-start
    std::int64_t alloc_at_start = 0;
    std::int64_t release_at_end = 0;

    StreamId stream() const { return stream_of(kind); }
    OpRef ref() const { return {kind, block, iter, backward_copy}; }
};

struct MemoryTracker {
    std::int64_t current = 0;
    std::int64_t peak = 0;
    std::int64_t budget = 0;
    std::vector<std::pair<double, std::int64_t>> timeline;

    void record(double time, std::int64_t delta);
};

struct PriorityQueues {
    using MinHeap = std::priority_queue<int, std::vector<int>, std::greater<int>>;
    MinHeap pq_d2h;
    MinHeap pq_opt;
};

bool memory_guard(const MemoryTracker& tracker, std::int64_t alloc_bytes,
                  std::int64_t pending_grad_bytes);

struct CompletedOp {
    OpKind kind;
    int block = 0;
    int iter = 0;
    bool backward_copy = false;
    StreamId stream = StreamId::Compute;
    double start = 0.0;
    double end = 0.0;
};

struct SimResult {
    std::vector<double> iter_times;
    double steady_state_time = 0.0;
    std::int64_t peak_gpu = 0;
    std::vector<CompletedOp> trace;  // in completion order
    std::vector<std::pair<double, std::int64_t>> mem_timeline;
    double throughput = 0.0;
};

class MemoryExceededError : public std::runtime_error {
public:
    MemoryExceededError(const std::string& what, OpRef op, double time,
                        std::int64_t attempted, std::int64_t budget);
    OpRef op() const { return op_; }
    double time() const { return time_; }
    std::int64_t attempted_bytes() const { return attempted_; }
    std::int64_t budget_bytes() const { return budget_; }

private:
    OpRef op_;
    double time_;
    std::int64_t attempted_;
    std::int64_t budget_;
};

std::vector<StreamOp> build_iteration_ops(const ModelProfile& profile,
                                          const Strategy& s, int iter);

SimResult run(const ModelProfile& profile, const Strategy& s,
              const HardwareSpec& hw, int n_iters, bool priority_sched);

void write_chrome_trace(std::ostream& out, const std::vector<CompletedOp>& trace);

void write_memory_csv(std::ostream& out,
                      const std::vector<std::pair<double, std::int64_t>>& timeline);

}  // namespace hetsim
