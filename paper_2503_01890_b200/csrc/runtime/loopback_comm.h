// In-process loopback communicator: N trainers (ranks) sharing ONE GPU exchange data with the
// same in-place collective semantics the executor gets from NCCL (all-gather of bf16 shards,
// reduce-scatter sum of bf16 gradients, all-reduce sum of f32 / bf16). It exists so the data
// parallel path — shard offsets, 1/N gradient scaling, replicated-embedding all-reduce and the
// side-stream ordering of every collective — can be executed end to end on a single-GPU box
// (NCCL refuses two ranks on one device). Not a transport: everything is device memcpy / a
// fixed-order sum kernel on one internal stream. The bf16 reduce-scatter reproduces NCCL's ring
// algorithm (chunk r accumulated from rank r+1 around the ring to r, bf16 rounding per hop); the
// all-reduces accumulate in fp32 and round once.
//
// Rendezvous: each rank numbers its collective calls; call k blocks the calling host thread
// until every rank has posted call k (with an event marking its inputs ready on its stream);
// the last poster enqueues the data movement on the internal stream after all posters'
// events and records a done event, which every rank's stream then waits on.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

namespace ah {

class LoopbackComm {
public:
    enum Op { kAllGatherBf16, kReduceScatterBf16, kAllReduceF32, kAllReduceBf16 };
    explicit LoopbackComm(int nranks);
    ~LoopbackComm();
    int size() const { return n_; }
    // buf: this rank's buffer; count: shard elements (gather / scatter) or total elements
    // (all-reduce); stream: the rank's stream (inputs ready on it, outputs awaited on it).
    cudaError_t call(int rank, Op op, void* buf, size_t count, cudaStream_t stream);

private:
    struct Post {
        void* buf = nullptr;
        cudaEvent_t ready = nullptr;
    };
    struct Slot {
        Op op;
        size_t count = 0;
        std::vector<Post> posts;
        int posted = 0, consumed = 0;
        bool done = false;
        cudaError_t err = cudaSuccess;
        cudaEvent_t done_ev = nullptr;
    };
    cudaError_t perform(Slot& s);
    int n_;
    cudaStream_t stream_ = nullptr;
    std::mutex mu_;
    std::condition_variable cv_;
    std::vector<long long> seq_;     // per-rank next call number
    std::map<long long, Slot> slots_;
    void* scratch_ = nullptr;        // device array of source pointers for the sum kernel
};

}  // namespace ah
