// In-process loopback communicator (loopback_comm.h).
#include "loopback_comm.h"

#include <stdexcept>
#include <string>

#include "../kernels/kernels.h"

namespace ah {

LoopbackComm::LoopbackComm(int nranks) : n_(nranks), seq_((size_t)nranks, 0) {
    if (nranks < 1 || nranks > 8) throw std::invalid_argument("loopback comm: 1..8 ranks");
    if (cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking) != cudaSuccess)
        throw std::runtime_error("loopback comm: stream");
}

LoopbackComm::~LoopbackComm() {
    cudaStreamSynchronize(stream_);
    for (auto& kv : slots_) {
        for (Post& p : kv.second.posts)
            if (p.ready) cudaEventDestroy(p.ready);
        if (kv.second.done_ev) cudaEventDestroy(kv.second.done_ev);
    }
    cudaStreamDestroy(stream_);
}

cudaError_t LoopbackComm::perform(Slot& s) {
    cudaError_t e = cudaSuccess;
    for (Post& p : s.posts)
        if (e == cudaSuccess) e = cudaStreamWaitEvent(stream_, p.ready, 0);
    const size_t c = s.count;
    switch (s.op) {
        case kAllGatherBf16:  // rank r's shard [r*c, (r+1)*c) -> every other rank's buffer
            for (int r = 0; r < n_ && e == cudaSuccess; ++r)
                for (int q = 0; q < n_ && e == cudaSuccess; ++q)
                    if (q != r)
                        e = cudaMemcpyAsync(static_cast<uint16_t*>(s.posts[(size_t)q].buf) + (size_t)r * c,
                                            static_cast<uint16_t*>(s.posts[(size_t)r].buf) + (size_t)r * c, c * 2,
                                            cudaMemcpyDeviceToDevice, stream_);
            break;
        case kReduceScatterBf16: {  // chunk r, NCCL ring order: starts at rank r+1, hops r+2 .. r-1,
            // ends at its owner r; each hop rounds the running partial to bf16 -> rank r's chunk r
            for (int r = 0; r < n_ && e == cudaSuccess; ++r) {
                const void* src[8];
                for (int k = 0; k < n_; ++k) {
                    const int q = (r + 1 + k) % n_;
                    src[k] = static_cast<uint16_t*>(s.posts[(size_t)q].buf) + (size_t)r * c;
                }
                e = launch_sum_ranks(static_cast<uint16_t*>(s.posts[(size_t)r].buf) + (size_t)r * c, src, n_, c, false,
                                     stream_, /*ring=*/true);
            }
            break;
        }
        case kAllReduceF32:
        case kAllReduceBf16: {  // sum into rank 0's buffer, then broadcast
            const bool f32 = s.op == kAllReduceF32;
            const void* src[8];
            for (int q = 0; q < n_; ++q) src[q] = s.posts[(size_t)q].buf;
            e = launch_sum_ranks(s.posts[0].buf, src, n_, c, f32, stream_);
            for (int q = 1; q < n_ && e == cudaSuccess; ++q)
                e = cudaMemcpyAsync(s.posts[(size_t)q].buf, s.posts[0].buf, c * (f32 ? 4 : 2), cudaMemcpyDeviceToDevice,
                                    stream_);
            break;
        }
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.done_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(s.done_ev, stream_);
    return e;
}

cudaError_t LoopbackComm::call(int rank, Op op, void* buf, size_t count, cudaStream_t stream) {
    if (rank < 0 || rank >= n_) return cudaErrorInvalidValue;
    cudaEvent_t ready = nullptr;
    cudaError_t e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ready, stream);
    if (e != cudaSuccess) return e;
    std::unique_lock<std::mutex> lk(mu_);
    const long long k = seq_[(size_t)rank]++;
    Slot& s = slots_[k];
    if (s.posts.empty()) {
        s.posts.resize((size_t)n_);
        s.op = op;
        s.count = count;
    } else if (s.op != op || s.count != count) {
        return cudaErrorInvalidValue;  // ranks disagree on the collective sequence
    }
    s.posts[(size_t)rank] = {buf, ready};
    if (++s.posted == n_) {
        s.err = perform(s);
        s.done = true;
        cv_.notify_all();
    } else {
        cv_.wait(lk, [&] { return s.done; });
    }
    e = s.err;
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, s.done_ev, 0);
    if (++s.consumed == n_) {  // every rank has its wait enqueued: retire the slot
        for (Post& p : s.posts) cudaEventDestroy(p.ready);
        cudaEventDestroy(s.done_ev);
        slots_.erase(k);
    }
    return e;
}

}  // namespace ah
