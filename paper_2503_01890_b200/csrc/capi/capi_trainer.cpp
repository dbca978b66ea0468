// extern "C" boundary of the training executor (include/autohete.h, "Training executor").
#include <cstring>
#include <stdexcept>
#include <string>

#include "autohete.h"
#include "../runtime/executor.h"
#include "capi_util.h"
#include "hetsim/planner.hpp"
#include "hetsim/simulator.hpp"

namespace {

template <class F>
int guarded(F&& f) {
    int rc = AH_OK;
    try {
        f();
    } catch (const hetsim::InfeasibleError& e) {
        rc = ah::set_error(AH_ERR_INFEASIBLE, e.what());
    } catch (const hetsim::MemoryExceededError& e) {
        rc = ah::set_error(AH_ERR_MEMORY, e.what());
    } catch (const std::invalid_argument& e) {
        rc = ah::set_error(AH_ERR_INVALID, e.what());
    } catch (const std::exception& e) {
        const std::string w = e.what();
        rc = ah::set_error(w.find("CUDA") != std::string::npos || w.find("cuda") != std::string::npos ? AH_ERR_CUDA
                                                                                                       : AH_ERR_INTERNAL,
                           w);
    }
    if (rc != AH_OK) cudaGetLastError();  // reported here; keep it out of later launch checks
    return rc;
}

ah::Trainer* T(void* p) { return static_cast<ah::Trainer*>(p); }

int copy_out(const std::string& s, char* buf, size_t cap) {
    if (!buf || cap == 0) return (int)s.size() + 1;
    const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
    return (int)s.size() + 1;
}

}  // namespace

extern "C" {

int ah_trainer_create(const ah_trainer_config* cfg, void** out) {
    if (!cfg || !out) return ah::set_error(AH_ERR_INVALID, "ah_trainer_create: null argument");
    return guarded([&] { *out = new ah::Trainer(*cfg); });
}

int ah_trainer_destroy(void* tr) {
    return guarded([&] { delete T(tr); });
}

int ah_trainer_submit(void* tr, const int32_t* tokens, const int32_t* targets, int32_t on_device) {
    if (!tr || !tokens || !targets) return ah::set_error(AH_ERR_INVALID, "ah_trainer_submit: null argument");
    return guarded([&] { T(tr)->submit(tokens, targets, on_device != 0); });
}

int ah_trainer_drain(void* tr, float* loss) {
    if (!tr) return ah::set_error(AH_ERR_INVALID, "ah_trainer_drain: null trainer");
    return guarded([&] {
        const float l = T(tr)->drain();
        if (loss) *loss = l;
    });
}

int ah_trainer_step(void* tr, const int32_t* tokens, const int32_t* targets, float* loss) {
    if (!tr || !tokens || !targets) return ah::set_error(AH_ERR_INVALID, "ah_trainer_step: null argument");
    return guarded([&] {
        const float l = T(tr)->step(tokens, targets);
        if (loss) *loss = l;
    });
}

int ah_trainer_stats_get(void* tr, ah_trainer_stats* out) {
    if (!tr || !out) return ah::set_error(AH_ERR_INVALID, "ah_trainer_stats_get: null argument");
    return guarded([&] { T(tr)->stats(out); });
}

int ah_trainer_reset_stats(void* tr) {
    if (!tr) return ah::set_error(AH_ERR_INVALID, "null trainer");
    return guarded([&] { T(tr)->reset_stats(); });
}

int ah_trainer_calibrate(void* tr, ah_calibration* out) {
    if (!tr || !out) return ah::set_error(AH_ERR_INVALID, "ah_trainer_calibrate: null argument");
    return guarded([&] { T(tr)->calibrate(out); });
}

int ah_trainer_apply_calibration(void* tr, int32_t keep_strategy, int32_t* applied) {
    if (!tr) return ah::set_error(AH_ERR_INVALID, "null trainer");
    return guarded([&] {
        const bool a = T(tr)->apply_calibration(keep_strategy != 0);
        if (applied) *applied = a ? 1 : 0;
    });
}

int ah_trainer_set_schedule(void* tr, int32_t priority_sched) {
    if (!tr) return ah::set_error(AH_ERR_INVALID, "null trainer");
    return guarded([&] { T(tr)->set_schedule(priority_sched != 0); });
}

int ah_trainer_schedule(void* tr, char* buf, size_t cap) {
    if (!tr) return ah::set_error(AH_ERR_INVALID, "null trainer");
    std::string s;
    const hetsim::SimResult& r = T(tr)->simulated();
    for (const auto& op : r.trace) {
        if (op.iter != 2) continue;
        s += std::string(hetsim::stream_name(op.stream)) + ":" + hetsim::op_code(op.kind) + "_" +
             std::to_string(op.block) + (op.backward_copy ? "b" : "") + " ";
    }
    return copy_out(s, buf, cap);
}

int ah_trainer_read_master(void* tr, int32_t block, float* out, size_t n) {
    if (!tr || !out) return ah::set_error(AH_ERR_INVALID, "null argument");
    return guarded([&] { T(tr)->read_master(block, out, n); });
}

int64_t ah_trainer_master_size(void* tr, int32_t block) {
    if (!tr) return -1;
    return (int64_t)T(tr)->master_size(block);
}

int ah_trainer_trace(void* tr, char* buf, size_t cap) {
    if (!tr) return ah::set_error(AH_ERR_INVALID, "null trainer");
    std::string s;
    const int rc = guarded([&] { s = T(tr)->trace_json(); });
    if (rc != AH_OK) return rc;
    return copy_out(s, buf, cap);
}

int ah_trainer_memory_csv(void* tr, char* buf, size_t cap, int64_t* peak_bytes) {
    if (!tr) return ah::set_error(AH_ERR_INVALID, "null trainer");
    std::string s;
    const int rc = guarded([&] { s = T(tr)->memory_csv(peak_bytes); });
    if (rc != AH_OK) return rc;
    return copy_out(s, buf, cap);
}

}  // extern "C"

namespace ah {
ah_hw_profile profile_block(const ah_trainer_config& cfg);
}

extern "C" {

int ah_trainer_timer(void* tr, int32_t stop, float* ms) {
    if (!tr) return ah::set_error(AH_ERR_INVALID, "null trainer");
    return guarded([&] {
        const float v = T(tr)->timer(stop != 0);
        if (ms) *ms = v;
    });
}

int ah_profile_block(const ah_trainer_config* cfg, ah_hw_profile* out) {
    if (!cfg || !out) return ah::set_error(AH_ERR_INVALID, "ah_profile_block: null argument");
    return guarded([&] { *out = ah::profile_block(*cfg); });
}

}  // extern "C"

#include <nccl.h>

#include "../runtime/loopback_comm.h"

extern "C" {

int ah_dp_unique_id(uint8_t* out) {
    if (!out) return ah::set_error(AH_ERR_INVALID, "ah_dp_unique_id: null out");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return ah::set_error(AH_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out, &id, sizeof(id));
    return AH_OK;
}

int ah_dp_loopback_create(int32_t nranks, void** comm) {
    if (!comm) return ah::set_error(AH_ERR_INVALID, "ah_dp_loopback_create: null out");
    try {
        *comm = new ah::LoopbackComm(nranks);
    } catch (const std::exception& e) {
        return ah::set_error(AH_ERR_INVALID, std::string("ah_dp_loopback_create: ") + e.what());
    }
    return AH_OK;
}

int ah_dp_loopback_call(void* comm, int32_t rank, int32_t op, void* buf, size_t count, void* stream) {
    if (!comm || !buf || op < 0 || op > 3) return ah::set_error(AH_ERR_INVALID, "ah_dp_loopback_call: bad argument");
    return ah::cuda_status(static_cast<ah::LoopbackComm*>(comm)->call(rank, static_cast<ah::LoopbackComm::Op>(op), buf,
                                                                      count, static_cast<cudaStream_t>(stream)),
                           "ah_dp_loopback_call");
}

int ah_dp_loopback_destroy(void* comm) {
    delete static_cast<ah::LoopbackComm*>(comm);
    return AH_OK;
}

namespace {
int nccl_status(ncclResult_t r, const char* where) {
    if (r == ncclSuccess) return AH_OK;
    return ah::set_error(AH_ERR_NCCL, std::string(where) + ": " + ncclGetErrorString(r));
}
ncclComm_t C_(void* c) { return static_cast<ncclComm_t>(c); }
}  // namespace

int ah_nccl_comm_create(const uint8_t* nccl_id, int32_t nranks, int32_t rank, void** comm) {
    if (!nccl_id || !comm || nranks < 1 || rank < 0 || rank >= nranks)
        return ah::set_error(AH_ERR_INVALID, "ah_nccl_comm_create: bad argument");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclComm_t c = nullptr;
    const int rc = nccl_status(ncclCommInitRank(&c, nranks, id, rank), "ncclCommInitRank");
    if (rc == AH_OK) *comm = c;
    return rc;
}

int ah_nccl_comm_destroy(void* comm) {
    if (!comm) return ah::set_error(AH_ERR_INVALID, "ah_nccl_comm_destroy: null comm");
    return nccl_status(ncclCommDestroy(C_(comm)), "ncclCommDestroy");
}

int ah_nccl_reduce_scatter_bf16(const uint16_t* send, uint16_t* recv, size_t count, void* comm, void* stream) {
    if (!send || !recv || !comm) return ah::set_error(AH_ERR_INVALID, "ah_nccl_reduce_scatter_bf16: null argument");
    return nccl_status(ncclReduceScatter(send, recv, count, ncclBfloat16, ncclSum, C_(comm),
                                         static_cast<cudaStream_t>(stream)),
                       "ncclReduceScatter");
}

int ah_nccl_all_gather_bf16(const uint16_t* send, uint16_t* recv, size_t count, void* comm, void* stream) {
    if (!send || !recv || !comm) return ah::set_error(AH_ERR_INVALID, "ah_nccl_all_gather_bf16: null argument");
    return nccl_status(ncclAllGather(send, recv, count, ncclBfloat16, C_(comm), static_cast<cudaStream_t>(stream)),
                       "ncclAllGather");
}

int ah_nccl_all_reduce(void* buf, size_t count, int32_t dtype, void* comm, void* stream) {
    if (!buf || !comm || (dtype != 0 && dtype != 1)) return ah::set_error(AH_ERR_INVALID, "ah_nccl_all_reduce: bad argument");
    return nccl_status(ncclAllReduce(buf, buf, count, dtype ? ncclBfloat16 : ncclFloat32, ncclSum, C_(comm),
                                     static_cast<cudaStream_t>(stream)),
                       "ncclAllReduce");
}

int ah_dp_shard(int64_t n, int32_t rank, int32_t dp_size, int64_t* offset, int64_t* len, int64_t* shard) {
    if (n < 0 || dp_size < 1 || rank < 0 || rank >= dp_size || !offset || !len || !shard)
        return ah::set_error(AH_ERR_INVALID, "ah_dp_shard: bad argument");
    const int64_t per = ((n + dp_size - 1) / dp_size + 7) / 8 * 8;
    const int64_t off = per * rank;
    *shard = per;
    *offset = off;
    *len = off >= n ? 0 : (n - off < per ? n - off : per);
    return AH_OK;
}

}  // extern "C"
