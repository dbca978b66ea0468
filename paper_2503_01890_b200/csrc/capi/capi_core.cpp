// extern "C" boundary: optimizer, cast and host-link entry points (include/autohete.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <omp.h>
#include <stdexcept>
#include <string>

#include "autohete.h"
#include "../kernels/kernels.h"
#include "../runtime/adam_scalars.h"
#include "capi_util.h"

namespace ah {
void cpu_adam(const ah_adam_hparams& hp, float* p, float* m, float* v, const uint16_t* g,
              uint16_t* p_bf16, std::size_t n, float inv_scale, int nthreads);
double host_stream_gbps(float* p, float* m, float* v, uint16_t* g, std::size_t n, int nthreads, int reps);
}

namespace ah {
thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return AH_OK;
    cudaGetLastError();  // reported here: do not let it resurface at the next launch check
    return set_error(AH_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
}  // namespace ah

using ah::cuda_status;
using ah::set_error;

extern "C" {

const char* ah_last_error(void) { return ah::g_last_error.c_str(); }
int ah_abi_version(void) { return 5; }

int ah_adam_step(const ah_adam_hparams* hp, float* p, float* m, float* v, const uint16_t* g,
                 uint16_t* p_bf16, size_t n, float inv_scale, const int32_t* skip_flag,
                 float* stats, void* stream) {
    if (!hp || (n && (!p || !m || !v || !g))) return set_error(AH_ERR_INVALID, "ah_adam_step: null argument");
    const ah::AdamConsts c = ah::derive_adam_scalars(*hp);
    ah::AdamArgs a;
    a.p = p;
    a.m = m;
    a.v = v;
    a.g = g;
    a.p_bf16 = p_bf16;
    a.n = n;
    a.decay = c.decay;
    a.beta1 = c.beta1;
    a.one_minus_beta1 = c.one_minus_beta1;
    a.beta2 = c.beta2;
    a.one_minus_beta2 = c.one_minus_beta2;
    a.step_size = c.step_size;
    a.inv_sqrt_bc2 = c.inv_sqrt_bc2;
    a.eps = c.eps;
    a.inv_scale = inv_scale;
    a.skip = skip_flag;
    a.stats = stats;
    return cuda_status(ah::launch_adam(a, static_cast<cudaStream_t>(stream)), "ah_adam_step");
}

int ah_grad_stats(const uint16_t* g, size_t n, float inv_scale, float* stats, void* stream) {
    if ((n && !g) || !stats) return set_error(AH_ERR_INVALID, "ah_grad_stats: null argument");
    return cuda_status(ah::launch_grad_stats(g, n, inv_scale, stats, static_cast<cudaStream_t>(stream)),
                       "ah_grad_stats");
}

int ah_cast_f32_bf16(const float* src, uint16_t* dst, size_t n, void* stream) {
    if (n && (!src || !dst)) return set_error(AH_ERR_INVALID, "ah_cast_f32_bf16: null argument");
    return cuda_status(ah::launch_cast_f32_bf16(src, dst, n, static_cast<cudaStream_t>(stream)),
                       "ah_cast_f32_bf16");
}

int ah_cpu_adam(const ah_adam_hparams* hp, float* p, float* m, float* v, const uint16_t* g,
                uint16_t* p_bf16, size_t n, float inv_scale, int nthreads) {
    if (!hp || (n && (!p || !m || !v || !g))) return set_error(AH_ERR_INVALID, "ah_cpu_adam: null argument");
    try {
        ah::cpu_adam(*hp, p, m, v, g, p_bf16, n, inv_scale, nthreads);
    } catch (const std::exception& e) {
        return set_error(AH_ERR_INTERNAL, e.what());
    }
    return AH_OK;
}

int ah_host_alloc(void** ptr, size_t bytes) {
    if (!ptr) return set_error(AH_ERR_INVALID, "ah_host_alloc: null out pointer");
    return cuda_status(cudaHostAlloc(ptr, bytes, cudaHostAllocPortable), "cudaHostAlloc");
}
int ah_host_free(void* ptr) { return cuda_status(cudaFreeHost(ptr), "cudaFreeHost"); }
int ah_host_register(void* ptr, size_t bytes) {
    return cuda_status(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable), "cudaHostRegister");
}
int ah_host_unregister(void* ptr) { return cuda_status(cudaHostUnregister(ptr), "cudaHostUnregister"); }

int ah_copy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
    return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice,
                                       static_cast<cudaStream_t>(stream)),
                       "ah_copy_h2d");
}
int ah_copy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
    return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost,
                                       static_cast<cudaStream_t>(stream)),
                       "ah_copy_d2h");
}

int ah_stream_create(void** stream, int high_priority) {
    if (!stream) return set_error(AH_ERR_INVALID, "ah_stream_create: null out pointer");
    int lo = 0, hi = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetStreamPriorityRange");
    cudaStream_t s;
    e = cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, high_priority ? hi : lo);
    if (e != cudaSuccess) return cuda_status(e, "cudaStreamCreateWithPriority");
    *stream = s;
    return AH_OK;
}
int ah_profile_host(size_t n, int32_t nthreads, ah_host_profile* out) {
    if (!out || n == 0) return set_error(AH_ERR_INVALID, "ah_profile_host: bad argument");
    if (nthreads <= 0) nthreads = omp_get_num_procs();
    float *p = nullptr, *m = nullptr, *v = nullptr;
    uint16_t* g = nullptr;
    cudaError_t e = cudaHostAlloc((void**)&p, n * 4, cudaHostAllocPortable);
    if (e == cudaSuccess) e = cudaHostAlloc((void**)&m, n * 4, cudaHostAllocPortable);
    if (e == cudaSuccess) e = cudaHostAlloc((void**)&v, n * 4, cudaHostAllocPortable);
    if (e == cudaSuccess) e = cudaHostAlloc((void**)&g, n * 2, cudaHostAllocPortable);
    int rc = AH_OK;
    if (e != cudaSuccess) {
        rc = cuda_status(e, "ah_profile_host: cudaHostAlloc");
    } else {
#pragma omp parallel for schedule(static) num_threads(nthreads)
        for (size_t i = 0; i < n; ++i) {
            p[i] = 0.01f;
            m[i] = 0.f;
            v[i] = 0.f;
            g[i] = 0x3c00;
        }
        out->threads = nthreads;
        out->stream_gbps = ah::host_stream_gbps(p, m, v, g, n, nthreads, 4);
        ah_adam_hparams hp{1e-4f, 0.9f, 0.999f, 1e-8f, 0.01f, 1};
        ah::cpu_adam(hp, p, m, v, g, g, n, 1.f, nthreads);  // warm
        double best = 1e30;
        for (int r = 0; r < 3; ++r) {
            hp.step = r + 2;
            const double t0 = omp_get_wtime();
            ah::cpu_adam(hp, p, m, v, g, g, n, 1.f, nthreads);
            best = std::min(best, omp_get_wtime() - t0);
        }
        out->adam_params_per_s = (double)n / best;
        out->adam_gbps = 28.0 * (double)n / best / 1e9;
    }
    for (void* q : {(void*)p, (void*)m, (void*)v, (void*)g})
        if (q) cudaFreeHost(q);
    return rc;
}

int ah_stream_destroy(void* stream) {
    return cuda_status(cudaStreamDestroy(static_cast<cudaStream_t>(stream)), "cudaStreamDestroy");
}

}  // extern "C"
