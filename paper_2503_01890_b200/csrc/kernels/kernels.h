// Internal launcher interface between the C-ABI / runtime and the sm_100a kernels.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace ah {

// Host-precomputed AdamW scalars (see derive_adam_scalars in csrc/runtime/adam_scalars.h).
struct AdamArgs {
    float* p = nullptr;
    float* m = nullptr;
    float* v = nullptr;
    const uint16_t* g = nullptr;
    uint16_t* p_bf16 = nullptr;  // nullable
    size_t n = 0;
    float decay, beta1, one_minus_beta1, beta2, one_minus_beta2, step_size, inv_sqrt_bc2, eps;
    float inv_scale = 1.f;
    const int* skip = nullptr;   // nullable device flag
    float* stats = nullptr;      // nullable AH_STATS_FLOATS buffer (include/autohete.h)
};

cudaError_t launch_adam(const AdamArgs& a, cudaStream_t stream);
// dst[i] = sum over q < n (in order) of srcs[q][i] (loopback collectives): fp32 accumulation, or
// (ring, bf16) NCCL ring's per-hop bf16 rounding of the running partial.
cudaError_t launch_sum_ranks(void* dst, const void* const* srcs, int n, size_t count, bool f32, cudaStream_t st,
                             bool ring = false);
cudaError_t launch_cast_f32_bf16(const float* src, uint16_t* dst, size_t n, cudaStream_t stream);
cudaError_t launch_grad_stats(const uint16_t* g, size_t n, float inv_scale, float* stats,
                              cudaStream_t stream);

}  // namespace ah

#include <atomic>
#include <utility>
namespace ah {
// Number of kernels this library has launched (for the bench's gpu_launches claim).
inline std::atomic<long long>& kernel_launch_counter() {
    static std::atomic<long long> c{0};
    return c;
}
inline cudaError_t launched(int n) {
    kernel_launch_counter().fetch_add(n, std::memory_order_relaxed);
    return cudaGetLastError();
}

// Programmatic dependent launch (on unless AH_PDL=0): kernels whose every global-memory access
// follows pdl_wait() (common.cuh) are launched with programmatic stream serialisation, so their
// launch and prologue (barrier init, TMEM allocation, tensor-map prefetch) overlap the tail of
// the previous kernel on the stream instead of following its completion.
bool pdl_enabled();

#ifdef __CUDACC__
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                      Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (cluster > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = cluster;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    if (pdl_enabled()) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);  // callers count via launched()
}
#endif
}  // namespace ah
