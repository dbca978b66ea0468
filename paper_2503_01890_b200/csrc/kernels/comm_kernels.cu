// Fixed-order sum of up to 8 rank buffers (the loopback communicator's reduction; see
// csrc/runtime/loopback_comm.h). fp32 accumulation in rank order; bf16 or fp32 in/out.
// dst may alias one of the sources (element-wise: every thread reads all inputs first).
#include "common.cuh"
#include "kernels.h"

namespace ah {
namespace {

struct Srcs {
    const void* p[8];
};

template <bool kF32>
__global__ void sum_ranks_kernel(void* dst, Srcs s, int n, size_t count) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        float a = 0.f;
        for (int q = 0; q < n; ++q)
            a += kF32 ? static_cast<const float*>(s.p[q])[i]
                      : bf16_bits_to_f32(static_cast<const uint16_t*>(s.p[q])[i]);
        if (kF32)
            static_cast<float*>(dst)[i] = a;
        else
            static_cast<uint16_t*>(dst)[i] = (uint16_t)f32_to_bf16_bits(a);
    }
}

}  // namespace

cudaError_t launch_sum_ranks(void* dst, const void* const* srcs, int n, size_t count, bool f32, cudaStream_t st) {
    if (n < 1 || n > 8) return cudaErrorInvalidValue;
    if (count == 0) return cudaSuccess;
    Srcs s{};
    for (int q = 0; q < n; ++q) s.p[q] = srcs[q];
    const size_t want = (count + 255) / 256;
    const int grid = (int)(want < (size_t)kNumSMs * 8 ? want : (size_t)kNumSMs * 8);
    if (f32)
        sum_ranks_kernel<true><<<grid, 256, 0, st>>>(dst, s, n, count);
    else
        sum_ranks_kernel<false><<<grid, 256, 0, st>>>(dst, s, n, count);
    return launched(1);
}

}  // namespace ah
