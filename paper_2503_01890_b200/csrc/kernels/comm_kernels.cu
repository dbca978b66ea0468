// Fixed-order sum of up to 8 rank buffers (the loopback communicator's reduction; see
// csrc/runtime/loopback_comm.h). bf16 or fp32 in/out, sources summed in the order given.
//   ring = false: fp32 accumulation, one rounding at the end;
//   ring = true (bf16): the per-hop rounding of NCCL's ring reduce-scatter — every hop adds the
//   incoming bf16 partial and the local bf16 value in fp32 and rounds the result to bf16, so the
//   loopback reproduces what NCCL's ring computes for the same source order.
// dst may alias one of the sources (element-wise: every thread reads all inputs first).
#include "common.cuh"
#include "kernels.h"

namespace ah {
namespace {

struct Srcs {
    const void* p[8];
};

template <bool kF32, bool kRing>
__global__ void sum_ranks_kernel(void* dst, Srcs s, int n, size_t count) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        float a = 0.f;
        for (int q = 0; q < n; ++q) {
            a += kF32 ? static_cast<const float*>(s.p[q])[i]
                      : bf16_bits_to_f32(static_cast<const uint16_t*>(s.p[q])[i]);
            if (kRing) a = bf16_bits_to_f32(f32_to_bf16_bits(a));  // the hop's bf16 partial
        }
        if (kF32)
            static_cast<float*>(dst)[i] = a;
        else
            static_cast<uint16_t*>(dst)[i] = (uint16_t)f32_to_bf16_bits(a);
    }
}

}  // namespace

cudaError_t launch_sum_ranks(void* dst, const void* const* srcs, int n, size_t count, bool f32, cudaStream_t st,
                             bool ring) {
    if (n < 1 || n > 8) return cudaErrorInvalidValue;
    if (count == 0) return cudaSuccess;
    Srcs s{};
    for (int q = 0; q < n; ++q) s.p[q] = srcs[q];
    const size_t want = (count + 255) / 256;
    const int grid = (int)(want < (size_t)kNumSMs * 8 ? want : (size_t)kNumSMs * 8);
    if (f32)
        sum_ranks_kernel<true, false><<<grid, 256, 0, st>>>(dst, s, n, count);
    else if (ring)
        sum_ranks_kernel<false, true><<<grid, 256, 0, st>>>(dst, s, n, count);
    else
        sum_ranks_kernel<false, false><<<grid, 256, 0, st>>>(dst, s, n, count);
    return launched(1);
}

}  // namespace ah
