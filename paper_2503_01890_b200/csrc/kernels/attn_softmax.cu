// Register-resident causal softmax forward / backward and a wider deterministic column-sum
// finish (second generation of the HBM-bound helpers of the attention and bias gradients).
// One warp per score row; the row (<= 2048 scores) is read from HBM exactly once with 16-byte
// vector loads, kept in registers for the max / sum / normalise passes, and written once.
#include "common.cuh"
#include "gpt_kernels.h"
#include "kernels.h"

namespace ah {
namespace gpt {
namespace {

constexpr int kMaxChunks = 16;  // float4 per lane -> rows up to 2048

template <int CH>
__global__ void __launch_bounds__(256) softmax_fwd_reg_kernel(const float* __restrict__ S, uint16_t* __restrict__ P,
                                                            long long rows, int s) {
    const long long gr = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (gr >= rows) return;
    const int i = (int)(gr % s);
    const float4* sr = reinterpret_cast<const float4*>(S + gr * s);
    float4 v[CH];
    float mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int q = c * 32 + lane;  // float4 index
        if (4 * q <= i) {
            v[c] = sr[q];
            const int j0 = 4 * q;
            if (j0 + 1 > i) v[c].y = -INFINITY;
            if (j0 + 2 > i) v[c].z = -INFINITY;
            if (j0 + 3 > i) v[c].w = -INFINITY;
        } else {
            v[c] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        }
        mx = fmaxf(mx, fmaxf(fmaxf(v[c].x, v[c].y), fmaxf(v[c].z, v[c].w)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        v[c].x = __expf(v[c].x - mx);
        v[c].y = __expf(v[c].y - mx);
        v[c].z = __expf(v[c].z - mx);
        v[c].w = __expf(v[c].w - mx);
        sum += (v[c].x + v[c].y) + (v[c].z + v[c].w);
    }
    const float inv = 1.f / warp_sum(sum);
    const int end = min(s, (i / 128 + 1) * 128);  // zero-fill to the end of i's 128-row tile
    uint2* pr = reinterpret_cast<uint2*>(P + gr * s);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int q = c * 32 + lane;
        if (4 * q < end)
            pr[q] = make_uint2(pack_bf16x2(v[c].x * inv, v[c].y * inv), pack_bf16x2(v[c].z * inv, v[c].w * inv));
    }
}

template <int CH>
__global__ void __launch_bounds__(256) softmax_bwd_reg_kernel(const uint16_t* __restrict__ P,
                                                            const float* __restrict__ dP,
                                                            uint16_t* __restrict__ dS, long long rows, int s) {
    const long long gr = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (gr >= rows) return;
    const int i = (int)(gr % s);
    const uint2* pr = reinterpret_cast<const uint2*>(P + gr * s);
    const float4* dr = reinterpret_cast<const float4*>(dP + gr * s);
    float4 p[CH], g[CH];
    float d = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int q = c * 32 + lane;
        if (4 * q <= i) {
            const uint2 w = pr[q];
            p[c] = make_float4(bf16_bits_to_f32(w.x & 0xffffu), bf16_bits_to_f32(w.x >> 16),
                               bf16_bits_to_f32(w.y & 0xffffu), bf16_bits_to_f32(w.y >> 16));
            g[c] = dr[q];
            const int j0 = 4 * q;  // P is exactly 0 above the diagonal; dP there is garbage
            if (j0 + 1 > i) g[c].y = 0.f;
            if (j0 + 2 > i) g[c].z = 0.f;
            if (j0 + 3 > i) g[c].w = 0.f;
        } else {
            p[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            g[c] = p[c];
        }
        d += (p[c].x * g[c].x + p[c].y * g[c].y) + (p[c].z * g[c].z + p[c].w * g[c].w);
    }
    d = warp_sum(d);
    const int end = min(s, (i / 128 + 1) * 128);
    uint2* out = reinterpret_cast<uint2*>(dS + gr * s);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int q = c * 32 + lane;
        if (4 * q < end)
            out[q] = make_uint2(pack_bf16x2(p[c].x * (g[c].x - d), p[c].y * (g[c].y - d)),
                                pack_bf16x2(p[c].z * (g[c].z - d), p[c].w * (g[c].w - d)));
    }
}

// out[n] = sum_{r ascending} part[r][n]; 8 row groups x 32 columns per CTA, fixed order.
__global__ void __launch_bounds__(256) colsum_finish_wide_kernel(const float* __restrict__ part, int R, int N,
                                                               void* out, int out_f32) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ float red[8][33];
    const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int n = blockIdx.x * 32 + c;
    float t = 0.f;
    if (n < N)
        for (int r = g; r < R; r += 8) t += part[(size_t)r * N + n];
    red[g][c] = t;
    __syncthreads();
    if (g == 0 && n < N) {
        float a = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) a += red[q][c];
        if (out_f32)
            static_cast<float*>(out)[n] = a;
        else
            static_cast<uint16_t*>(out)[n] = (uint16_t)f32_to_bf16_bits(a);
    }
}

template <int CH>
cudaError_t fwd_launch(const float* S, uint16_t* P, long long rows, int s, cudaStream_t st) {
    softmax_fwd_reg_kernel<CH><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(S, P, rows, s);
    return launched(1);
}
template <int CH>
cudaError_t bwd_launch(const uint16_t* P, const float* dP, uint16_t* dS, long long rows, int s, cudaStream_t st) {
    softmax_bwd_reg_kernel<CH><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(P, dP, dS, rows, s);
    return launched(1);
}

}  // namespace

cudaError_t softmax_fwd2(const float* S, uint16_t* P, long long rows, int s, cudaStream_t st) {
    if (s % 128 != 0 || s > 2048) return softmax_fwd(S, P, rows, s, st);
    const int ch = s / 128;  // float4 per lane
    if (ch <= 4) return fwd_launch<4>(S, P, rows, s, st);
    if (ch <= 8) return fwd_launch<8>(S, P, rows, s, st);
    return fwd_launch<kMaxChunks>(S, P, rows, s, st);
}

cudaError_t softmax_bwd2(const uint16_t* P, const float* dP, uint16_t* dS, long long rows, int s, cudaStream_t st) {
    if (s % 128 != 0 || s > 2048) return softmax_bwd(P, dP, dS, rows, s, st);
    const int ch = s / 128;
    if (ch <= 4) return bwd_launch<4>(P, dP, dS, rows, s, st);
    if (ch <= 8) return bwd_launch<8>(P, dP, dS, rows, s, st);
    return bwd_launch<kMaxChunks>(P, dP, dS, rows, s, st);
}

cudaError_t colsum_finish_wide(const float* part, int R, int N, void* out, int out_f32, cudaStream_t st) {
    launch_ex(colsum_finish_wide_kernel, dim3((N + 31) / 32), dim3(256), 0, st, 1, part, R, N, out, out_f32);
    return launched(1);
}

}  // namespace gpt
}  // namespace ah
