// Fused mixed-precision AdamW for sm_100a (realises OpKind::GpuOptim, reference
// proj/core/src/simulator.cpp:217-226, duration model workload.cpp:71).
//
// One pass over HBM per parameter: read bf16 grad (2 B) + fp32 master/m/v (12 B), write
// fp32 master/m/v (12 B) + bf16 working copy (2 B) = 28 algorithmic bytes/param. 128-bit
// vector loads/stores (8 params per vector step), two steps in flight per thread, grid sized
// to 4 resident CTAs x 148 SMs with a grid-stride loop. Grad unscale is fused; optional
// by-product statistics (sum of squared unscaled grads, count of non-finite grads) are
// reduced with warp shuffles, one atomic pair per CTA. An optional device-side skip flag
// turns the launch into a no-op (dynamic loss-scaling overflow skip).
//
// Arithmetic is IEEE round-to-nearest with no contraction (explicit __f*_rn), in exactly
// the order of oracle/adam_oracle.c and csrc/runtime/cpu_adam.cpp, so the GPU result is
// bit-identical to both CPU implementations.
#include "common.cuh"
#include "kernels.h"

namespace ah {

namespace {

struct AdamScalars {
    float decay;         // 1 - lr*wd
    float beta1, one_minus_beta1;
    float beta2, one_minus_beta2;
    float step_size;     // lr / (1 - beta1^t)
    float inv_sqrt_bc2;  // 1 / sqrt(1 - beta2^t)
    float eps;
    float inv_scale;
};

struct Stat {
    float sumsq = 0.f;
    unsigned nonfinite = 0;
};

__device__ __forceinline__ float adam_one(float& p, float& m, float& v, float g,
                                          const AdamScalars& k) {
    p = __fmul_rn(p, k.decay);
    m = __fadd_rn(__fmul_rn(k.beta1, m), __fmul_rn(k.one_minus_beta1, g));
    v = __fadd_rn(__fmul_rn(k.beta2, v), __fmul_rn(k.one_minus_beta2, __fmul_rn(g, g)));
    const float denom = __fadd_rn(__fmul_rn(__fsqrt_rn(v), k.inv_sqrt_bc2), k.eps);
    p = __fsub_rn(p, __fmul_rn(k.step_size, __fdiv_rn(m, denom)));
    return p;
}

__device__ __forceinline__ void account(Stat& st, float g) {
    st.sumsq = __fadd_rn(st.sumsq, __fmul_rn(g, g));
    st.nonfinite += isfinite(g) ? 0u : 1u;
}

constexpr int kThreads = 256;
constexpr int kUnroll = 2;

struct F8 {
    float x[8];
};

__device__ __forceinline__ void ld8(F8& d, const float* q) {
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(d.x[0]), "=f"(d.x[1]), "=f"(d.x[2]), "=f"(d.x[3])
                 : "l"(q));
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(d.x[4]), "=f"(d.x[5]), "=f"(d.x[6]), "=f"(d.x[7])
                 : "l"(q + 4));
}
__device__ __forceinline__ void st8(float* q, const F8& d) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q), "f"(d.x[0]),
                 "f"(d.x[1]), "f"(d.x[2]), "f"(d.x[3])
                 : "memory");
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(q + 4), "f"(d.x[4]),
                 "f"(d.x[5]), "f"(d.x[6]), "f"(d.x[7])
                 : "memory");
}

template <bool kWriteBf16, bool kStats>
__global__ void __launch_bounds__(kThreads, 2)
adam_vec_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                const uint16_t* __restrict__ g, uint16_t* __restrict__ pout, size_t n_vec,
                AdamScalars k, const int* __restrict__ skip, float* __restrict__ stats) {
    if (skip != nullptr && *skip != 0) return;
    Stat st;
    const size_t stride = (size_t)gridDim.x * kThreads;
    for (size_t base = (size_t)blockIdx.x * kThreads + threadIdx.x; base < n_vec;
         base += stride * kUnroll) {
        uint4 gv[kUnroll];
        F8 pv[kUnroll], mv[kUnroll], vv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const size_t j = base + (size_t)u * stride;
            if (j < n_vec) {
                gv[u] = ld_stream_u4(g + j * 8);
                ld8(pv[u], p + j * 8);
                ld8(mv[u], m + j * 8);
                ld8(vv[u], v + j * 8);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const size_t j = base + (size_t)u * stride;
            if (j >= n_vec) continue;
            const uint32_t gw[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint32_t bits = (e & 1) ? (gw[e >> 1] >> 16) : (gw[e >> 1] & 0xffffu);
                const float gf = __fmul_rn(bf16_bits_to_f32(bits), k.inv_scale);
                if (kStats) account(st, gf);
                adam_one(pv[u].x[e], mv[u].x[e], vv[u].x[e], gf, k);
            }
            st8(p + j * 8, pv[u]);
            st8(m + j * 8, mv[u]);
            st8(v + j * 8, vv[u]);
            if (kWriteBf16)
                st_u4(pout + j * 8,
                      make_uint4(pack_bf16x2(pv[u].x[0], pv[u].x[1]), pack_bf16x2(pv[u].x[2], pv[u].x[3]),
                                 pack_bf16x2(pv[u].x[4], pv[u].x[5]), pack_bf16x2(pv[u].x[6], pv[u].x[7])));
        }
    }
    if (kStats) {
        __shared__ float s_sum[kThreads / 32];
        __shared__ unsigned s_bad[kThreads / 32];
        const float ws = warp_sum(st.sumsq);
        const unsigned wb = warp_sum_u(st.nonfinite);
        if ((threadIdx.x & 31) == 0) {
            s_sum[threadIdx.x >> 5] = ws;
            s_bad[threadIdx.x >> 5] = wb;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            float a = threadIdx.x < kThreads / 32 ? s_sum[threadIdx.x] : 0.f;
            unsigned b = threadIdx.x < kThreads / 32 ? s_bad[threadIdx.x] : 0u;
            a = warp_sum(a);
            b = warp_sum_u(b);
            if (threadIdx.x == 0) {
                atomicAdd(stats, a);
                if (b) atomicAdd(reinterpret_cast<unsigned*>(stats + 1), b);
            }
        }
    }
}

// Scalar path: the < 8-element tail, or buffers that are not 16-byte aligned.
__global__ void adam_scalar_kernel(float* p, float* m, float* v, const uint16_t* g,
                                   uint16_t* pout, size_t begin, size_t n, AdamScalars k,
                                   const int* skip, float* stats) {
    if (skip != nullptr && *skip != 0) return;
    Stat st;
    for (size_t i = begin + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const float gf = __fmul_rn(bf16_bits_to_f32(g[i]), k.inv_scale);
        if (stats) account(st, gf);
        float pp = p[i], mm = m[i], vq = v[i];
        adam_one(pp, mm, vq, gf, k);
        p[i] = pp;
        m[i] = mm;
        v[i] = vq;
        if (pout) pout[i] = (uint16_t)f32_to_bf16_bits(pp);
    }
    if (stats) {
        const float ws = warp_sum(st.sumsq);
        const unsigned wb = warp_sum_u(st.nonfinite);
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(stats, ws);
            if (wb) atomicAdd(reinterpret_cast<unsigned*>(stats + 1), wb);
        }
    }
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ src, uint16_t* __restrict__ dst,
                                     size_t n_vec) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_vec; j += stride) {
        const float4 a = ld_f4(src + j * 8);
        const float4 b = ld_f4(src + j * 8 + 4);
        st_u4(dst + j * 8, make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w),
                                      pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w)));
    }
}

__global__ void cast_tail_kernel(const float* src, uint16_t* dst, size_t begin, size_t n) {
    for (size_t i = begin + threadIdx.x; i < n; i += blockDim.x)
        dst[i] = (uint16_t)f32_to_bf16_bits(src[i]);
}

__global__ void grad_stats_kernel(const uint16_t* __restrict__ g, size_t n, float inv_scale,
                                  float* __restrict__ stats, bool vec) {
    Stat st;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t n_vec = vec ? n / 8 : 0;
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_vec; j += stride) {
        const uint4 w = ld_stream_u4(g + j * 8);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint32_t bits = (e & 1) ? (ws[e >> 1] >> 16) : (ws[e >> 1] & 0xffffu);
            account(st, __fmul_rn(bf16_bits_to_f32(bits), inv_scale));
        }
    }
    for (size_t i = n_vec * 8 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        account(st, __fmul_rn(bf16_bits_to_f32(g[i]), inv_scale));
    const float a = warp_sum(st.sumsq);
    const unsigned b = warp_sum_u(st.nonfinite);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(stats, a);
        if (b) atomicAdd(reinterpret_cast<unsigned*>(stats + 1), b);
    }
}

bool aligned16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; }

int grid_for(size_t work_items, int threads, int per_sm) {
    const size_t want = (work_items + threads - 1) / threads;
    const size_t cap = (size_t)kNumSMs * per_sm;
    return (int)(want < cap ? (want == 0 ? 1 : want) : cap);
}

}  // namespace

cudaError_t launch_adam(const AdamArgs& a, cudaStream_t stream) {
    AdamScalars k;
    k.decay = a.decay;
    k.beta1 = a.beta1;
    k.one_minus_beta1 = a.one_minus_beta1;
    k.beta2 = a.beta2;
    k.one_minus_beta2 = a.one_minus_beta2;
    k.step_size = a.step_size;
    k.inv_sqrt_bc2 = a.inv_sqrt_bc2;
    k.eps = a.eps;
    k.inv_scale = a.inv_scale;
    if (a.n == 0) return cudaSuccess;
    const bool vec = aligned16(a.p) && aligned16(a.m) && aligned16(a.v) && aligned16(a.g) &&
                     (a.p_bf16 == nullptr || aligned16(a.p_bf16));
    size_t done = 0;
    if (vec) {
        const size_t n_vec = a.n / 8;
        if (n_vec) {
            const int grid = grid_for((n_vec + kUnroll - 1) / kUnroll, kThreads, 2);
            if (a.p_bf16 && a.stats)
                adam_vec_kernel<true, true><<<grid, kThreads, 0, stream>>>(a.p, a.m, a.v, a.g, a.p_bf16, n_vec, k, a.skip, a.stats);
            else if (a.p_bf16)
                adam_vec_kernel<true, false><<<grid, kThreads, 0, stream>>>(a.p, a.m, a.v, a.g, a.p_bf16, n_vec, k, a.skip, a.stats);
            else if (a.stats)
                adam_vec_kernel<false, true><<<grid, kThreads, 0, stream>>>(a.p, a.m, a.v, a.g, a.p_bf16, n_vec, k, a.skip, a.stats);
            else
                adam_vec_kernel<false, false><<<grid, kThreads, 0, stream>>>(a.p, a.m, a.v, a.g, a.p_bf16, n_vec, k, a.skip, a.stats);
        }
        done = n_vec * 8;
    }
    if (done < a.n) {
        const int grid = vec ? 1 : grid_for(a.n, 256, 4);
        adam_scalar_kernel<<<grid, 256, 0, stream>>>(a.p, a.m, a.v, a.g, a.p_bf16, done, a.n, k,
                                                      a.skip, a.stats);
    }
    return launched(1);
}

cudaError_t launch_cast_f32_bf16(const float* src, uint16_t* dst, size_t n, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    size_t done = 0;
    if (aligned16(src) && aligned16(dst)) {
        const size_t n_vec = n / 8;
        if (n_vec) cast_f32_bf16_kernel<<<grid_for(n_vec, 256, 8), 256, 0, stream>>>(src, dst, n_vec);
        done = n_vec * 8;
    }
    if (done < n) cast_tail_kernel<<<1, 256, 0, stream>>>(src, dst, done, n);
    return launched(1);
}

cudaError_t launch_grad_stats(const uint16_t* g, size_t n, float inv_scale, float* stats,
                              cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const bool vec = aligned16(g);
    grad_stats_kernel<<<grid_for(vec ? n / 8 + 1 : n, 256, 8), 256, 0, stream>>>(g, n, inv_scale,
                                                                               stats, vec);
    return launched(1);
}

}  // namespace ah
