// Fused mixed-precision AdamW for sm_100a (realises OpKind::GpuOptim, reference
// proj/core/src/simulator.cpp:217-226, duration model workload.cpp:71).
//
// One pass over HBM per parameter: read bf16 grad (2 B) + fp32 master/m/v (12 B), write
// fp32 master/m/v (12 B) + bf16 working copy (2 B) = 28 algorithmic bytes/param. adam_tma_kernel
// is a persistent CTA per SM fed by a TMA bulk-copy ring (a register-streaming variant measured
// 5.39 vs 6.11 TB/s at 1 B params and was removed). Grad unscale is fused;
// optional statistics (sum of squared unscaled grads, count of non-finite grads) are reduced
// with warp shuffles inside a CTA and across CTAs in a fixed order by the last CTA to finish
// (stats_commit: no float atomics, so the result is bitwise reproducible). An optional device-
// side skip flag turns the launch into a no-op (overflow skip; the executor points it at the
// non-finite count of a grad_stats pre-pass).
//
// Arithmetic is IEEE round-to-nearest with no contraction (explicit __f*_rn), in exactly
// the order of oracle/adam_oracle.c and csrc/runtime/cpu_adam.cpp, so the GPU result is
// bit-identical to both CPU implementations.
#include <cstdlib>

#include "autohete.h"
#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

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

// Statistics buffer (AH_STATS_FLOATS floats, include/autohete.h): [0] sum g^2, [1] (uint32)
// non-finite count — both accumulated across launches in stream order — [2] (uint32) ticket,
// [4 + 2c], [5 + 2c] the partials of CTA c. Called by one thread per CTA with the CTA total:
// the CTA that takes the last ticket sums every partial in CTA order, adds the launch total to
// [0]/[1] and re-arms the ticket, so the result does not depend on CTA completion order.
constexpr int kStatsMaxCtas = 256;
static_assert(4 + 2 * kStatsMaxCtas <= AH_STATS_FLOATS, "stats scratch");
__device__ __forceinline__ void stats_commit(float* stats, float sum, unsigned bad) {
    float* part = stats + 4;
    unsigned* ticket = reinterpret_cast<unsigned*>(stats + 2);
    __stcg(part + 2 * blockIdx.x, sum);
    __stcg(reinterpret_cast<unsigned*>(part) + 2 * blockIdx.x + 1, bad);
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    if (t != gridDim.x - 1) return;
    __threadfence();
    float s = 0.f;
    unsigned b = 0;
    for (unsigned c = 0; c < gridDim.x; ++c) {
        s = __fadd_rn(s, __ldcg(part + 2 * c));
        b += __ldcg(reinterpret_cast<const unsigned*>(part) + 2 * c + 1);
    }
    stats[0] = __fadd_rn(stats[0], s);
    reinterpret_cast<unsigned*>(stats)[1] += b;
    *ticket = 0u;
    __threadfence();
}

// CTA reduction (up to 1024 threads) in warp order, then stats_commit.
__device__ __forceinline__ void block_stats_commit(float* stats, const Stat& st) {
    __shared__ float s_sum[32];
    __shared__ unsigned s_bad[32];
    const float ws = warp_sum(st.sumsq);
    const unsigned wb = warp_sum_u(st.nonfinite);
    if ((threadIdx.x & 31) == 0) {
        s_sum[threadIdx.x >> 5] = ws;
        s_bad[threadIdx.x >> 5] = wb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.f;
        unsigned b = 0;
        for (unsigned w = 0; w < (blockDim.x >> 5); ++w) {
            a = __fadd_rn(a, s_sum[w]);
            b += s_bad[w];
        }
        stats_commit(stats, a, b);
    }
}

// The update kernel: a persistent CTA per SM streams tiles of kTile params
// (p, m, v fp32 + g bf16 = 14 B/param) HBM -> shared memory with 1-D bulk copies
// (cp.async.bulk ... mbarrier::complete_tx) issued by one producer thread into a kStages-deep
// ring, so ~(kStages-1) x 28 KB of reads are in flight per SM independent of how many warps are
// issuing arithmetic. 16 consumer warps read their 4 params per tile from shared memory
// (conflict-free 16-B accesses), run the same IEEE arithmetic as adam_vec_kernel and write
// p/m/v (+ bf16 p) straight to HBM with coalesced 16-B stores, then release the slot.
constexpr int kTile = 2048;
constexpr int kStages = 6;
constexpr int kConsumerWarps = 16;
constexpr int kTmaThreads = (kConsumerWarps + 1) * 32;
constexpr size_t kStageBytes = (size_t)kTile * 14;
constexpr size_t kTmaSmem = kStages * kStageBytes + 2 * kStages * 8;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}

template <bool kWriteBf16, bool kStats>
__global__ void __launch_bounds__(kTmaThreads, 1)
adam_tma_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                const uint16_t* __restrict__ g, uint16_t* __restrict__ pout, size_t n_main,
                AdamScalars k, const int* __restrict__ skip, float* __restrict__ stats) {
    pdl_launch_dependents();
    pdl_wait();
    if (skip != nullptr && *skip != 0) return;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t n_tiles = (n_main + kTile - 1) / kTile;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(tc::smem_u32(&full[s]), 1);
            tc::mbar_init(tc::smem_u32(&empty[s]), kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kConsumerWarps) {  // producer
        if (lane == 0) {
            uint64_t policy;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
            int s = 0;
            uint32_t phase = 0;
            for (size_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                if (t >= blockIdx.x + (size_t)kStages * gridDim.x) tc::mbar_wait(tc::smem_u32(&empty[s]), phase ^ 1);
                const size_t base = t * kTile;
                const uint32_t cnt = (uint32_t)(n_main - base < (size_t)kTile ? n_main - base : kTile);
                uint8_t* st = smem + s * kStageBytes;
                const uint32_t bar = tc::smem_u32(&full[s]);
                tc::mbar_expect_tx(bar, cnt * 14);
                bulk_g2s(tc::smem_u32(st), p + base, cnt * 4, bar, policy);
                bulk_g2s(tc::smem_u32(st + kTile * 4), m + base, cnt * 4, bar, policy);
                bulk_g2s(tc::smem_u32(st + kTile * 8), v + base, cnt * 4, bar, policy);
                bulk_g2s(tc::smem_u32(st + kTile * 12), g + base, cnt * 2, bar, policy);
                if (++s == kStages) { s = 0; phase ^= 1; }
            }
        }
        return;
    }

    Stat acc;
    int s = 0;
    uint32_t phase = 0;
    const int e0 = threadIdx.x * 4;  // this thread's 4 params within the tile
    for (size_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const size_t base = t * kTile;
        const size_t cnt = n_main - base < (size_t)kTile ? n_main - base : kTile;
        tc::mbar_wait(tc::smem_u32(&full[s]), phase);
        const uint8_t* st = smem + s * kStageBytes;
        if ((size_t)e0 < cnt) {  // cnt is a multiple of 8
            float4 pp = *reinterpret_cast<const float4*>(st + e0 * 4);
            float4 mm = *reinterpret_cast<const float4*>(st + kTile * 4 + e0 * 4);
            float4 vv = *reinterpret_cast<const float4*>(st + kTile * 8 + e0 * 4);
            const uint2 gw = *reinterpret_cast<const uint2*>(st + kTile * 12 + e0 * 2);
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&empty[s]));
            float* pv = &pp.x;
            float* mv = &mm.x;
            float* vq = &vv.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t w = e < 2 ? gw.x : gw.y;
                const uint32_t bits = (e & 1) ? (w >> 16) : (w & 0xffffu);
                const float gf = __fmul_rn(bf16_bits_to_f32(bits), k.inv_scale);
                if (kStats) account(acc, gf);
                adam_one(pv[e], mv[e], vq[e], gf, k);
            }
            st_f4(p + base + e0, pp);
            st_f4(m + base + e0, mm);
            st_f4(v + base + e0, vv);
            if (kWriteBf16) {
                const uint2 o = make_uint2(pack_bf16x2(pp.x, pp.y), pack_bf16x2(pp.z, pp.w));
                asm volatile("st.global.L1::no_allocate.v2.u32 [%0], {%1,%2};" ::"l"(pout + base + e0), "r"(o.x),
                             "r"(o.y)
                             : "memory");
            }
        } else {
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&empty[s]));
        }
        if (++s == kStages) { s = 0; phase ^= 1; }
    }
    if (kStats) {
        __shared__ float s_sum[kConsumerWarps];
        __shared__ unsigned s_bad[kConsumerWarps];
        const float ws = warp_sum(acc.sumsq);
        const unsigned wb = warp_sum_u(acc.nonfinite);
        if (lane == 0) {
            s_sum[warp] = ws;
            s_bad[warp] = wb;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
        if (threadIdx.x < 32) {
            float a = threadIdx.x < kConsumerWarps ? s_sum[threadIdx.x] : 0.f;
            unsigned b = threadIdx.x < kConsumerWarps ? s_bad[threadIdx.x] : 0u;
            a = warp_sum(a);
            b = warp_sum_u(b);
            if (threadIdx.x == 0) stats_commit(stats, a, b);
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
    if (stats) block_stats_commit(stats, st);
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ src, uint16_t* __restrict__ dst,
                                     size_t n_vec) {
    pdl_launch_dependents();
    pdl_wait();
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

__global__ void __launch_bounds__(1024, 1) grad_stats_kernel(const uint16_t* __restrict__ g, size_t n, float inv_scale,
                                                          float* __restrict__ stats, bool vec) {
    pdl_launch_dependents();
    pdl_wait();
    // one 1024-thread CTA per SM (the fixed-order cross-CTA scratch caps the CTA count, so the
    // CTAs are large), 4 loads in flight per thread (~10 MB device-wide) and 4 independent partial
    // sums per thread (combined in a fixed order) so the add chains do not serialise
    constexpr int kU = 4;
    Stat st[kU];
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t n_vec = vec ? n / 8 : 0;
    for (size_t j0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j0 < n_vec; j0 += stride * kU) {
        uint4 w[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const size_t j = j0 + (size_t)u * stride;
            w[u] = j < n_vec ? ld_stream_u4(g + j * 8) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint32_t bits = (e & 1) ? (ws[e >> 1] >> 16) : (ws[e >> 1] & 0xffffu);
                account(st[u], __fmul_rn(bf16_bits_to_f32(bits), inv_scale));  // zero padding adds +0
            }
        }
    }
    for (size_t i = n_vec * 8 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        account(st[0], __fmul_rn(bf16_bits_to_f32(g[i]), inv_scale));
    Stat t;
    for (int u = 0; u < kU; ++u) {
        t.sumsq = __fadd_rn(t.sumsq, st[u].sumsq);
        t.nonfinite += st[u].nonfinite;
    }
    block_stats_commit(stats, t);
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
            const size_t tiles = (n_vec * 8 + kTile - 1) / kTile;
            const int grid = (int)(tiles < (size_t)kNumSMs ? tiles : (size_t)kNumSMs);
            static bool attr = [] {
                cudaFuncSetAttribute(adam_tma_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
                cudaFuncSetAttribute(adam_tma_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
                cudaFuncSetAttribute(adam_tma_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
                cudaFuncSetAttribute(adam_tma_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
                return true;
            }();
            (void)attr;
            const size_t nm = n_vec * 8;
            if (a.p_bf16 && a.stats)
                launch_ex((adam_tma_kernel<true, true>), dim3(grid), dim3(kTmaThreads), kTmaSmem, stream, 1, a.p, a.m, a.v, a.g, a.p_bf16, nm, k, a.skip, a.stats);
            else if (a.p_bf16)
                launch_ex((adam_tma_kernel<true, false>), dim3(grid), dim3(kTmaThreads), kTmaSmem, stream, 1, a.p, a.m, a.v, a.g, a.p_bf16, nm, k, a.skip, a.stats);
            else if (a.stats)
                launch_ex((adam_tma_kernel<false, true>), dim3(grid), dim3(kTmaThreads), kTmaSmem, stream, 1, a.p, a.m, a.v, a.g, a.p_bf16, nm, k, a.skip, a.stats);
            else
                launch_ex((adam_tma_kernel<false, false>), dim3(grid), dim3(kTmaThreads), kTmaSmem, stream, 1, a.p, a.m, a.v, a.g, a.p_bf16, nm, k, a.skip, a.stats);
        }
        done = n_vec * 8;
    }
    if (done < a.n) {
        int grid = vec ? 1 : grid_for(a.n, 256, 4);
        if (a.stats && grid > kStatsMaxCtas) grid = kStatsMaxCtas;
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
        if (n_vec) launch_ex(cast_f32_bf16_kernel, dim3(grid_for(n_vec, 256, 8)), dim3(256), 0, stream, 1, src, dst, n_vec);
        done = n_vec * 8;
    }
    if (done < n) cast_tail_kernel<<<1, 256, 0, stream>>>(src, dst, done, n);
    return launched(1);
}

cudaError_t launch_grad_stats(const uint16_t* g, size_t n, float inv_scale, float* stats,
                              cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const bool vec = aligned16(g);
    const int grid = grid_for(vec ? n / 32 + 1 : n, 1024, 1);  // <= kNumSMs <= kStatsMaxCtas
    launch_ex(grad_stats_kernel, dim3(grid), dim3(1024), 0, stream, 1, g, n, inv_scale, stats, vec);
    return launched(1);
}

}  // namespace ah
