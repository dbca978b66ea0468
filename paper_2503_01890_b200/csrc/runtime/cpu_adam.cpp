// Host AdamW for optimizer-offloaded blocks (realises OpKind::CpuOptim, reference
// proj/core/src/simulator.cpp:210-216, duration model workload.cpp:70).
//
// Host layout per offloaded block is the paper's 14 B/param (PAPER.md:217-223,
// costmodel.cpp:44-46): fp32 master / m / v (12 B) + one bf16 buffer that holds the
// gradient after GradOffload and is overwritten in place with the updated bf16 parameters
// for the next iteration's ParamPrefetch.
//
// Work is split into contiguous 64 KiB-aligned chunks across an OpenMP team; the inner loop
// is written for the auto-vectoriser (AVX-512 / AVX2 clones selected at load time).
// Arithmetic order and rounding are identical to the GPU kernel (no FMA contraction: the
// file is compiled with -ffp-contract=off), so CPU and GPU updates agree bit-for-bit.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <omp.h>

#include "adam_scalars.h"

namespace ah {

namespace {

inline float bf16_to_f32(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

inline uint16_t f32_to_bf16(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    const uint32_t rne = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
    const uint32_t qnan = (u >> 16) | 0x40u;
    return static_cast<uint16_t>(((u & 0x7fffffffu) > 0x7f800000u) ? qnan : rne);
}

template <bool kOut>
inline void adam_loop(float* __restrict p, float* __restrict m, float* __restrict v,
                      const uint16_t* __restrict g, uint16_t* __restrict out, std::size_t n,
                      const AdamConsts& k, float inv_scale) {
#pragma omp simd
    for (std::size_t i = 0; i < n; ++i) {
        const float gf = bf16_to_f32(g[i]) * inv_scale;
        float pi = p[i] * k.decay;
        const float mi = k.beta1 * m[i] + k.one_minus_beta1 * gf;
        const float vi = k.beta2 * v[i] + k.one_minus_beta2 * (gf * gf);
        const float denom = std::sqrt(vi) * k.inv_sqrt_bc2 + k.eps;
        pi = pi - k.step_size * (mi / denom);
        p[i] = pi;
        m[i] = mi;
        v[i] = vi;
        if (kOut) out[i] = f32_to_bf16(pi);
    }
}

__attribute__((target_clones("arch=sapphirerapids", "arch=znver4", "avx2", "default")))
void adam_span(float* __restrict p, float* __restrict m, float* __restrict v,
               const uint16_t* __restrict g, uint16_t* __restrict out, std::size_t n,
               AdamConsts k, float inv_scale) {
    if (out)
        adam_loop<true>(p, m, v, g, out, n, k, inv_scale);
    else
        adam_loop<false>(p, m, v, g, out, n, k, inv_scale);
}

}  // namespace

void cpu_adam(const ah_adam_hparams& hp, float* p, float* m, float* v, const uint16_t* g,
              uint16_t* p_bf16, std::size_t n, float inv_scale, int nthreads) {
    const AdamConsts k = derive_adam_scalars(hp);
    if (nthreads <= 0) nthreads = omp_get_num_procs();
    // (Non-temporal stores of the bf16 output / of p, m, v were measured slower on the 10B plan:
    // 1512 / 1674 vs 1423 ms per step — the in-place update re-writes lines it just read.)
    // Chunks are handed out dynamically (4 at a time = 256 KiB runs per stream): the lane threads
    // share the cores with this team, and under a static split one preempted thread held the
    // whole op back. Every element is independent, so the assignment does not change a bit.
    constexpr std::size_t kChunk = 16384;  // 64 KiB of fp32 per stream per chunk
    const std::size_t n_chunks = (n + kChunk - 1) / kChunk;
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads) if (n_chunks > 1)
    for (std::size_t c = 0; c < n_chunks; ++c) {
        const std::size_t a = c * kChunk;
        const std::size_t len = (a + kChunk <= n) ? kChunk : n - a;
        adam_span(p + a, m + a, v + a, g + a, p_bf16 ? p_bf16 + a : nullptr, len, k, inv_scale);
    }
}

// Overflow-skip path of CpuOptim: the shared host buffer holds the block's gradients after
// GradOffload; the next ParamPrefetch must find bf16(master) there again.
void cpu_cast_f32_bf16(const float* src, uint16_t* dst, std::size_t n, int nthreads) {
    if (nthreads <= 0) nthreads = omp_get_num_procs();
#pragma omp parallel for simd schedule(static) num_threads(nthreads)
    for (std::size_t i = 0; i < n; ++i) dst[i] = f32_to_bf16(src[i]);
}

// Host-DRAM roofline of CpuOptim (runtime profiler): the same in-place streams as the host
// AdamW — fp32 p/m/v read + written, bf16 g read + written (28 B/param) — with trivial
// arithmetic, over `nthreads` threads and the host AdamW's work split (64 KiB chunks handed out
// dynamically), so it bounds the AdamW from above. Returns GB/s of the best of `reps` timed
// passes after one untimed pass.
namespace {
__attribute__((target_clones("arch=sapphirerapids", "arch=znver4", "avx2", "default")))
void stream_span(float* __restrict p, float* __restrict m, float* __restrict v, uint16_t* __restrict g, std::size_t n) {
#pragma omp simd
    for (std::size_t i = 0; i < n; ++i) {
        p[i] *= 0.999f;
        m[i] *= 0.999f;
        v[i] *= 0.999f;
        g[i] ^= 1u;
    }
}
}  // namespace

double host_stream_gbps(float* p, float* m, float* v, uint16_t* g, std::size_t n, int nthreads, int reps) {
    if (nthreads <= 0) nthreads = omp_get_num_procs();
    constexpr std::size_t kChunk = 16384;
    const std::size_t n_chunks = (n + kChunk - 1) / kChunk;
    double best = 0.0;
    for (int r = -1; r < reps; ++r) {
        const double t0 = omp_get_wtime();
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
        for (std::size_t c = 0; c < n_chunks; ++c) {
            const std::size_t a = c * kChunk;
            stream_span(p + a, m + a, v + a, g + a, (a + kChunk <= n) ? kChunk : n - a);
        }
        const double dt = omp_get_wtime() - t0;
        if (r >= 0 && dt > 0 && 28.0 * (double)n / dt / 1e9 > best) best = 28.0 * (double)n / dt / 1e9;
    }
    return best;
}

}  // namespace ah
