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
#include <emmintrin.h>
#include <omp.h>
#include <xmmintrin.h>

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

// Same arithmetic, blocks of 64 params computed into registers / L1 and the bf16 output (the
// buffer the next ParamPrefetch DMA reads) written with non-temporal 16-byte stores, so the
// H2D copy that follows would find the data in DRAM instead of dirty in the CPU caches
// (experiment; off by default, see cpu_adam below).
constexpr std::size_t kNtBlock = 64;
template <bool kNtAll>
inline void adam_loop_nt(float* __restrict p, float* __restrict m, float* __restrict v,
                         const uint16_t* __restrict g, uint16_t* __restrict out, std::size_t n,
                         const AdamConsts& k, float inv_scale) {
    alignas(64) float tp[kNtBlock], tm[kNtBlock], tv[kNtBlock];
    alignas(64) uint16_t to[kNtBlock];
    std::size_t i0 = 0;
    for (; i0 + kNtBlock <= n; i0 += kNtBlock) {
#pragma omp simd
        for (std::size_t j = 0; j < kNtBlock; ++j) {
            const std::size_t i = i0 + j;
            const float gf = bf16_to_f32(g[i]) * inv_scale;
            float pi = p[i] * k.decay;
            const float mi = k.beta1 * m[i] + k.one_minus_beta1 * gf;
            const float vi = k.beta2 * v[i] + k.one_minus_beta2 * (gf * gf);
            const float denom = std::sqrt(vi) * k.inv_sqrt_bc2 + k.eps;
            pi = pi - k.step_size * (mi / denom);
            tp[j] = pi;
            tm[j] = mi;
            tv[j] = vi;
            to[j] = f32_to_bf16(pi);
        }
        for (std::size_t j = 0; j < kNtBlock; j += 8)
            _mm_stream_si128(reinterpret_cast<__m128i*>(out + i0 + j), _mm_load_si128(reinterpret_cast<const __m128i*>(to + j)));
        if (kNtAll) {
            for (std::size_t j = 0; j < kNtBlock; j += 4) {
                _mm_stream_ps(p + i0 + j, _mm_load_ps(tp + j));
                _mm_stream_ps(m + i0 + j, _mm_load_ps(tm + j));
                _mm_stream_ps(v + i0 + j, _mm_load_ps(tv + j));
            }
        } else {
            std::memcpy(p + i0, tp, sizeof(tp));
            std::memcpy(m + i0, tm, sizeof(tm));
            std::memcpy(v + i0, tv, sizeof(tv));
        }
    }
    if (i0 < n) adam_loop<true>(p + i0, m + i0, v + i0, g + i0, out + i0, n - i0, k, inv_scale);
    _mm_sfence();  // the streaming stores are globally visible before the lane signals completion
}

__attribute__((target_clones("arch=sapphirerapids", "arch=znver4", "avx2", "default")))
void adam_span(float* __restrict p, float* __restrict m, float* __restrict v,
               const uint16_t* __restrict g, uint16_t* __restrict out, std::size_t n,
               AdamConsts k, float inv_scale, int nt) {
    const bool aligned = ((reinterpret_cast<std::uintptr_t>(p) | reinterpret_cast<std::uintptr_t>(m) |
                           reinterpret_cast<std::uintptr_t>(v)) & 15u) == 0 &&
                         (reinterpret_cast<std::uintptr_t>(out) & 15u) == 0;
    if (out && nt == 2 && aligned)
        adam_loop_nt<true>(p, m, v, g, out, n, k, inv_scale);
    else if (out && nt == 1 && aligned)
        adam_loop_nt<false>(p, m, v, g, out, n, k, inv_scale);
    else if (out)
        adam_loop<true>(p, m, v, g, out, n, k, inv_scale);
    else
        adam_loop<false>(p, m, v, g, out, n, k, inv_scale);
}

}  // namespace

void cpu_adam(const ah_adam_hparams& hp, float* p, float* m, float* v, const uint16_t* g,
              uint16_t* p_bf16, std::size_t n, float inv_scale, int nthreads) {
    const AdamConsts k = derive_adam_scalars(hp);
    if (nthreads <= 0) nthreads = omp_get_num_procs();
    // AH_CPU_ADAM_NT: 0 regular stores (default), 1 streaming bf16 output, 2 + streaming p/m/v.
    // Measured on the 16-vCPU box (10B, 15 offloaded blocks): 1423 / 1512 / 1674 ms per step —
    // streaming stores do not speed the following H2D DMA up, so they stay off.
    static const int nt = [] {
        const char* e = std::getenv("AH_CPU_ADAM_NT");
        return e ? std::atoi(e) : 0;
    }();
    constexpr std::size_t kChunk = 16384;  // 64 KiB of fp32 per stream per chunk
    const std::size_t n_chunks = (n + kChunk - 1) / kChunk;
#pragma omp parallel for schedule(static) num_threads(nthreads) if (n_chunks > 1)
    for (std::size_t c = 0; c < n_chunks; ++c) {
        const std::size_t a = c * kChunk;
        const std::size_t len = (a + kChunk <= n) ? kChunk : n - a;
        adam_span(p + a, m + a, v + a, g + a, p_bf16 ? p_bf16 + a : nullptr, len, k, inv_scale, nt);
    }
}

}  // namespace ah
