/* ORACLE / TEST INFRASTRUCTURE — CPU restatement of the mixed-precision AdamW step.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library; the product never does.
 *
 * Parity status: the reference implements NO optimizer arithmetic — its optimizer exists
 * only as the durations t_opt_cpu = m_p / cpu_optim_rate and t_opt_gpu = m_p /
 * gpu_optim_rate (/root/reference/proj/core/src/workload.cpp:70-71) attached to
 * OpKind::CpuOptim / OpKind::GpuOptim (proj/core/src/simulator.cpp:210-226). The state
 * layout is pinned by the reference: fp32 master + m + v = 12 B/param plus a shared 2-byte
 * param/grad buffer (proj/core/src/costmodel.cpp:44-46).
 * The update rule itself is standard AdamW with bias correction and decoupled weight decay
 * (the paper trains with Adam). Hence Adam parity is "unpinned by the
 * reference": this restatement is cross-checked against torch.optim.AdamW (fp32, CPU) in
 * tests/test_adam_oracle.py, and the product kernels must match THIS file bit-for-bit.
 *
 * Per element, fp32, round-to-nearest, no contraction (-ffp-contract=off):
 *   g  = bf16(g) * inv_scale
 *   p  = p * (1 - lr*wd)
 *   m  = b1*m + (1-b1)*g
 *   v  = b2*v + (1-b2)*(g*g)
 *   p  = p - step_size * (m / (sqrt(v) * inv_sqrt_bc2 + eps))
 *   out = bf16_rne(p)
 * with step_size = lr/(1-b1^t), inv_sqrt_bc2 = 1/sqrt(1-b2^t) derived in double on the host.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

typedef struct {
    float lr, beta1, beta2, eps, weight_decay;
    int32_t step;
} oracle_adam_hparams;

static inline float bf16_to_f32(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* round-to-nearest-even; NaN -> quiet NaN with the payload's top bits (branch-free select) */
static inline uint16_t f32_to_bf16(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    const uint32_t qnan = (u >> 16) | 0x40u;
    const uint32_t rne = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
    return (uint16_t)(((u & 0x7fffffffu) > 0x7f800000u) ? qnan : rne);
}

uint16_t oracle_f32_to_bf16(float f) { return f32_to_bf16(f); }

/* AVX-512 (x86-64-v4) and baseline clones, picked at load time: the timed CPU baseline is the
 * vectorised restatement BASELINE.md §3 asks for. Vectorisation does not change a result:
 * IEEE +,*,/,sqrt per element, no contraction, no reassociation (no -ffast-math). */
__attribute__((target_clones("arch=x86-64-v4", "default")))
void oracle_adam_f32(const oracle_adam_hparams* hp, float* p, float* m, float* v,
                     const uint16_t* g, uint16_t* out, size_t n, float inv_scale) {
    const double lr = hp->lr, b1 = hp->beta1, b2 = hp->beta2, wd = hp->weight_decay;
    const double t = hp->step < 1 ? 1.0 : (double)hp->step;
    const float decay = (float)(1.0 - lr * wd);
    const float beta1 = hp->beta1, omb1 = (float)(1.0 - b1);
    const float beta2 = hp->beta2, omb2 = (float)(1.0 - b2);
    const float step_size = (float)(lr / (1.0 - pow(b1, t)));
    const float inv_sqrt_bc2 = (float)(1.0 / sqrt(1.0 - pow(b2, t)));
    const float eps = hp->eps;
#define ADAM_BODY                                                   \
        const float gf = bf16_to_f32(g[i]) * inv_scale;             \
        float pi = p[i] * decay;                                     \
        const float mi = beta1 * m[i] + omb1 * gf;                   \
        const float vi = beta2 * v[i] + omb2 * (gf * gf);            \
        const float denom = sqrtf(vi) * inv_sqrt_bc2 + eps;          \
        pi = pi - step_size * (mi / denom);                          \
        p[i] = pi;                                                   \
        m[i] = mi;                                                   \
        v[i] = vi;
    if (out) {
        for (size_t i = 0; i < n; ++i) {
            ADAM_BODY
            out[i] = f32_to_bf16(pi);
        }
    } else {
        for (size_t i = 0; i < n; ++i) {
            ADAM_BODY
        }
    }
#undef ADAM_BODY
}

/* Same rule evaluated in double (torch-style formula: division by sqrt(bc2)) — used only to
 * bound the fp32 rounding error of the restatement itself. */
void oracle_adam_f64(const oracle_adam_hparams* hp, double* p, double* m, double* v,
                     const uint16_t* g, size_t n, double inv_scale) {
    const double lr = hp->lr, b1 = hp->beta1, b2 = hp->beta2, wd = hp->weight_decay;
    const double t = hp->step < 1 ? 1.0 : (double)hp->step;
    const double bc1 = 1.0 - pow(b1, t), bc2 = 1.0 - pow(b2, t);
    for (size_t i = 0; i < n; ++i) {
        const double gf = (double)bf16_to_f32(g[i]) * inv_scale;
        p[i] *= 1.0 - lr * wd;
        m[i] = b1 * m[i] + (1.0 - b1) * gf;
        v[i] = b2 * v[i] + (1.0 - b2) * gf * gf;
        p[i] -= (lr / bc1) * m[i] / (sqrt(v[i]) / sqrt(bc2) + (double)hp->eps);
    }
}

/* Statistics the fused kernel reports: sum of squared unscaled grads (double accumulation)
 * and the number of non-finite grads. */
void oracle_grad_stats(const uint16_t* g, size_t n, float inv_scale, double* sumsq,
                       int64_t* nonfinite) {
    double s = 0.0;
    int64_t bad = 0;
    for (size_t i = 0; i < n; ++i) {
        const float gf = bf16_to_f32(g[i]) * inv_scale;
        if (!isfinite(gf)) {
            ++bad;
        }
        s += (double)gf * (double)gf;
    }
    *sumsq = s;
    *nonfinite = bad;
}

void oracle_cast_f32_bf16(const float* src, uint16_t* dst, size_t n) {
    for (size_t i = 0; i < n; ++i) dst[i] = f32_to_bf16(src[i]);
}

/* Multi-threaded copy of oracle_adam_f32 for the timed CPU baseline (bench.py cpu_baseline
 * and --impl reference): same arithmetic, OpenMP over contiguous chunks. */
void oracle_adam_f32_mt(const oracle_adam_hparams* hp, float* p, float* m, float* v,
                        const uint16_t* g, uint16_t* out, size_t n, float inv_scale,
                        int nthreads) {
    const size_t chunk = 1u << 16;
    const long nch = (long)((n + chunk - 1) / chunk);
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (long c = 0; c < nch; ++c) {
        const size_t a = (size_t)c * chunk;
        const size_t len = a + chunk <= n ? chunk : n - a;
        oracle_adam_f32(hp, p + a, m + a, v + a, g + a, out ? out + a : NULL, len, inv_scale);
    }
}
