// Row-parallel LayerNorm for the GPT block (Compute lane of OpKind::Forward / Backward /
// Recompute, reference proj/core/src/simulator.cpp:125-198; the op has no reference kernel).
//
// Layout: one CTA of h/8 threads owns a contiguous chunk of rows; thread t owns the 8 columns
// [8t, 8t+8) of every row, so a row is read from HBM exactly once (16-byte loads) and each
// column-reduction accumulator lives in the register of the thread that owns the column. The
// two row statistics are reduced across the CTA with warp shuffles + one barrier into a
// parity-double-buffered smem slot, and the next row's loads are issued before that barrier so
// every SM keeps ~2 rows x (x, dy, dres) in flight.
//
// The backward fuses what used to be four passes over the T x h activations: dx (with the
// residual-path gradient added), the LayerNorm dgamma / dbeta column sums, and optionally the
// bias gradients that are column sums of the residual-path gradient (b_fc2: sum of dres) and of
// the output (b_proj: sum of dx). Column partials go to part[cta][4h] in fixed row order and
// are finished by one fixed-order reduction over the CTAs: deterministic, no float atomics.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gpt_kernels.h"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace ah {
namespace gpt {
namespace {

constexpr float kLnEps = 1e-5f;
__device__ __forceinline__ uint32_t tc_smem(const void* p) { return tc::smem_u32(p); }

__device__ __forceinline__ void unpack8(const uint4& w, float (&f)[8]) {
    const uint32_t a[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = bf16_bits_to_f32(a[i] & 0xffffu);
        f[2 * i + 1] = bf16_bits_to_f32(a[i] >> 16);
    }
}
__device__ __forceinline__ uint4 ldg16(const void* p) { return *reinterpret_cast<const uint4*>(p); }

// Sum four values over the CTA; every thread gets the totals. Fixed order (warp tree, then
// warps in index order) so the result is identical on every launch. The smem slot alternates
// so consecutive calls need one barrier each.
__device__ __forceinline__ float4 cta_sum4(float4 v, float4* red, int& slot) {
    v.x = warp_sum(v.x);
    v.y = warp_sum(v.y);
    v.z = warp_sum(v.z);
    v.w = warp_sum(v.w);
    const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
    float4* r = red + slot * 32;
    if ((threadIdx.x & 31) == 0) r[w] = v;
    __syncthreads();
    float4 t = r[0];
    for (int q = 1; q < nw; ++q) {
        const float4 u = r[q];
        t.x += u.x;
        t.y += u.y;
        t.z += u.z;
        t.w += u.w;
    }
    slot ^= 1;
    return t;
}

// Two-value variant (the forward's per-row-pair mean / variance): half the shuffles.
__device__ __forceinline__ float2 cta_sum2v(float a, float b, float4* red, int& slot) {
    a = warp_sum(a);
    b = warp_sum(b);
    const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
    float2* r = reinterpret_cast<float2*>(red + slot * 32);
    if ((threadIdx.x & 31) == 0) r[w] = make_float2(a, b);
    __syncthreads();
    float2 t = r[0];
    for (int q = 1; q < nw; ++q) {
        const float2 u = r[q];
        t.x += u.x;
        t.y += u.y;
    }
    slot ^= 1;
    return t;
}

// Two rows per iteration share each barrier, so the ring holds 2 iterations of rows (measured at
// 8192 x 2048: fused backward 37.5 vs 43–45 µs with 3 iterations in flight, plain 30.4 vs 31).
constexpr int kRing = 4;

__device__ __forceinline__ void bulk_row(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bar_init(uint64_t* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_smem(b)));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(tc_smem(b)), "r"(parity)
                     : "memory");
}

// Shared-memory plan of one CTA: kRing stages of NT rows (x [, dy [, dres]]), per-row stats,
// one mbarrier per stage.
// The ring is kRing deep unless that would not fit in ~190 KB.
struct RingPlan {
    uint32_t stage_bytes, stats_off, bar_off, total;
    int ring;
    __host__ __device__ RingPlan(int h, int nt, int rows) {
        stage_bytes = (uint32_t)(nt * h * 2);
        const int fit = (int)((190u * 1024u) / stage_bytes) & ~1;
        ring = fit < kRing ? (fit < 2 ? 2 : fit) : kRing;
        stats_off = (uint32_t)ring * stage_bytes;
        bar_off = (stats_off + (uint32_t)rows * 8 + 15) & ~15u;
        total = bar_off + kRing * 8;
    }
};

__device__ __forceinline__ uint4 pack8_rn(const float (&o)[8]) {
    return make_uint4(pack_bf16x2_rn(o[0], o[1]), pack_bf16x2_rn(o[2], o[3]), pack_bf16x2_rn(o[4], o[5]),
                      pack_bf16x2_rn(o[6], o[7]));
}

// Forward: thread 0 streams rows into the ring with 1-D bulk copies; a pair of rows' stages is
// released by the pair's first statistics barrier (every thread holds its values by then).
__global__ void __launch_bounds__(768) ln_fwd_rows_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ g,
                                                          const uint16_t* __restrict__ b, uint16_t* __restrict__ y,
                                                          float* __restrict__ mean, float* __restrict__ rstd, int T,
                                                          int h, int rows) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ float4 red[64];
    const RingPlan plan(h, 1, 0);
    const int ring = plan.ring;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + plan.bar_off);
    int slot = 0;
    const int c = threadIdx.x * 8;
    const int r0 = blockIdx.x * rows, n = min(T, r0 + rows) - r0;
    const uint32_t rb = (uint32_t)h * 2;
    auto issue = [&](int j, int st) {
        bar_expect(&bars[st], rb);
        bulk_row(tc_smem(sm + st * plan.stage_bytes), x + (size_t)(r0 + j) * h, rb, tc_smem(&bars[st]));
    };
    pdl_launch_dependents();
    pdl_wait();
    if (threadIdx.x == 0) {
        for (int i = 0; i < ring; ++i) bar_init(&bars[i]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int j = 0; j < n && j < ring; ++j) issue(j, j);
    }
    float gg[8], bb[8];
    unpack8(ldg16(g + c), gg);
    unpack8(ldg16(b + c), bb);
    const float inv_h = 1.0f / (float)h;
    __syncthreads();
    int st = 0;  // stage of row j (even: rows j, j+1 sit in stages st, st+1)
    uint32_t ph = 0;
    for (int j = 0; j < n; j += 2) {
        const bool two = j + 1 < n;
        float fa[8], fb[8];
        bar_wait(&bars[st], ph);
        unpack8(*reinterpret_cast<const uint4*>(sm + st * plan.stage_bytes + c * 2), fa);
        if (two) {
            bar_wait(&bars[st + 1], ph);
            unpack8(*reinterpret_cast<const uint4*>(sm + (st + 1) * plan.stage_bytes + c * 2), fb);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) fb[i] = 0.f;
        }
        float sa = 0.f, sb = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            sa += fa[i];
            sb += fb[i];
        }
        const float2 m = cta_sum2v(sa, sb, red, slot);
        if (threadIdx.x == 0) {  // both stages are free: refill them
            if (j + ring < n) issue(j + ring, st);
            if (j + 1 + ring < n) issue(j + 1 + ring, st + 1);
        }
        st += 2;
        if (st == ring) {
            st = 0;
            ph ^= 1u;
        }
        const float mua = m.x * inv_h, mub = m.y * inv_h;
        float va = 0.f, vb = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            va += (fa[i] - mua) * (fa[i] - mua);
            vb += (fb[i] - mub) * (fb[i] - mub);
        }
        const float2 v = cta_sum2v(va, vb, red, slot);
        const float rsa = rsqrtf(v.x * inv_h + kLnEps), rsb = rsqrtf(v.y * inv_h + kLnEps);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            fa[i] = (fa[i] - mua) * rsa * gg[i] + bb[i];
            fb[i] = (fb[i] - mub) * rsb * gg[i] + bb[i];
        }
        const int r = r0 + j;
        st_u4(y + (size_t)r * h + c, pack8_rn(fa));
        if (two) st_u4(y + (size_t)(r + 1) * h + c, pack8_rn(fb));
        if (threadIdx.x == 0) {
            mean[r] = mua;
            rstd[r] = rsa;
            if (two) {
                mean[r + 1] = mub;
                rstd[r + 1] = rsb;
            }
        }
    }
}

// Forward, warp per row with the whole row in registers (h = 256 * NC): all NC 16-byte loads
// of a row are issued before any arithmetic, the two statistics are warp-shuffle reductions (no
// CTA barrier), so ~6 rows per SM are in flight with no shared-memory staging at all.
template <int NC>
__global__ void __launch_bounds__(256) ln_fwd_warp_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ g,
                                                         const uint16_t* __restrict__ b, uint16_t* __restrict__ y,
                                                         float* __restrict__ mean, float* __restrict__ rstd, int T) {
    constexpr int h = NC * 256;
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    pdl_launch_dependents();
    pdl_wait();
    if (row >= T) return;
    const uint16_t* xr = x + (size_t)row * h + lane * 8;
    uint4 w[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) w[k] = ld_stream_u4(xr + k * 256);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        float f[8];
        unpack8(w[k], f);
#pragma unroll
        for (int i = 0; i < 8; ++i) s += f[i];
    }
    const float mu = warp_sum(s) * (1.0f / h);
    float v = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        float f[8];
        unpack8(w[k], f);
#pragma unroll
        for (int i = 0; i < 8; ++i) v += (f[i] - mu) * (f[i] - mu);
    }
    const float rs = rsqrtf(warp_sum(v) * (1.0f / h) + kLnEps);
    uint16_t* yr = y + (size_t)row * h + lane * 8;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        float f[8], gg[8], bb[8];
        unpack8(w[k], f);
        unpack8(ldg16(g + k * 256 + lane * 8), gg);
        unpack8(ldg16(b + k * 256 + lane * 8), bb);
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = (f[i] - mu) * rs * gg[i] + bb[i];
        st_u4(yr + k * 256, pack8_rn(f));
    }
    if (lane == 0) {
        mean[row] = mu;
        rstd[row] = rs;
    }
}

// One row of the backward, first half: xhat in place, row partial sums, column accumulators.
template <bool kRes>
struct BwdRow {
    float xf[8], df[8];
    uint4 rw;
    float mu, rs;
};

template <bool kRes, bool kColRes, bool kColDx>
__global__ void __launch_bounds__(768) ln_bwd_rows_kernel(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ x,
                                                          const float* __restrict__ mean, const float* __restrict__ rstd,
                                                          const uint16_t* __restrict__ g, const uint16_t* dres,
                                                          uint16_t* dx, float* __restrict__ part, int T, int h,
                                                          int rows) {
    constexpr int NT = kRes ? 3 : 2;
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ float4 red[64];
    const RingPlan plan(h, NT, rows);
    const int ring = plan.ring;
    float2* stats = reinterpret_cast<float2*>(sm + plan.stats_off);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + plan.bar_off);
    int slot = 0;
    const int c = threadIdx.x * 8;
    const int r0 = blockIdx.x * rows, n = min(T, r0 + rows) - r0;
    const uint32_t rb = (uint32_t)h * 2;
    auto issue = [&](int j, int st) {
        uint8_t* d = sm + st * plan.stage_bytes;
        const size_t off = (size_t)(r0 + j) * h;
        bar_expect(&bars[st], NT * rb);
        bulk_row(tc_smem(d), x + off, rb, tc_smem(&bars[st]));
        bulk_row(tc_smem(d + rb), dy + off, rb, tc_smem(&bars[st]));
        if (kRes) bulk_row(tc_smem(d + 2 * rb), dres + off, rb, tc_smem(&bars[st]));
    };
    pdl_launch_dependents();
    pdl_wait();
    if (threadIdx.x == 0) {
        for (int i = 0; i < ring; ++i) bar_init(&bars[i]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int j = 0; j < n && j < ring; ++j) issue(j, j);
    }
    for (int j = threadIdx.x; j < n; j += blockDim.x) stats[j] = make_float2(mean[r0 + j], rstd[r0 + j]);
    float gg[8];
    unpack8(ldg16(g + c), gg);
    const float inv_h = 1.0f / (float)h;
    float adg[8], adb[8], ares[8], adx[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) adg[i] = adb[i] = ares[i] = adx[i] = 0.f;
    __syncthreads();

    auto load = [&](BwdRow<kRes>& R, int j, int st, uint32_t ph, float4& sums, bool lo) {
        bar_wait(&bars[st], ph);
        const uint8_t* d = sm + st * plan.stage_bytes + c * 2;
        unpack8(*reinterpret_cast<const uint4*>(d), R.xf);
        unpack8(*reinterpret_cast<const uint4*>(d + rb), R.df);
        if (kRes) R.rw = *reinterpret_cast<const uint4*>(d + 2 * rb);
        const float2 mr = stats[j];
        R.mu = mr.x;
        R.rs = mr.y;
        const float nb = -R.mu * R.rs;
        // paired fp32 (FFMA2 / FADD2 / FMUL2): the row loop is issue-bound
        const unsigned long long rs2 = tc::f2pack(R.rs, R.rs), nb2 = tc::f2pack(nb, nb);
        unsigned long long s1 = 0ull, s2 = 0ull;  // (even, odd) column partial sums
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
            const unsigned long long xh = tc::ffma2(tc::f2pack(R.xf[i], R.xf[i + 1]), rs2, nb2);  // xhat
            const unsigned long long d = tc::f2pack(R.df[i], R.df[i + 1]);
            const unsigned long long dg = tc::fmul2(d, tc::f2pack(gg[i], gg[i + 1]));
            s1 = tc::fadd2(s1, dg);
            s2 = tc::ffma2(dg, xh, s2);
            unsigned long long ag = tc::ffma2(d, xh, tc::f2pack(adg[i], adg[i + 1]));
            unsigned long long ab = tc::fadd2(tc::f2pack(adb[i], adb[i + 1]), d);
            tc::f2unpack(xh, R.xf[i], R.xf[i + 1]);
            tc::f2unpack(ag, adg[i], adg[i + 1]);
            tc::f2unpack(ab, adb[i], adb[i + 1]);
        }
        float a0, a1, b0, b1;
        tc::f2unpack(s1, a0, a1);
        tc::f2unpack(s2, b0, b1);
        if (lo) {
            sums.x = a0 + a1;
            sums.y = b0 + b1;
        } else {
            sums.z = a0 + a1;
            sums.w = b0 + b1;
        }
    };
    auto emit = [&](const BwdRow<kRes>& R, int j, float m1, float m2) {
        float o[8];
        const unsigned long long nm2 = tc::f2pack(-m2, -m2), nm1 = tc::f2pack(-m1, -m1), rs2 = tc::f2pack(R.rs, R.rs);
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
            const unsigned long long dg = tc::fmul2(tc::f2pack(R.df[i], R.df[i + 1]), tc::f2pack(gg[i], gg[i + 1]));
            const unsigned long long t = tc::fadd2(tc::ffma2(tc::f2pack(R.xf[i], R.xf[i + 1]), nm2, dg), nm1);
            tc::f2unpack(tc::fmul2(rs2, t), o[i], o[i + 1]);
        }
        if (kRes) {
            float rf[8];
            unpack8(R.rw, rf);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                o[i] += rf[i];
                if (kColRes) ares[i] += rf[i];
            }
        }
        const uint4 packed = pack8_rn(o);
        st_u4(dx + (size_t)(r0 + j) * h + c, packed);
        if (kColDx) {  // bias gradient = column sum of the stored (bf16) output
            float q[8];
            unpack8(packed, q);
#pragma unroll
            for (int i = 0; i < 8; ++i) adx[i] += q[i];
        }
    };

    int st = 0;
    uint32_t ph = 0;
    for (int j = 0; j < n; j += 2) {
        const bool two = j + 1 < n;
        BwdRow<kRes> A, B;
        float4 sums = make_float4(0.f, 0.f, 0.f, 0.f);
        load(A, j, st, ph, sums, true);
        if (two) load(B, j + 1, st + 1, ph, sums, false);
        const float4 t = cta_sum4(sums, red, slot);
        if (threadIdx.x == 0) {  // every thread has read both stages
            if (j + ring < n) issue(j + ring, st);
            if (j + 1 + ring < n) issue(j + 1 + ring, st + 1);
        }
        st += 2;
        if (st == ring) {
            st = 0;
            ph ^= 1u;
        }
        emit(A, j, t.x * inv_h, t.y * inv_h);
        if (two) emit(B, j + 1, t.z * inv_h, t.w * inv_h);
    }
    float* dst = part + (size_t)blockIdx.x * 4 * h;
    st_f4(dst + c, make_float4(adg[0], adg[1], adg[2], adg[3]));
    st_f4(dst + c + 4, make_float4(adg[4], adg[5], adg[6], adg[7]));
    st_f4(dst + h + c, make_float4(adb[0], adb[1], adb[2], adb[3]));
    st_f4(dst + h + c + 4, make_float4(adb[4], adb[5], adb[6], adb[7]));
    if (kColRes) {
        st_f4(dst + 2 * h + c, make_float4(ares[0], ares[1], ares[2], ares[3]));
        st_f4(dst + 2 * h + c + 4, make_float4(ares[4], ares[5], ares[6], ares[7]));
    }
    if (kColDx) {
        st_f4(dst + 3 * h + c, make_float4(adx[0], adx[1], adx[2], adx[3]));
        st_f4(dst + 3 * h + c + 4, make_float4(adx[4], adx[5], adx[6], adx[7]));
    }
}

// out_k[n] = bf16(sum over r < R of part[r][k*h + n]) for the nseg segments of width h.
// CTA = 8 float4 column groups (32 columns) x 64 row lanes, 8 independent row loads in flight
// per thread; row lanes are combined with warp shuffles (4 per warp) and then across the 16
// warps in smem. Every step has a fixed order, so the result is deterministic.
struct SegOut {
    uint16_t* p[4];
};
__global__ void __launch_bounds__(512) ln_finish_kernel(const float* __restrict__ part, int R, int ld, int h, int nseg,
                                                        SegOut out) {
    __shared__ float4 red[16][8];
    const int cg = threadIdx.x & 7, rl = threadIdx.x >> 3;  // rl: 0..63
    pdl_launch_dependents();
    pdl_wait();
    const int n = (blockIdx.x * 8 + cg) * 4;
    const int N = nseg * h;
    float4 acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n < N) {
        for (int r = rl; r < R; r += 512) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (r + 64 * u < R) {
                    const float4 v = *reinterpret_cast<const float4*>(part + (size_t)(r + 64 * u) * ld + n);
                    acc[u].x += v.x;
                    acc[u].y += v.y;
                    acc[u].z += v.z;
                    acc[u].w += v.w;
                }
            }
        }
    }
    float4 t = acc[0];
#pragma unroll
    for (int u = 1; u < 8; ++u) {
        t.x += acc[u].x;
        t.y += acc[u].y;
        t.z += acc[u].z;
        t.w += acc[u].w;
    }
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {  // the warp's 4 row lanes of this column group
        t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
        t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
        t.z += __shfl_xor_sync(0xffffffffu, t.z, o);
        t.w += __shfl_xor_sync(0xffffffffu, t.w, o);
    }
    if ((threadIdx.x & 31) < 8) red[threadIdx.x >> 5][cg] = t;
    __syncthreads();
    if (threadIdx.x < 8 && n < N) {
        float4 a = red[0][cg];
        for (int q = 1; q < 16; ++q) {
            a.x += red[q][cg].x;
            a.y += red[q][cg].y;
            a.z += red[q][cg].z;
            a.w += red[q][cg].w;
        }
        const int k = n / h;  // h % 4 == 0: the 4 columns stay in one segment
        uint16_t* o = out.p[k] + (n - k * h);
        o[0] = (uint16_t)f32_to_bf16_bits(a.x);
        o[1] = (uint16_t)f32_to_bf16_bits(a.y);
        o[2] = (uint16_t)f32_to_bf16_bits(a.z);
        o[3] = (uint16_t)f32_to_bf16_bits(a.w);
    }
}

// One full wave: CTAs = SMs x resident CTAs per SM (capped by the partials buffer), so no SM
// runs a second, partial round of row chunks.
template <bool R, bool CR, bool CX>
int launch_bwd(cudaStream_t st, const uint16_t* dy, const uint16_t* x, const float* mean, const float* rstd,
               const uint16_t* g, const uint16_t* dres, uint16_t* dx, float* part, int T, int h) {
    auto kern = ln_bwd_rows_kernel<R, CR, CX>;
    static bool attr = [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        return true;
    }();
    (void)attr;
    const int threads = h / 8, nt = R ? 3 : 2;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, RingPlan(h, nt, (T + kNumSMs - 1) / kNumSMs).total);
    const int cap = ln_bwd_ctas(T), ctas = std::min(cap, kNumSMs * std::max(1, occ));
    const int rows = (T + ctas - 1) / ctas, grid = (T + rows - 1) / rows;
    launch_ex(kern, dim3(grid), dim3(threads), RingPlan(h, nt, rows).total, st, 1, dy, x, mean, rstd, g, dres, dx, part, T,
              h, rows);
    return grid;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

bool ln_rows_supported(int h) { return h % 256 == 0 && h / 8 <= 768; }

cudaError_t ln_fwd_rows(const uint16_t* x, const uint16_t* g, const uint16_t* b, uint16_t* y, float* mean,
                        float* rstd, int T, int h, cudaStream_t st) {
    if (T <= 0) return cudaSuccess;
    switch (h) {  // register-resident warp-per-row forms for the common widths
        case 768: launch_ex(ln_fwd_warp_kernel<3>, dim3((T + 7) / 8), dim3(256), 0, st, 1, x, g, b, y, mean, rstd, T); return launched(1);
        case 1024: launch_ex(ln_fwd_warp_kernel<4>, dim3((T + 7) / 8), dim3(256), 0, st, 1, x, g, b, y, mean, rstd, T); return launched(1);
        case 2048: launch_ex(ln_fwd_warp_kernel<8>, dim3((T + 7) / 8), dim3(256), 0, st, 1, x, g, b, y, mean, rstd, T); return launched(1);
        case 4096: launch_ex(ln_fwd_warp_kernel<16>, dim3((T + 7) / 8), dim3(256), 0, st, 1, x, g, b, y, mean, rstd, T); return launched(1);
        // 10B width: 24 x 16-B loads per lane (253 registers, no spill): 44.6 vs 61.9 us for the
        // ring kernel at 8192 x 6144 (4.5 vs 3.3 TB/s); at 8192 columns the row no longer fits
        case 6144: launch_ex(ln_fwd_warp_kernel<24>, dim3((T + 7) / 8), dim3(256), 0, st, 1, x, g, b, y, mean, rstd, T); return launched(1);
        default: break;
    }
    const int threads = h / 8;
    if (!aligned16(x) || !aligned16(y)) return cudaErrorMisalignedAddress;  // bulk copies need 16-B rows
    static bool attr = [] {
        cudaFuncSetAttribute(ln_fwd_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        return true;
    }();
    (void)attr;
    const RingPlan plan(h, 1, 0);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ln_fwd_rows_kernel, threads, plan.total);
    const int want = kNumSMs * std::max(1, occ);
    const int rows = (T + want - 1) / want;
    launch_ex(ln_fwd_rows_kernel, dim3((T + rows - 1) / rows), dim3(threads), plan.total, st, 1, x, g, b, y, mean, rstd, T, h,
              rows);
    return launched(1);
}

cudaError_t ln_bwd_rows(const uint16_t* dy, const uint16_t* x, const float* mean, const float* rstd,
                        const uint16_t* g, const uint16_t* dres, uint16_t* dx, uint16_t* dgdb, uint16_t* dres_colsum,
                        uint16_t* dx_colsum, float* part, int T, int h, cudaStream_t st) {
    if (T <= 0) return cudaSuccess;
    if (!aligned16(dy) || !aligned16(x) || !aligned16(dx) || (dres && !aligned16(dres))) return cudaErrorMisalignedAddress;
    const bool r = dres != nullptr, cr = r && dres_colsum != nullptr, cx = dx_colsum != nullptr;
    int grid;
    if (!r && !cx)
        grid = launch_bwd<false, false, false>(st, dy, x, mean, rstd, g, dres, dx, part, T, h);
    else if (!r && cx)
        grid = launch_bwd<false, false, true>(st, dy, x, mean, rstd, g, dres, dx, part, T, h);
    else if (!cr && !cx)
        grid = launch_bwd<true, false, false>(st, dy, x, mean, rstd, g, dres, dx, part, T, h);
    else if (!cr && cx)
        grid = launch_bwd<true, false, true>(st, dy, x, mean, rstd, g, dres, dx, part, T, h);
    else if (!cx)
        grid = launch_bwd<true, true, false>(st, dy, x, mean, rstd, g, dres, dx, part, T, h);
    else
        grid = launch_bwd<true, true, true>(st, dy, x, mean, rstd, g, dres, dx, part, T, h);
    // segments: dgamma | dbeta (contiguous in dgdb) | colsum(dres) | colsum(dx)
    SegOut out{{dgdb, dgdb + h, nullptr, nullptr}};
    int nseg = 2;
    if (cr) out.p[nseg++] = dres_colsum;
    if (cx) {
        if (!cr) {  // keep segment index == part column block: finish segment 3 separately
            launch_ex(ln_finish_kernel, dim3((2 * h + 31) / 32), dim3(512), 0, st, 1, part, grid, 4 * h, h, 2, out);
            SegOut o2{{dx_colsum, nullptr, nullptr, nullptr}};
            launch_ex(ln_finish_kernel, dim3((h + 31) / 32), dim3(512), 0, st, 1, (const float*)(part + 3 * h), grid, 4 * h, h, 1,
                      o2);
            return launched(3);
        }
        out.p[nseg++] = dx_colsum;
    }
    launch_ex(ln_finish_kernel, dim3((nseg * h + 31) / 32), dim3(512), 0, st, 1, part, grid, 4 * h, h, nseg, out);
    return launched(2);
}

}  // namespace gpt
}  // namespace ah
