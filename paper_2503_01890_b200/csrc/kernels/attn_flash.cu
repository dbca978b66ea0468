// Flash-style causal attention on tcgen05 (sm_100a): the forward keeps only O and the per-row
// log-sum-exp; the backward recomputes P from Q, K and the log-sum-exp.
//
// Forward (flash_fwd_k64_kernel): persistent, two CTAs per SM, each walking snake-ordered
// (128-query tile, head, sequence) items, heavy (long causal) items first:
//   S_j = Q K_j^T            128 queries x 64 keys, tcgen05.mma into one of two TMEM score buffers
//                             (S_{j+1} is computed while the softmax works on S_j)
//   online softmax            4 warps, thread = query row (row_chunk: 32-key chunks, one TMEM read
//                             per score, paired FFMA2 / FADD2, a quarter of the exponentials on the
//                             FMA pipe)
//   O += P_j V_j              P_j (bf16) written back into its score buffer, A read from TMEM
// Softmax runs in the log2 domain, p = 2^(S * scale * log2e - m), with lazy rescaling: the running
// max m only moves (and l / O / the tile's stored P chunks are rescaled) when a chunk max exceeds
// it by more than 2^8. Output O / l and lse2 = m + log2(l) per row (the backward's statistics).
//
// Backward (flash_bwd_t_kernel): persistent over (128-key tile, head, sequence) items, scores
// formed key-major so P^T and dS^T are the TMEM A operands of the dV / dK MMAs:
//   S^T = K Q_i^T, P^T = 2^(S^T * scale * log2e - lse2_i)      (recomputed, never stored)
//   dP^T = V dO_i^T; dS^T = P^T * (dP^T - D_i)                 (D = rowsum(dO * O))
//   dV += P^T dO_i, dK += dS^T Q_i                             (TMEM accumulators)
// dS^T also goes to HBM for the deterministic dQ = dS K GEMM (no cross-CTA atomics).
//
// Operand staging: every tile is a K-major SWIZZLE_128B box pair (two 64-column atoms; 128 rows,
// 64 for the forward's K / V); read as the MN-major operand of its transpose it gives V, dO, Q for
// free. Backward warp roles: 0 TMA producer, 1 MMA issuer (one thread), 2 TMEM allocator, 4..
// softmax / epilogue.
// Shapes: head_dim = 128, seq_len % 128 == 0 (others take the unfused GEMM path, gpt_model.cpp).
#include <cuda.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "gpt_kernels.h"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace ah {
namespace gpt {
namespace {

using namespace ah::tc;

constexpr int kHD = 128, kT = 128;
constexpr uint32_t kTile = kT * kHD * 2;  // 32 KB
constexpr int kThreads = 384;
constexpr float kRescaleLog2 = 8.f;       // lazy rescale threshold (p <= 2^8 between rescales)

// K-major SWIZZLE_128B operand, K step t (16 elements) of a 128-wide tile.
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int t) {
    return sdesc(base + (t >> 2) * (kTile / 2) + (t & 3) * 32, 16, 1024);
}
// The same tile read as the MN-major operand of its transpose: K step t = 16 stored rows.
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int t) { return sdesc(base + t * 2048, kTile / 2, 1024); }

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

__device__ __forceinline__ void load_tile(uint32_t dst, const CUtensorMap* m, uint32_t bar, int row, int head, int b) {
    tma_load_4d(dst, m, bar, 0, row, head, b);
    tma_load_4d(dst + kTile / 2, m, bar, 64, row, head, b);
}

__device__ __forceinline__ void ld64(uint32_t taddr, float (&v)[64]) {
    ld32(taddr, *reinterpret_cast<float(*)[32]>(v));
    ld32(taddr + 32, *reinterpret_cast<float(*)[32]>(v + 32));
}

struct FwdParams {
    int s, nh, B, h;
    float sl2;        // softmax scale * log2(e)
    uint16_t* O;      // [B][s][h], head slice at head * hd
    float* lse2;      // [B][nh][s]
};


// ---------------------------------------------------------------------------------------
// Persistent forward pipeline: a CTA walks a snake-ordered list of (query tile, head, sequence)
// items, heavy (long causal) items first, and keeps the pipeline full across items: the K/V ring
// and the two TMEM score buffers continue across item boundaries, and the next item's first score
// tile is issued while the softmax warps run the current item's epilogue. P_j (bf16) is written
// back by the softmax warps into its own score buffer and fed to O += P_j V_j straight from TMEM
// (tcgen05.mma A-from-TMEM), so P never touches shared memory and softmax j+1 never waits for the
// P V MMA of tile j (the score buffer of j is only reused by S_{j+2}, which the MMA thread issues
// after P_j V_j: tcgen05.mma executes in issue order). O += P V with A from TMEM:
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

struct FwdItems {
    int nqt, nh, B, total, G, c;
    __device__ int count() const {  // items of CTA c
        const int full = total / G, rem = total % G;
        int k = full;
        if (rem) k += ((full & 1) == 0 ? c < rem : (G - 1 - c) < rem) ? 1 : 0;
        return k;
    }
    __device__ void get(int k, int& qt, int& head, int& b) const {  // k-th item of CTA c (snake order)
        const int w = k * G + ((k & 1) == 0 ? c : G - 1 - c);
        const int per = nh * B;
        qt = nqt - 1 - w / per;
        const int rem = w % per;
        head = rem % nh;
        b = rem / nh;
    }
};

// ---------------------------------------------------------------------------------------
// Row-per-thread softmax of the forward: a thread owns one query row and the keys of a score
// tile, read from TMEM in 32-key chunks (one TMEM read per score). The
// exponentials use the running row max (lazy rescale: p <= 2^8 between rescales) while each
// chunk's max is checked; a chunk whose max exceeds it by more than 2^8 takes the out-of-line
// slow path (new max; l, the tile's partial sums, its stored P chunks and O rescaled). P chunk c
// (bf16 pairs) lands in score columns [16c, 16c + 16), already read. A quarter of the
// exponentials run on the FMA pipe (ex2_poly) and the scale / sum arithmetic is paired (FFMA2 /
// FADD2): the loop is MUFU- and issue-bound. The chunk loop is rolled so the whole softmax code
// stays in the instruction cache (fully unrolled variants ran chunks 2-5x slower whenever
// warps executed different variants).

// 2^x on the FMA pipe for x in [-120, 9]: x = n + f (n = round(x), |f| <= 1/2), 2^f by a degree-3
// near-minimax polynomial (max rel. error 7.5e-5, far below the bf16 rounding of P), 2^n added to
// the exponent field. Masked keys never take this path (they need an exact 0).
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -120.f);
    const float t = x + 12582912.f;  // 1.5 * 2^23: round(x) in the low mantissa bits
    const float f = x - (t - 12582912.f);
    float p = fmaf(0.05517052f, f, 0.24260917f);
    p = fmaf(p, f, 0.69326102f);
    p = fmaf(p, f, 0.9999282f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ void ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t x[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]), "=r"(x[8]),
          "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(x[i]);
}

// Slow path (rare): P chunks [0, c) of this tile and O times alpha. O must hold every P V issued
// for this item: the one of the previous tile may still run (S_{j+1} is issued before P_j V_j).
__device__ __noinline__ void row_rescale(float alpha, int c, uint32_t sbuf, uint32_t obuf, int j, uint32_t pv_bar,
                                         uint32_t g) {
#pragma unroll 1
    for (int cc = 0; cc < c; ++cc) {
        float pw[16];
        ld16(sbuf + cc * 16, pw);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const uint32_t u = __float_as_uint(pw[i]);
            pw[i] = __uint_as_float(pack_bf16x2_rn(__uint_as_float(u << 16) * alpha, __uint_as_float(u & 0xffff0000u) * alpha));
        }
        st16(sbuf + cc * 16, pw);
    }
    if (j > 0) {
        mbar_wait(pv_bar, (g - 1) & 1);
        fence_after();
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
            float o[32];
            ld32(obuf + cc * 32, o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            st32(obuf + cc * 32, o);
        }
    }
}

// kMask: the diagonal chunk (keys > row masked to an exact 0); kPoly: ex2 of a quarter on the FMA pipe.
template <bool kMask, bool kPoly>
__device__ __forceinline__ void row_chunk(int c, uint32_t sbuf, uint32_t obuf, int lane, int j, uint32_t g, float sl2,
                                          float& mb, float& l, unsigned long long (&ad2)[2], uint32_t pv_bar) {
    float v[32];
    ld32(sbuf + c * 32, v);
    float cm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        if (kMask && i > lane) v[i] = -INFINITY;
        cm[i & 3] = fmaxf(cm[i & 3], v[i]);
    }
    const float ym = fmaxf(fmaxf(cm[0], cm[1]), fmaxf(cm[2], cm[3])) * sl2;  // chunk max, scaled
    if (mb == -INFINITY) mb = ym;  // the item's first chunk (key 0 <= q: finite)
    const bool up = ym - mb > kRescaleLog2;
    if (__any_sync(0xffffffffu, up)) {
        const float alpha = up ? ex2_approx(mb - ym) : 1.f;
        row_rescale(alpha, c, sbuf, obuf, j, pv_bar, g);
        if (up) mb = ym;
        l *= alpha;
        const unsigned long long a2 = f2pack(alpha, alpha);
        ad2[0] = fmul2(ad2[0], a2);
        ad2[1] = fmul2(ad2[1], a2);
    }
    const unsigned long long s2 = f2pack(sl2, sl2), nb2 = f2pack(-mb, -mb);
    float pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        float x0, x1;
        f2unpack(ffma2(f2pack(v[2 * i], v[2 * i + 1]), s2, nb2), x0, x1);
        const bool poly = kPoly && (i & 3) == 3;
        const float p0 = poly ? ex2_poly(x0) : ex2_approx(x0), p1 = poly ? ex2_poly(x1) : ex2_approx(x1);
        ad2[i & 1] = fadd2(ad2[i & 1], f2pack(p0, p1));
        pk[i] = __uint_as_float(pack_bf16x2_rn(p0, p1));
    }
    st16(sbuf + c * 16, pk);
}

// ---------------------------------------------------------------------------------------
// Forward with 64-key score tiles, two CTAs per SM. Each CTA is a single-query-tile pipeline
// (persistent over snake-ordered items, S double-buffered ahead of P V), a score tile is 128 queries x 64 keys, so a CTA needs
// only 256 TMEM columns (S double-buffered: 0-63, 64-127; O: 128-255) and ~106 KB of shared
// memory, and two CTAs share every SM. The softmax is row-per-thread (row_chunk: one TMEM read
// per score, lazy max, paired arithmetic, a quarter of the exponentials on the FMA pipe) with 4
// warps per CTA, so each SM sub-partition runs two independent softmax warps (one per CTA)
// while the tensor pipe serves both CTAs: one warp alone cannot hide its own TMEM / MUFU
// latencies (a row-per-thread 128-key variant with one CTA per SM measured 54.7 us; the previous
// forward, two warps per row exchanging the row max through shared memory, 51.4 us; this one 48.7).
constexpr int kKT = 64;                                  // keys per score tile
constexpr uint32_t kTileKV = kKT * kHD * 2;             // 16 KB: two 64-column SWIZZLE_128B atoms
__device__ __forceinline__ uint64_t kdesc_kv(uint32_t base, int t) {  // K (64 rows) as K-major B
    return sdesc(base + (t >> 2) * (kTileKV / 2) + (t & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t mndesc_kv(uint32_t base, int t) {  // V (64 rows) as MN-major B, K step t
    return sdesc(base + t * 2048, kTileKV / 2, 1024);
}
__device__ __forceinline__ void load_kv(uint32_t dst, const CUtensorMap* m, uint32_t bar, int row, int head, int b) {
    tma_load_4d(dst, m, bar, 0, row, head, b);
    tma_load_4d(dst + kTileKV / 2, m, bar, 64, row, head, b);
}

__global__ void __launch_bounds__(192, 2)
flash_fwd_k64_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, const FwdParams A) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = align1024(smem_raw);
    uint8_t* sQ = sm;                          // one Q tile (32 KB)
    uint8_t* sK = sm + kTile;                  // [2] x 16 KB
    uint8_t* sV = sm + kTile + 2 * kTileKV;    // [2] x 16 KB
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kTile + 4 * kTileKV);
    uint64_t* q_full = bar;
    uint64_t* q_empty = bar + 1;
    uint64_t* k_full = bar + 2;    // [2]
    uint64_t* k_empty = bar + 4;   // [2]
    uint64_t* v_full = bar + 6;    // [2]
    uint64_t* v_empty = bar + 8;   // [2]
    uint64_t* s_full = bar + 10;   // [2]
    uint64_t* s_free = bar + 12;   // [2]
    uint64_t* p_full = bar + 14;   // [2] (by tile parity, see the kernel above)
    uint64_t* o_full = bar + 16;
    uint64_t* o_free = bar + 17;
    uint64_t* pv_done = bar + 18;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bar + 19);
    uint8_t* slabs = sm + kTile + 4 * kTileKV + 1024;  // 4 softmax warps x 2 KB (32 x 32 bf16, SWIZZLE_64B)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    FwdItems items{A.s / kT, A.nh, A.B, (A.s / kT) * A.nh * A.B, (int)gridDim.x, (int)blockIdx.x};
    const int n_items = items.count();

    if (warp == 0) {
        if (lane == 0) {
            for (const CUtensorMap* m : {&tmQ, &tmK, &tmV})
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
            mbar_init(smem_u32(q_full), 1);
            mbar_init(smem_u32(q_empty), 1);
            for (int i = 0; i < 2; ++i) {
                mbar_init(smem_u32(&k_full[i]), 1);
                mbar_init(smem_u32(&k_empty[i]), 1);
                mbar_init(smem_u32(&v_full[i]), 1);
                mbar_init(smem_u32(&v_empty[i]), 1);
                mbar_init(smem_u32(&s_full[i]), 1);
                mbar_init(smem_u32(&s_free[i]), 4);
                mbar_init(smem_u32(&p_full[i]), 4);
            }
            mbar_init(smem_u32(o_full), 1);
            mbar_init(smem_u32(o_free), 4);
            mbar_init(smem_u32(pv_done), 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncwarp();
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_holder;  // S/P[0] 0-63, S/P[1] 64-127, O 128-255
    pdl_launch_dependents();
    pdl_wait();

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer: Q per item, K / V per 64-key tile =====
            uint32_t g = 0;
            for (int it = 0; it < n_items; ++it) {
                int qt, head, b;
                items.get(it, qt, head, b);
                mbar_wait(smem_u32(q_empty), ((uint32_t)it & 1) ^ 1);
                mbar_expect_tx(smem_u32(q_full), kTile);
                load_tile(smem_u32(sQ), &tmQ, smem_u32(q_full), qt * kT, head, b);
                const int nk = 2 * qt + 2;
                for (int j = 0; j < nk; ++j, ++g) {
                    const int st = g & 1;
                    const uint32_t ph = (g >> 1) & 1;
                    mbar_wait(smem_u32(&k_empty[st]), ph ^ 1);
                    mbar_expect_tx(smem_u32(&k_full[st]), kTileKV);
                    load_kv(smem_u32(sK + st * kTileKV), &tmK, smem_u32(&k_full[st]), j * kKT, head, b);
                    mbar_wait(smem_u32(&v_empty[st]), ph ^ 1);
                    mbar_expect_tx(smem_u32(&v_full[st]), kTileKV);
                    load_kv(smem_u32(sV + st * kTileKV), &tmV, smem_u32(&v_full[st]), j * kKT, head, b);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer: S(g+1) ahead of P(g) V(g), across items =====
            constexpr uint32_t idS = idesc_bf16(128, kKT, 0, 0);  // Q (K-major) x K^T (K-major)
            constexpr uint32_t idO = idesc_bf16(128, 128, 0, 1);  // P (TMEM, K-major) x V (MN-major)
            int s_it = 0, s_j = 0, s_nk = 0;
            uint32_t s_g = 0;
            auto issue_next_S = [&]() {
                const int st = s_g & 1;
                const uint32_t ph = (s_g >> 1) & 1;
                if (s_j == 0) {
                    int qt_, h_, b_;
                    items.get(s_it, qt_, h_, b_);
                    s_nk = 2 * qt_ + 2;
                    mbar_wait(smem_u32(q_full), (uint32_t)s_it & 1);
                }
                mbar_wait(smem_u32(&k_full[st]), ph);
                mbar_wait(smem_u32(&s_free[st]), ph ^ 1);
                fence_after();
                const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK + st * kTileKV);
#pragma unroll
                for (int t = 0; t < 8; ++t) mma_f16(tmem + st * kKT, kdesc(qa, t), kdesc_kv(ka, t), idS, t > 0);
                commit(smem_u32(&s_full[st]));
                commit(smem_u32(&k_empty[st]));
                if (++s_j == s_nk) {  // the item's last score tile: its Q buffer is free after this MMA
                    commit(smem_u32(q_empty));
                    s_j = 0;
                    ++s_it;
                }
                ++s_g;
            };
            if (n_items > 0) issue_next_S();
            uint32_t g = 0;
            for (int it = 0; it < n_items; ++it) {
                int qt, head, b;
                items.get(it, qt, head, b);
                const int nk = 2 * qt + 2;
                for (int j = 0; j < nk; ++j, ++g) {
                    if (s_it < n_items) issue_next_S();  // scores of the next tile overlap softmax of this one
                    const int st = g & 1;
                    if (j == 0 && it >= 1) mbar_wait(smem_u32(o_free), ((uint32_t)it - 1) & 1);  // O drained
                    mbar_wait(smem_u32(&p_full[st]), (g >> 1) & 1);
                    mbar_wait(smem_u32(&v_full[st]), (g >> 1) & 1);
                    fence_after();
                    const uint32_t va = smem_u32(sV + st * kTileKV);
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        mma_f16_ts(tmem + 128, tmem + st * kKT + t * 8, mndesc_kv(va, t), idO, (j > 0 || t > 0) ? 1u : 0u);
                    commit(smem_u32(pv_done));
                    commit(smem_u32(&v_empty[st]));
                }
                commit(smem_u32(o_full));
            }
        }
    } else {  // ===== softmax / epilogue (warps 2-5), thread = query row 32 * quarter + lane =====
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = uint32_t(quarter * 32) << 16;
        const uint32_t obuf = tmem + lane_base + 128;
        const float sl2 = A.sl2;
        uint8_t* slab = slabs + (warp - 2) * 2048;
        uint32_t g = 0;
        int pend_it = -1;
        float pend_inv = 0.f;
        int pend_col = 0, pend_row0 = 0;
        auto epilogue = [&]() {
            mbar_wait(smem_u32(o_full), (uint32_t)pend_it & 1);
            fence_after();
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                float v[32];
                ld32(obuf + c * 32, v);
                const float inv = pend_inv;
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slab free
                __syncwarp();
#pragma unroll
                for (int k8 = 0; k8 < 4; ++k8)
                    *reinterpret_cast<uint4*>(slab + lane * 64 + ((k8 ^ ((lane >> 1) & 3)) << 4)) =
                        make_uint4(pack_bf16x2_rn(v[8 * k8] * inv, v[8 * k8 + 1] * inv), pack_bf16x2_rn(v[8 * k8 + 2] * inv, v[8 * k8 + 3] * inv),
                                   pack_bf16x2_rn(v[8 * k8 + 4] * inv, v[8 * k8 + 5] * inv), pack_bf16x2_rn(v[8 * k8 + 6] * inv, v[8 * k8 + 7] * inv));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                     reinterpret_cast<uint64_t>(&tmO)),
                                 "r"(smem_u32(slab)), "r"(pend_col + c * 32), "r"(pend_row0)
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(o_free));
            pend_it = -1;
        };
        for (int it = 0; it < n_items; ++it) {
            int qt, head, b;
            items.get(it, qt, head, b);
            const int q = qt * kT + r;
            const int nk = 2 * qt + 2;
            float mb = -INFINITY, l = 0.f;
            for (int j = 0; j < nk; ++j, ++g) {
                const int st = g & 1;
                mbar_wait(smem_u32(&s_full[st]), (g >> 1) & 1);
                fence_after();
                const uint32_t sbuf = tmem + lane_base + st * kKT;
                unsigned long long ad2[2] = {0ull, 0ull};
#pragma unroll 1
                for (int c = 0; c < 2; ++c) {
                    const int cd = 2 * (j - 2 * qt) + c;  // 32-key chunk within the diagonal 128-key block (< 0: below it)
                    if (cd < quarter)
                        row_chunk<false, true>(c, sbuf, obuf, lane, j, g, sl2, mb, l, ad2, smem_u32(pv_done));
                    else if (cd == quarter)
                        row_chunk<true, false>(c, sbuf, obuf, lane, j, g, sl2, mb, l, ad2, smem_u32(pv_done));
                    else {  // keys after this row quarter: all masked
                        float z[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) z[i] = 0.f;
                        st16(sbuf + c * 16, z);
                    }
                }
                float a0, a1, a2, a3;
                f2unpack(ad2[0], a0, a1);
                f2unpack(ad2[1], a2, a3);
                l += (a0 + a1) + (a2 + a3);
                fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(smem_u32(&s_free[st]));
                    mbar_arrive(smem_u32(&p_full[st]));
                }
                if (j == 0 && pend_it >= 0) epilogue();  // previous item: its last P V was issued before this P
            }
            A.lse2[((size_t)b * A.nh + head) * A.s + q] = mb + __log2f(l);
            pend_it = it;
            pend_inv = 1.f / l;
            pend_col = head * kHD;
            pend_row0 = b * A.s + qt * kT + quarter * 32;
        }
        if (pend_it >= 0) epilogue();
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // O written
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    }
}

struct BwdParams {
    int s, nh, B, h;
    float sl2, scale;
    const float* lse2;  // [B][nh][s]
    const float* D;     // [B][nh][s]
    uint16_t* dS;       // [B][nh][s][s]
    uint16_t* dqkv;     // [B][s][3h]
};


// ---------------------------------------------------------------------------------------
// Persistent backward schedule: one CTA per SM walks a snake-ordered list of (key tile, head,
// sequence) items, heavy (many query tiles) first.
struct BwdItems {
    int nt, nh, B, total, G, c;
    __device__ int count() const {
        const int full = total / G, rem = total % G;
        int k = full;
        if (rem) k += ((full & 1) == 0 ? c < rem : (G - 1 - c) < rem) ? 1 : 0;
        return k;
    }
    __device__ void get(int k, int& kt, int& head, int& b) const {
        const int w = k * G + ((k & 1) == 0 ? c : G - 1 - c);
        const int per = nh * B;
        kt = w / per;  // 0 = the most query tiles
        const int rem = w % per;
        head = rem % nh;
        b = rem / nh;
    }
};


// ---------------------------------------------------------------------------------------
// Transposed persistent backward (the default). Per (key tile, head, sequence) item and query
// tile i, the scores are formed key-major, S^T = K Q_i^T and dP^T = V dO_i^T, so a softmax
// thread owns one KEY row and the per-query statistics (lse2, D) are 128-float vectors that the
// producer streams into shared memory next to Q_i / dO_i. P^T and dS^T are then exactly the
// K-major A operands of dV += P^T dO_i and dK += dS^T Q_i: each half-warp writes its 64 query
// columns (bf16 pairs) into the first 32 TMEM columns of its own half of the S^T / dP^T buffer
// and the MMAs read A straight from TMEM — no shared-memory staging of P / dS, no cross-half
// barrier (tcgen05.mma executes in issue order, so S^T_{i+1} / dP^T_{i+1} are issued after the
// dV_i / dK_i that read the same columns). dS^T also goes to HBM for the deterministic
// dQ = (dS^T)^T K GEMM (MN-major A). TMEM: S^T 0-127, dP^T 128-255, dV 256-383, dK 384-511.
// (A variant staging P^T through a K-major smem tile so S^T_{i+1} could run before dV_i measured
// 151 us vs 129 us for this one at B=8, s=1024, 16 heads.)
// TMEM A operand of K step t (16 queries) inside a score buffer at column `base`: half h's
// 64 queries sit in columns [base + 64h, base + 64h + 32).
__device__ __forceinline__ void bulk_g2s_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ uint32_t tsA(uint32_t base, int t) { return base + (t >> 2) * 64 + (t & 3) * 8; }

__global__ void __launch_bounds__(kThreads, 1)
flash_bwd_t_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                   const __grid_constant__ CUtensorMap tmdS, const __grid_constant__ CUtensorMap tmdQKV,
                   const BwdParams A) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = align1024(smem_raw);
    // dS^T (and the dV / dK epilogue) leaves through per-warp 32 x 64 smem slabs and TMA bulk stores when the dynamic smem
    // base is 1024-aligned (the request has no alignment slack left for the slabs); otherwise
    // each thread stores its 128-byte row directly
    const bool tma_ds = sm == smem_raw;
    uint8_t* slabs = sm + 6 * kTile + 3072;  // [8 softmax warps][32 rows x 128 B], SWIZZLE_128B images
    uint8_t* sK = sm;
    uint8_t* sV = sm + kTile;
    uint8_t* sQ = sm + 2 * kTile;   // [2]
    uint8_t* sdO = sm + 4 * kTile;  // [2]
    float* sStat = reinterpret_cast<float*>(sm + 6 * kTile);  // [2 stages][lse2 128 | D 128]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 6 * kTile + 2048);
    uint64_t* kv_full = bar;
    uint64_t* kv_empty = bar + 1;
    uint64_t* st_full = bar + 2;   // [2]
    uint64_t* st_empty = bar + 4;  // [2]
    uint64_t* s_full = bar + 6;
    uint64_t* s_free = bar + 7;
    uint64_t* dp_full = bar + 8;
    uint64_t* dp_free = bar + 9;
    uint64_t* p_full = bar + 10;
    uint64_t* ds_full = bar + 11;
    uint64_t* acc_full = bar + 12;
    uint64_t* acc_free = bar + 13;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bar + 14);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt = A.s / kT;
    BwdItems items{nt, A.nh, A.B, nt * A.nh * A.B, (int)gridDim.x, (int)blockIdx.x};
    const int n_items = items.count();

    if (warp == 0 && lane == 0) {
        for (const CUtensorMap* m : {&tmQ, &tmK, &tmV, &tmdO})
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
        mbar_init(smem_u32(kv_full), 1);
        mbar_init(smem_u32(kv_empty), 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&st_full[i]), 1);
            mbar_init(smem_u32(&st_empty[i]), 1);
        }
        mbar_init(smem_u32(s_full), 1);
        mbar_init(smem_u32(s_free), 8);
        mbar_init(smem_u32(dp_full), 1);
        mbar_init(smem_u32(dp_free), 8);
        mbar_init(smem_u32(p_full), 8);
        mbar_init(smem_u32(ds_full), 8);
        mbar_init(smem_u32(acc_full), 1);
        mbar_init(smem_u32(acc_free), 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_holder;
    pdl_launch_dependents();  // setup above overlapped the previous kernel (PDL); data from here on
    pdl_wait();

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer: K, V per item; Q, dO per query tile =====
            uint32_t g = 0;
            for (int it = 0; it < n_items; ++it) {
                int kt, head, b;
                items.get(it, kt, head, b);
                if (it > 0) mbar_wait(smem_u32(kv_empty), (it - 1) & 1);
                mbar_expect_tx(smem_u32(kv_full), 2 * kTile);
                load_tile(smem_u32(sK), &tmK, smem_u32(kv_full), kt * kT, head, b);
                load_tile(smem_u32(sV), &tmV, smem_u32(kv_full), kt * kT, head, b);
                const size_t srow = ((size_t)b * A.nh + head) * A.s;
                for (int qi = kt; qi < nt; ++qi, ++g) {
                    const int st = g & 1;
                    mbar_wait(smem_u32(&st_empty[st]), ((g >> 1) & 1) ^ 1);
                    const uint32_t fb = smem_u32(&st_full[st]);
                    mbar_expect_tx(fb, 2 * kTile + 1024);
                    load_tile(smem_u32(sQ + st * kTile), &tmQ, fb, qi * kT, head, b);
                    load_tile(smem_u32(sdO + st * kTile), &tmdO, fb, qi * kT, head, b);
                    bulk_g2s_1d(smem_u32(sStat + st * 256), A.lse2 + srow + (size_t)qi * kT, 512, fb);
                    bulk_g2s_1d(smem_u32(sStat + st * 256 + 128), A.D + srow + (size_t)qi * kT, 512, fb);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer: S^T(g+1), dV(g), dK(g), dP^T(g+1) =====
            constexpr uint32_t idSS = idesc_bf16(128, 128, 0, 0);  // K (K-major) x Q^T (K-major)
            constexpr uint32_t idAB = idesc_bf16(128, 128, 0, 1);  // P^T / dS^T (K-major) x dO / Q (MN-major)
            const uint32_t ka = smem_u32(sK), va = smem_u32(sV);
            // tile sequence of this CTA: g -> (item, first / last tile of the item)
            int c_it = 0, c_i = 0, c_nq = 0;  // cursor of the next S^T to issue
            uint32_t c_g = 0;
            auto cursor_item = [&]() {
                int kt, h_, b_;
                items.get(c_it, kt, h_, b_);
                c_nq = nt - kt;
            };
            auto issue_S = [&]() {  // S^T at the cursor = K Q^T, then advance the cursor
                const uint32_t g = c_g;
                const int st = g & 1;
                if (c_i == 0) mbar_wait(smem_u32(kv_full), c_it & 1);
                mbar_wait(smem_u32(&st_full[st]), (g >> 1) & 1);
                mbar_wait(smem_u32(s_free), (g & 1) ^ 1);
                fence_after();
                const uint32_t qa = smem_u32(sQ + st * kTile);
#pragma unroll
                for (int t = 0; t < 8; ++t) mma_f16(tmem, kdesc(ka, t), kdesc(qa, t), idSS, t > 0);
                commit(smem_u32(s_full));
                ++c_g;
                if (++c_i == c_nq) {
                    c_i = 0;
                    if (++c_it < n_items) cursor_item();
                }
            };
            auto issue_dP = [&](uint32_t g, bool last) {  // dP^T_g = V dO_g^T (last: K / V free after it)
                const int st = g & 1;
                mbar_wait(smem_u32(dp_free), (g & 1) ^ 1);
                fence_after();
                const uint32_t da = smem_u32(sdO + st * kTile);
#pragma unroll
                for (int t = 0; t < 8; ++t) mma_f16(tmem + 128, kdesc(va, t), kdesc(da, t), idSS, t > 0);
                commit(smem_u32(dp_full));
                if (last) commit(smem_u32(kv_empty));
            };
            if (n_items > 0) {
                cursor_item();
                const bool single = c_nq == 1;
                issue_S();
                issue_dP(0, single);
            }
            uint32_t g = 0;
            for (int it = 0; it < n_items; ++it) {
                int kt, head, b;
                items.get(it, kt, head, b);
                const int nq = nt - kt;
                for (int i = 0; i < nq; ++i, ++g) {
                    const int st = g & 1;
                    const uint32_t qa = smem_u32(sQ + st * kTile), da = smem_u32(sdO + st * kTile);
                    if (i == 0 && it > 0) mbar_wait(smem_u32(acc_free), (it - 1) & 1);  // epilogue read dV / dK
                    mbar_wait(smem_u32(p_full), g & 1);
                    fence_after();
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        mma_f16_ts(tmem + 256, tsA(tmem, t), mndesc(da, t), idAB, (i > 0 || t > 0) ? 1u : 0u);
                    if (i + 1 < nq) issue_S();  // P^T_g consumed in order before S^T_{g+1}
                    mbar_wait(smem_u32(ds_full), g & 1);
                    fence_after();
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        mma_f16_ts(tmem + 384, tsA(tmem + 128, t), mndesc(qa, t), idAB, (i > 0 || t > 0) ? 1u : 0u);
                    commit(smem_u32(&st_empty[st]));
                    if (i + 1 < nq) {
                        issue_dP(g + 1, i + 2 == nq);  // dS^T_g consumed in order before dP^T_{g+1}
                    } else {
                        commit(smem_u32(acc_full));
                        if (it + 1 < n_items) {  // first dP^T of the next item overlaps this epilogue
                            int kn, hn, bn;
                            items.get(it + 1, kn, hn, bn);
                            issue_S();
                            issue_dP(g + 1, kn == nt - 1);
                        }
                    }
                }
            }
        }
    } else if (warp >= 4) {  // ===== P^T, dS^T (thread = key row); epilogue =====
        const int half = (warp - 4) >> 2, quarter = warp & 3;  // queries [64 * half, 64 * half + 64)
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = uint32_t(quarter * 32) << 16;
        const float sl2 = A.sl2;
        uint32_t g = 0;
        for (int it = 0; it < n_items; ++it) {
            int kt, head, b;
            items.get(it, kt, head, b);
            const int nq = nt - kt;
            uint16_t* dsrow = A.dS + (((size_t)b * A.nh + head) * A.s + (size_t)kt * kT + r) * A.s + half * 64;
            for (int i = 0; i < nq; ++i, ++g) {
                const int qi = kt + i;
                const float* lse = sStat + (g & 1) * 256 + half * 64;  // 64 queries of this half
                const float* Dv = lse + 128;
                mbar_wait(smem_u32(s_full), g & 1);
                fence_after();
                uint32_t w[32];
                {
                    float v[64];
                    ld64(tmem + lane_base + half * 64, v);
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(s_free));
                    const unsigned long long s2 = f2pack(sl2, sl2);
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float4 l4 = reinterpret_cast<const float4*>(lse)[k];
                        float x0, x1, x2, x3;
                        f2unpack(ffma2(f2pack(v[4 * k], v[4 * k + 1]), s2, f2pack(-l4.x, -l4.y)), x0, x1);
                        f2unpack(ffma2(f2pack(v[4 * k + 2], v[4 * k + 3]), s2, f2pack(-l4.z, -l4.w)), x2, x3);
                        w[2 * k] = pack_bf16x2_rn(ex2_approx(x0), ex2_approx(x1));
                        w[2 * k + 1] = pack_bf16x2_rn(ex2_approx(x2), ex2_approx(x3));
                    }
                }
                if (qi == kt) {  // diagonal tile: P = 0 where the query precedes the key
                    const int lim = r - half * 64;  // keep query columns c >= lim
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        w[k] &= (2 * k >= lim ? 0x0000ffffu : 0u) | (2 * k + 1 >= lim ? 0xffff0000u : 0u);
                }
                st32(tmem + lane_base + half * 64, *reinterpret_cast<float(*)[32]>(w));  // P^T -> TMEM
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(p_full));
                mbar_wait(smem_u32(dp_full), g & 1);
                fence_after();
                uint32_t o[32];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    float v[32];
                    ld32(tmem + lane_base + 128 + half * 64 + c * 32, v);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const float4 d4 = reinterpret_cast<const float4*>(Dv + c * 32)[k];
                        const uint32_t p0 = w[c * 16 + 2 * k], p1 = w[c * 16 + 2 * k + 1];
                        o[c * 16 + 2 * k] = pack_bf16x2_rn(__uint_as_float(p0 << 16) * (v[4 * k] - d4.x),
                                                           __uint_as_float(p0 & 0xffff0000u) * (v[4 * k + 1] - d4.y));
                        o[c * 16 + 2 * k + 1] = pack_bf16x2_rn(__uint_as_float(p1 << 16) * (v[4 * k + 2] - d4.z),
                                                               __uint_as_float(p1 & 0xffff0000u) * (v[4 * k + 3] - d4.w));
                    }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(dp_free));
                st32(tmem + lane_base + 128 + half * 64, *reinterpret_cast<float(*)[32]>(o));  // dS^T -> TMEM
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(ds_full));
                if (tma_ds) {  // dS^T slab -> HBM (dQ GEMM): one bulk tensor store per warp and tile
                    uint8_t* slab = slabs + (warp - 4) * 4096;
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slab free
                    __syncwarp();
#pragma unroll
                    for (int k8 = 0; k8 < 8; ++k8)
                        *reinterpret_cast<uint4*>(slab + lane * 128 + ((k8 ^ (lane & 7)) << 4)) =
                            make_uint4(o[4 * k8], o[4 * k8 + 1], o[4 * k8 + 2], o[4 * k8 + 3]);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile(
                            "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                                reinterpret_cast<uint64_t>(&tmdS)),
                            "r"(smem_u32(slab)), "r"(qi * kT + half * 64), "r"(kt * kT + quarter * 32), "r"(head), "r"(b)
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                } else {
                    uint4* dst = reinterpret_cast<uint4*>(dsrow + (size_t)qi * kT);  // dS^T row -> HBM (dQ GEMM)
#pragma unroll
                    for (int k8 = 0; k8 < 8; ++k8) dst[k8] = make_uint4(o[4 * k8], o[4 * k8 + 1], o[4 * k8 + 2], o[4 * k8 + 3]);
                }
            }
            mbar_wait(smem_u32(acc_full), it & 1);
            fence_after();
            uint16_t* base = A.dqkv + ((size_t)b * A.s + (size_t)kt * kT + r) * 3 * A.h + (size_t)head * kHD + half * 64;
#pragma unroll 1
            for (int which = 0; which < 2; ++which) {  // 0: dV (col 256), 1: dK (col 384)
                uint16_t* dst = base + (which == 0 ? 2 * A.h : A.h);
                const float f = which == 0 ? 1.f : A.scale;
                uint8_t* slab = slabs + (warp - 4) * 4096;
                if (tma_ds) {  // the slab's previous bulk store (dS^T or dV) has been read
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                }
#pragma unroll 1
                for (int c = 0; c < 2; ++c) {
                    float v[32];
                    ld32(tmem + lane_base + 256 + which * 128 + half * 64 + c * 32, v);
#pragma unroll
                    for (int k8 = 0; k8 < 4; ++k8) {
                        const uint4 q = make_uint4(pack_bf16x2_rn(v[8 * k8] * f, v[8 * k8 + 1] * f), pack_bf16x2_rn(v[8 * k8 + 2] * f, v[8 * k8 + 3] * f),
                                                   pack_bf16x2_rn(v[8 * k8 + 4] * f, v[8 * k8 + 5] * f), pack_bf16x2_rn(v[8 * k8 + 6] * f, v[8 * k8 + 7] * f));
                        if (tma_ds)
                            *reinterpret_cast<uint4*>(slab + lane * 128 + (((c * 4 + k8) ^ (lane & 7)) << 4)) = q;
                        else
                            reinterpret_cast<uint4*>(dst + c * 32)[k8] = q;
                    }
                }
                if (tma_ds) {  // 32 key rows x 64 columns of dV / dK -> dqkv, one bulk tensor store
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        const int col = (which == 0 ? 2 * A.h : A.h) + head * kHD + half * 64;
                        asm volatile(
                            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                reinterpret_cast<uint64_t>(&tmdQKV)),
                            "r"(smem_u32(slab)), "r"(col), "r"(b * A.s + kt * kT + quarter * 32)
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(acc_free));
        }
        if (tma_ds && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // dS^T, dV, dK written
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// D[b][head][q] = sum_c dO[b, q, head*hd + c] * O[b, q, head*hd + c]. Half a warp per
// (b, q, head) row: 16 lanes x 16-byte loads cover the 128 head columns; grid-stride.
__global__ void attn_bwd_dot_kernel(const uint16_t* __restrict__ dO, const uint16_t* __restrict__ O, float* __restrict__ D,
                                    int B, int s, int nh) {
    pdl_launch_dependents();
    pdl_wait();
    const long long rows = (long long)B * s * nh;
    const int sub = threadIdx.x & 15;
    for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4; w < rows;
         w += ((long long)gridDim.x * blockDim.x) >> 4) {
        const size_t off = (size_t)w * kHD + sub * 8;  // (b*s + q)*h + head*hd == w*hd
        const uint4 a = *reinterpret_cast<const uint4*>(dO + off);
        const uint4 o = *reinterpret_cast<const uint4*>(O + off);
        const uint32_t au[4] = {a.x, a.y, a.z, a.w}, ou[4] = {o.x, o.y, o.z, o.w};
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            t += bf16_bits_to_f32(au[k] & 0xffffu) * bf16_bits_to_f32(ou[k] & 0xffffu) +
                 bf16_bits_to_f32(au[k] >> 16) * bf16_bits_to_f32(ou[k] >> 16);
#pragma unroll
        for (int o2 = 8; o2 > 0; o2 >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o2);
        if (sub == 0) {
            const int head = (int)(w % nh);
            const long long bq = w / nh;  // b * s + q
            const long long bb = bq / s, q = bq % s;
            D[(bb * nh + head) * s + q] = t;
        }
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// Head view {hd, s, nh, B} of a [B][s][ld] bf16 buffer (ld = 3h for qkv, h for dO), box 64 x 128.
bool head_view(CUtensorMap* m, const uint16_t* base, int s, int nh, int B, long long ld, int box_rows = 128) {
    EncodeFn fn = encode();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)kHD, (cuuint64_t)s, (cuuint64_t)nh, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)ld * 2, (cuuint64_t)kHD * 2, (cuuint64_t)s * ld * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [B][nh][s][s] bf16 probabilities-shaped buffer (dS), box 64 keys x 32 query rows (store slabs).
bool probs_view(CUtensorMap* m, uint16_t* base, int s, int nh, int B) {
    EncodeFn fn = encode();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)s, (cuuint64_t)s, (cuuint64_t)nh, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)s * 2, (cuuint64_t)s * s * 2, (cuuint64_t)nh * s * s * 2};
    cuuint32_t box[4] = {64, 32, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Row-major [rows][cols] bf16 matrix, box 64 columns x 32 rows, SWIZZLE_128B (per-warp store slabs).
bool rows_view(CUtensorMap* m, uint16_t* base, long long cols, long long rows, int box_cols = 64,
               CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
    EncodeFn fn = encode();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, 32};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes, bool& done) {
    if (done) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done = true;
    return e;
}

}  // namespace

bool flash_supported(int hd, int s) { return hd == kHD && s % kT == 0 && s >= kT; }

cudaError_t attn_rowdot(const uint16_t* dO, const uint16_t* O, float* D, int B, int s, int nh, cudaStream_t st) {
    launch_ex(attn_bwd_dot_kernel, dim3(kNumSMs * 8), dim3(256), 0, st, 1, dO, O, D, B, s, nh);
    return launched(1);
}

cudaError_t flash_fwd(const uint16_t* qkv, uint16_t* O, float* lse2, int B, int s, int nh, int hd, float scale,
                      cudaStream_t st) {
    if (!flash_supported(hd, s)) return cudaErrorInvalidValue;
    const int h = nh * hd;
    CUtensorMap mq, mk, mv;  // K / V in 64-key boxes (64-key score tiles)
    if (!head_view(&mq, qkv, s, nh, B, 3ll * h) || !head_view(&mk, qkv + h, s, nh, B, 3ll * h, kKT) ||
        !head_view(&mv, qkv + 2 * h, s, nh, B, 3ll * h, kKT))
        return cudaErrorInvalidValue;
    FwdParams a;
    a.s = s;
    a.nh = nh;
    a.B = B;
    a.h = h;
    a.sl2 = scale * 1.4426950408889634f;
    a.O = O;
    a.lse2 = lse2;
    const int items = (s / kT) * nh * B;
    const int grid = items < 2 * kNumSMs ? items : 2 * kNumSMs;  // two CTAs per SM
    CUtensorMap mo;  // O [B*s][h], box 32 x 32, SWIZZLE_64B (the epilogue slabs)
    if (!rows_view(&mo, O, h, (long long)B * s, 32, CU_TENSOR_MAP_SWIZZLE_64B)) return cudaErrorInvalidValue;
    // Q | K, V rings | barriers (1 KB) | epilogue slabs (2 KB per softmax warp)
    const size_t smem = 1024 + (size_t)kTile + 4 * (size_t)kTileKV + 1024 + 4 * 2048;
    static bool cfg = false;
    cudaError_t e = set_smem(flash_fwd_k64_kernel, smem, cfg);
    if (e != cudaSuccess) return e;
    launch_ex(flash_fwd_k64_kernel, dim3(grid), dim3(192), smem, st, 1, mq, mk, mv, mo, a);
    return launched(1);
}

cudaError_t flash_bwd(const uint16_t* qkv, const uint16_t* O, const uint16_t* dO, const float* lse2, float* D,
                      uint16_t* dS, uint16_t* dqkv, int B, int s, int nh, int hd, float scale, cudaStream_t st) {
    if (!flash_supported(hd, s)) return cudaErrorInvalidValue;
    const int h = nh * hd;
    cudaError_t e = attn_rowdot(dO, O, D, B, s, nh, st);
    if (e != cudaSuccess) return e;
    CUtensorMap mq, mk, mv, mdo, mds;
    if (!head_view(&mq, qkv, s, nh, B, 3ll * h) || !head_view(&mk, qkv + h, s, nh, B, 3ll * h) ||
        !head_view(&mv, qkv + 2 * h, s, nh, B, 3ll * h) || !head_view(&mdo, dO, s, nh, B, h) ||
        !probs_view(&mds, dS, s, nh, B))
        return cudaErrorInvalidValue;
    BwdParams a;
    a.s = s;
    a.nh = nh;
    a.B = B;
    a.h = h;
    a.sl2 = scale * 1.4426950408889634f;
    a.scale = scale;
    a.lse2 = lse2;
    a.D = D;
    a.dS = dS;
    a.dqkv = dqkv;
    // transposed persistent kernel: dS^T [B][nh][key][query]
    // tiles | lse/D stages (2 KB) | barriers (<= 1 KB) | 8 dS^T slabs (32 KB): the 227 KB maximum
    const size_t smem = 6 * (size_t)kTile + 3072 + 8 * 4096;
    static bool cfg3 = false;
    e = set_smem(flash_bwd_t_kernel, smem, cfg3);
    if (e != cudaSuccess) return e;
    const int items = (s / kT) * nh * B;
    CUtensorMap mdqkv;  // [B*s][3h] bf16, box 64 columns x 32 rows (the dV / dK slabs)
    if (!rows_view(&mdqkv, dqkv, 3ll * h, (long long)B * s)) return cudaErrorInvalidValue;
    launch_ex(flash_bwd_t_kernel, dim3(items < kNumSMs ? items : kNumSMs), dim3(kThreads), smem, st, 1, mq, mk, mv, mdo, mds,
              mdqkv, a);
    return launched(1);
}

}  // namespace gpt
}  // namespace ah
