// bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Realises the dense contractions of OpKind::Forward / Backward / Recompute (reference
// cost model t_fp = (2*m_p*b*s + 4*b*s^2*h)/rate, proj/core/src/workload.cpp:63): the four
// linear layers of a GPT block (fwd, dgrad, wgrad) and the attention score / value products.
//
//   C[z](m, n) = epilogue( alpha * sum_k A[z](m, k) * B[z](n, k) )
//
// A and B are each K-major ([rows][K], K contiguous) or MN-major ([K][rows], rows
// contiguous) so fwd (TN), dgrad (TT) and wgrad (NN) run without transposes. z indexes a
// two-level batch (e.g. head x sequence) addressed through 4-D TMA tensor maps.
//
// Structure (persistent over output tiles, 384 threads = 12 warps; for BN = 256 two CTAs of a
// cluster pair form one 256 x 256 tile with tcgen05.mma.cta_group::2, M = 256):
//   warps 0-7   epilogue, two per TMEM lane quarter: tcgen05.ld 32x32b -> registers -> alpha /
//               beta*C / bias / GELU (+ pre-activation aux) / GELU' / residual -> bf16 packs
//               -> per-warp 32 x 32 smem slab -> TMA bulk tensor store (fp32 C: direct stores)
//   warp 8      TMA producer: 128 x 64 A tile + B tile (its half under cta_group::2) per
//               stage, SWIZZLE_128B, STAGES-deep smem ring guarded by full/empty mbarriers
//   warp 9      MMA issuer: one elected thread issues tcgen05.mma (K = 16) x4 per stage into
//               a TMEM accumulator; commits free the smem stage; a commit per tile hands the
//               accumulator to the epilogue
//   warp 10     TMEM allocator (2 x BN fp32 columns: double-buffered accumulator so the
//               epilogue of tile i overlaps the MMAs of tile i+1)
// The single-thread producer / MMA roles take the highest warp ids (the sub-partition arbiter
// issues highest-warp-id first). A poorly filled last wave is split in K halves across CTA
// pairs (stream-K), with fixed-order partial sums (deterministic).
// Causal modes skip work that a causal mask zeroes: whole tiles above the diagonal, or the
// K range of a tile (P·V, dS·K, dS^T·Q, P^T·dO).
#include <cuda.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <string>
#include <vector>

#include "common.cuh"
#include "gemm.h"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace ah {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;  // warps 0-7: epilogue (two per TMEM lane quarter)
// The single-thread producer / MMA roles take the highest warp ids (the sub-partition arbiter
// issues highest-warp-id first), so epilogue ALU work cannot starve an MMA or TMA issue slot.
constexpr int kWarpTMA = 8, kWarpMMA = 9, kWarpAlloc = 10;
// The smem-transposed (staged) epilogue is compiled but disabled: with 8 epilogue warps its
// staging slabs do not fit beside a 4-stage BN=256 ring. Direct row stores are used.
constexpr int kStagedSmem = 0;

struct Params {
    int M, N, K;
    int batch1, batch2;
    int tiles_m, tiles_n, num_tiles, k_blocks;
    int a_mn, b_mn;
    void* C;
    int c_f32;
    long long ldc, c_s1, c_s2;
    const void* bias;
    int bias_f32;
    const uint16_t* res;
    long long ld_res, res_s1, res_s2;
    uint16_t* aux;
    long long ld_aux, aux_s1, aux_s2;
    float alpha, beta;
    int epi;
    int causal;
    int vec_c, vec_aux;      // 4-element vector access legal (staged path)
    int vec16_c, vec16_aux;  // 16-byte rows (direct path)
    int staged;              // smem-transposed epilogue (fp32 outputs)
    int vec_bias, vec16_res;  // 16-byte vector loads legal for bias / residual
    int tma_c;                // bf16 C written by TMA bulk stores from smem slabs
    int fast;                 // tma_c, alpha 1, beta 0, N % BN == 0, 16-byte operand rows: lean epilogue
    int sk;                   // stream-K work split (CS == 1, non-causal)
    float* sk_ws;             // [grid][BM][BN] fp32 prefix partials
    unsigned* sk_flags;       // [grid] release flags (== sk_epoch when the partial is ready)
    unsigned sk_epoch;
};

// ---------------------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}
// Pipeline waits of the producer / MMA / epilogue roles with a suspend-time hint: a role that
// is ahead (the TMA producer, the epilogue during the main loop) is parked by the hardware
// instead of re-issuing the probe — every probe is an issued warp instruction and power.
__device__ __forceinline__ void mbar_wait_hint(uint32_t bar, uint32_t parity, uint32_t ns) {
    if (ns == 0) return mbar_wait(bar, parity);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"(parity), "r"(ns)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0,
                                            int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// 32 lanes x 32 consecutive fp32 columns: thread i of the warp gets row (lane_base + i).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// SWIZZLE_128B shared-memory matrix descriptor (sm_100 format, version 1).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;  // descriptor version (Blackwell)
    d |= 2ull << 61;  // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// v[base .. base+8) += 8 bf16 values packed in w (paired adds: two columns per FADD2)
__device__ __forceinline__ void add8(float (&v)[32], int base, uint4 w) {
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e)
        tc::f2unpack(tc::fadd2(tc::f2pack(v[base + 2 * e], v[base + 2 * e + 1]),
                               tc::f2pack(__uint_as_float(u[e] << 16), __uint_as_float(u[e] & 0xffff0000u))),
                     v[base + 2 * e], v[base + 2 * e + 1]);
}

__device__ __forceinline__ float gelu_grad(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float th = tanh_fast(k0 * (x + k1 * x * x * x));
    return 0.5f * (1.f + th) + 0.5f * x * (1.f - th * th) * k0 * (1.f + 3.f * k1 * x * x);
}

__device__ __forceinline__ float gelu_tanh(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    return 0.5f * x * (1.f + tanh_fast(k0 * (x + k1 * x * x * x)));
}

// The same two GELU functions on a pair of values with paired fp32 arithmetic (FFMA2 / FMUL2:
// the lean epilogue is issue-bound and its issue slots are shared with the MMA / TMA issuers).
__device__ __forceinline__ void gelu_tanh2(float& x0, float& x1) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const unsigned long long x = tc::f2pack(x0, x1);
    const unsigned long long x2 = tc::fmul2(x, x);
    const unsigned long long t = tc::ffma2(x2, tc::f2pack(k0 * k1, k0 * k1), tc::f2pack(k0, k0));  // k0 (1 + k1 x^2)
    float u0, u1;
    tc::f2unpack(tc::fmul2(x, t), u0, u1);
    const unsigned long long th = tc::f2pack(tanh_fast(u0), tanh_fast(u1));
    const unsigned long long hx = tc::fmul2(x, tc::f2pack(0.5f, 0.5f));
    tc::f2unpack(tc::ffma2(hx, th, hx), x0, x1);  // 0.5 x (1 + th)
}

// v0, v1 *= gelu'(x0), gelu'(x1)
__device__ __forceinline__ void mul_gelu_grad2(float& v0, float& v1, float x0, float x1) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const unsigned long long x = tc::f2pack(x0, x1);
    const unsigned long long x2 = tc::fmul2(x, x);
    const unsigned long long t = tc::ffma2(x2, tc::f2pack(k0 * k1, k0 * k1), tc::f2pack(k0, k0));
    float u0, u1;
    tc::f2unpack(tc::fmul2(x, t), u0, u1);
    const float t0 = tanh_fast(u0), t1 = tanh_fast(u1);
    const unsigned long long th = tc::f2pack(t0, t1);
    const unsigned long long a = tc::ffma2(th, tc::f2pack(0.5f, 0.5f), tc::f2pack(0.5f, 0.5f));     // 0.5 (1 + th)
    const unsigned long long s = tc::ffma2(tc::f2pack(-t0, -t1), th, tc::f2pack(1.f, 1.f));       // 1 - th^2
    const unsigned long long d = tc::ffma2(x2, tc::f2pack(3.f * k0 * k1, 3.f * k0 * k1), tc::f2pack(k0, k0));  // k0 (1 + 3 k1 x^2)
    const unsigned long long b = tc::fmul2(tc::fmul2(x, tc::f2pack(0.5f, 0.5f)), s);              // 0.5 x (1 - th^2)
    tc::f2unpack(tc::fmul2(tc::f2pack(v0, v1), tc::ffma2(b, d, a)), v0, v1);
}

struct Tile {
    int z1, z2, tm, tn, kb0, kb1;
    bool skip;
    int role;  // 0: whole tile, 1: stream-K prefix (partial -> workspace), 2: stream-K suffix (adds it)
};

__device__ __forceinline__ Tile decode_at(const Params& P, int z, int tm, int tn, int BN) {
    Tile T;
    T.tm = tm;
    T.tn = tn;
    T.z1 = z % P.batch1;
    T.z2 = z / P.batch1;
    T.kb0 = 0;
    T.kb1 = P.k_blocks;
    T.skip = false;
    const int m0 = T.tm * BM;
    if (P.causal == kCausalSkipUpper) {
        T.skip = T.tn * BN > m0 + BM - 1;
    } else if (P.causal == kCausalKUptoM) {
        const int lim = (m0 + BM + BK - 1) / BK;
        T.kb1 = lim < T.kb1 ? lim : T.kb1;
    } else if (P.causal == kCausalKFromM) {
        T.kb0 = m0 / BK;
    }
    if (T.kb0 >= T.kb1) T.skip = true;
    return T;
}

// Cluster tile ct -> this CTA's tile. A cluster of CS CTAs shares one B tile (same tn, z) and
// takes CS consecutive M tiles; a rank past the last M tile computes an all-zero phantom tile
// (TMA zero-fills, the epilogue masks rows >= M) so every CTA of a cluster runs the same
// pipeline.
// Causal K-range modes: tile cost grows (KUptoM) or shrinks (KFromM) with the M tile, so tiles
// are enumerated heaviest M row first and dealt to CTAs in snake order (longest-processing-time
// first); z / N vary fastest inside an M row.
__device__ __forceinline__ bool causal_lpt(const Params& P) {
    return P.causal == kCausalKUptoM || P.causal == kCausalKFromM;
}

template <int CS>
__device__ __forceinline__ Tile decode(const Params& P, int ct, int BN, int crank) {
    if (CS == 1 && causal_lpt(P)) {
        const int per_m = P.tiles_n * P.batch1 * P.batch2;
        const int r = ct / per_m, rest = ct - r * per_m;
        const int tm = P.causal == kCausalKUptoM ? P.tiles_m - 1 - r : r;
        const int z = rest / P.tiles_n;
        return decode_at(P, z, tm, rest - z * P.tiles_n, BN);
    }
    // Grouped raster: bands of kBand cluster-tile rows, each band walked N column by N column
    // (rows fastest), so the ~74 tiles in flight cover kBand M rows x ~9 N columns: the A band
    // (kBand x 256 rows) stays in L2 while B streams once per band. Row-major order (N fastest)
    // put a whole M row in flight and re-read B from DRAM once per M row when B > L2 (the
    // 10B / 20B qkv, fc, fc2 and LM-head shapes: 226 MB of B x 32 M rows for qkv at h = 6144).
    constexpr int kBand = 16;
    const int tmg = (P.tiles_m + CS - 1) / CS;
    const int per_z = tmg * P.tiles_n;
    const int z = ct / per_z;
    const int rem = ct - z * per_z;
    const int band = rem / (kBand * P.tiles_n);
    const int rows = tmg - band * kBand < kBand ? tmg - band * kBand : kBand;
    const int r2 = rem - band * kBand * P.tiles_n;
    const int tn = r2 / rows;
    const int g = band * kBand + (r2 - tn * rows);
    return decode_at(P, z, g * CS + crank, tn, BN);
}

// ---- work assignment -------------------------------------------------------------------
// Data-parallel: cluster tiles strided over the grid (L2-friendly: concurrently running CTAs
// share A panels). Tail split (P.sk): the W full waves stay data-parallel and each of the
// remaining `tail` cluster tiles (2 * tail <= clusters) is split in two K halves on clusters
// 2u (prefix, processed FIRST, partial -> workspace slot + release flag per CTA) and 2u + 1
// (suffix, processed LAST, adds the partial before its epilogue), so the last wave costs half a
// tile instead of a whole one (512 tiles on 148 SMs: 3.5 instead of 4 tile times).
template <int CS>
__device__ __forceinline__ int num_segments(const Params& P) {
    const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;
    if (CS == 1 && causal_lpt(P)) {  // snake: round k takes k*ncl + (k even ? cid : ncl-1-cid)
        const int full = P.num_tiles / ncl, rem = P.num_tiles - full * ncl;
        return full + ((rem && ((full & 1) == 0 ? cid < rem : (ncl - 1 - cid) < rem)) ? 1 : 0);
    }
    if (!P.sk) return cid < P.num_tiles ? (P.num_tiles - 1 - cid) / ncl + 1 : 0;
    const int waves = P.num_tiles / ncl, tail = P.num_tiles - waves * ncl;
    return waves + (cid < 2 * tail ? 1 : 0);
}

template <int CS>
__device__ __forceinline__ Tile segment(const Params& P, int i, int BN, int crank) {
    if (CS == 1 && causal_lpt(P)) {
        const int ncl = gridDim.x, cid = blockIdx.x;
        Tile T = decode<CS>(P, i * ncl + ((i & 1) == 0 ? cid : ncl - 1 - cid), BN, crank);
        T.role = 0;
        return T;
    }
    if (!P.sk) {
        Tile T = decode<CS>(P, blockIdx.x / CS + i * (gridDim.x / CS), BN, crank);
        T.role = 0;
        return T;
    }
    const int G = gridDim.x / CS, c = blockIdx.x / CS, waves = P.num_tiles / G, tail = P.num_tiles - waves * G;
    const bool unit = c < 2 * tail;
    const bool prefix = unit && (c & 1) == 0;
    int t, k0 = 0, k1 = P.k_blocks, role = 0;
    if (prefix && i == 0) {
        t = waves * G + c / 2, k1 = P.k_blocks / 2, role = 1;
    } else if (unit && !prefix && i == waves) {
        t = waves * G + c / 2, k0 = P.k_blocks / 2, role = 2;
    } else {
        t = c + (i - (prefix ? 1 : 0)) * G;
    }
    Tile T = decode<CS>(P, t, BN, crank);
    T.kb0 = k0;
    T.kb1 = k1;
    T.role = role;
    return T;
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// ---- CTA pair (cta_group::2): one M=256 MMA over the two CTAs' smem, issued by rank 0 ----
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// TMA into this CTA's smem, completing bytes on the (possibly peer) barrier `bar` (cluster address)
__device__ __forceinline__ void tma_load_4d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                 int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// arrive on the barrier at the same smem offset in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
                 "h"((uint16_t)3)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// CS == 2: CTA pair. Each CTA stages its own 128 A rows and half (BN/2 rows) of the B tile;
// rank 0 issues tcgen05.mma.cta_group::2 with M = 256, which reads both CTAs' smem and writes
// each CTA's 128 accumulator rows into its own TMEM. Rank 0's full barrier collects both CTAs'
// TMA bytes; its commits arrive on both CTAs' empty / tmem-full barriers (multicast); both
// CTAs' epilogues release the accumulator on rank 0's tmem-empty barrier. Per SM, the MMA
// reads 32 KB of smem per k-block instead of 48 KB.
template <int BN, int STAGES, int CS>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const __grid_constant__ CUtensorMap tmC, const Params P) {
    static_assert(CS == 1 || (CS == 2 && BN == 256), "CTA pair: BN = 256");
    constexpr bool kPair = CS == 2;
    constexpr uint32_t A_BYTES = BM * BK * 2;
    constexpr uint32_t B_BYTES = (BN / CS) * BK * 2;  // this CTA's part of the B tile
    constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for SWIZZLE_128B atoms
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* tfull = bars + 2 * STAGES;
    uint64_t* tempty = bars + 2 * STAGES + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
    // TMA-store staging: per epilogue warp two 32x32 bf16 slabs (SWIZZLE_64B), 1 KB past the barriers
    uint8_t* cstage = reinterpret_cast<uint8_t*>(bars) + 1024;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int crank = CS > 1 ? (int)cluster_rank() : 0;

    if (warp == kWarpTMA && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(smem_u32(&tfull[a]), 1);
            mbar_init(smem_u32(&tempty[a]), kEpiWarps * CS);  // pair: both CTAs' epilogues (rank 0's)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == kWarpAlloc) {
        if (kPair) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                         "r"(2 * BN));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                         "r"(2 * BN));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    if (CS > 1)
        cluster_sync_all();  // peers' barriers initialised before any multicast lands
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    // setup above overlapped the previous kernel's tail (PDL); operands / outputs only from here
    pdl_launch_dependents();
    pdl_wait();

    if (warp == kWarpTMA) {
        if (lane == 0) {
            // ===== TMA producer =====
            int stage = 0;
            uint32_t phase = 0;
            const int nseg = num_segments<CS>(P);
            for (int si = 0; si < nseg; ++si) {
                const Tile T = segment<CS>(P, si, BN, crank);
                if (T.skip) continue;
                for (int kb = T.kb0; kb < T.kb1; ++kb) {
                    mbar_wait_hint(smem_u32(&empty[stage]), phase ^ 1, 0u);
                    const uint32_t a_dst = smem_u32(sA + stage * A_BYTES);
                    const uint32_t b_dst = smem_u32(sB + stage * B_BYTES);
                    const int k0 = kb * BK;
                    if (kPair) {  // both CTAs' bytes complete on rank 0's full barrier
                        const uint32_t fb = mapa_rank(smem_u32(&full[stage]), 0);
                        if (crank == 0) mbar_expect_tx(smem_u32(&full[stage]), 2 * STAGE_BYTES);
                        if (!P.a_mn) {
                            tma_load_4d_pair(a_dst, &tmA, fb, k0, T.tm * BM, T.z1, T.z2);
                        } else {
#pragma unroll
                            for (int j = 0; j < BM / 64; ++j)
                                tma_load_4d_pair(a_dst + j * (64 * BK * 2), &tmA, fb, T.tm * BM + j * 64, k0, T.z1, T.z2);
                        }
                        if (!P.b_mn) {
                            tma_load_4d_pair(b_dst, &tmB, fb, k0, T.tn * BN + crank * (BN / 2), T.z1, T.z2);
                        } else {
#pragma unroll
                            for (int jj = 0; jj < BN / 128; ++jj)
                                tma_load_4d_pair(b_dst + jj * (64 * BK * 2), &tmB, fb, T.tn * BN + crank * (BN / 2) + jj * 64,
                                                 k0, T.z1, T.z2);
                        }
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
                    const uint32_t fb = smem_u32(&full[stage]);
                    mbar_expect_tx(fb, STAGE_BYTES);
                    if (!P.a_mn) {
                        tma_load_4d(a_dst, &tmA, fb, k0, T.tm * BM, T.z1, T.z2);
                    } else {
#pragma unroll
                        for (int j = 0; j < BM / 64; ++j)
                            tma_load_4d(a_dst + j * (64 * BK * 2), &tmA, fb, T.tm * BM + j * 64, k0, T.z1, T.z2);
                    }
                    if (!P.b_mn) {
                        tma_load_4d(b_dst, &tmB, fb, k0, T.tn * BN, T.z1, T.z2);
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j)
                            tma_load_4d(b_dst + j * (64 * BK * 2), &tmB, fb, T.tn * BN + j * 64, k0, T.z1, T.z2);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == kWarpMMA) {
        if (lane == 0 && crank == 0) {
            // ===== MMA issuer (pair: rank 0 only) =====
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(P.a_mn) << 15) |
                                   (uint32_t(P.b_mn) << 16) | (uint32_t(BN >> 3) << 17) | (uint32_t((BM * CS) >> 4) << 24);
            // K-major: rows of 128 B, 8-row atoms 1024 B apart; K step of 16 = +32 B.
            // MN-major: 64-element (128 B) chunks BK rows deep (LBO = 64*BK*2 B apart), 8-row
            // K groups 1024 B apart; K step of 16 = +2048 B.
            const uint32_t a_lbo = P.a_mn ? 64 * BK * 2 : 16, a_sbo = 1024, a_kstep = P.a_mn ? 2048 : 32;
            const uint32_t b_lbo = P.b_mn ? 64 * BK * 2 : 16, b_sbo = 1024, b_kstep = P.b_mn ? 2048 : 32;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            const int nseg = num_segments<CS>(P);
            for (int si = 0; si < nseg; ++si) {
                const Tile T = segment<CS>(P, si, BN, crank);
                if (T.skip) continue;
                mbar_wait_hint(smem_u32(&tempty[acc]), acc_phase ^ 1, 0u);  // latency-critical
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = T.kb0; kb < T.kb1; ++kb) {
                    mbar_wait_hint(smem_u32(&full[stage]), phase, 0u);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(sA + stage * A_BYTES);
                    const uint32_t b_addr = smem_u32(sB + stage * B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t ad = smem_desc(a_addr + k * a_kstep, a_lbo, a_sbo);
                        const uint64_t bd = smem_desc(b_addr + k * b_kstep, b_lbo, b_sbo);
                        if (kPair)
                            tc_mma_pair(d_tmem, ad, bd, idesc, (kb > T.kb0 || k > 0) ? 1u : 0u);
                        else
                            tc_mma(d_tmem, ad, bd, idesc, (kb > T.kb0 || k > 0) ? 1u : 0u);
                    }
                    if (kPair)
                        tc_commit_pair(smem_u32(&empty[stage]));
                    else
                        tc_commit(smem_u32(&empty[stage]));
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (kPair)
                    tc_commit_pair(smem_u32(&tfull[acc]));
                else
                    tc_commit(smem_u32(&tfull[acc]));
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp < kEpiWarps) {
        // ===== epilogue =====
        // TMEM -> registers (thread = row, 32 columns) -> per-warp smem slab -> each lane
        // re-reads 4 consecutive columns of a row, so a warp instruction covers 4 rows x 32
        // columns (128 B fp32 / 64 B bf16 per row). The element-wise epilogue runs in this
        // phase: bias / residual / aux / C accesses are row-contiguous too.
        // two warps per TMEM lane quarter (one per half of the tile's 32-column chunks): two
        // epilogue warps per SM sub-partition, so the per-element work has the ILP to hide
        // under the next tile's MMAs
        const int q = warp & 3;  // TMEM lane quarter = 32-row slab of the tile
        const int half = warp >> 2;
        float* stage = reinterpret_cast<float*>(tmem_holder + 4) + warp * 32 * 36;
        const int sub = lane & 7, rsub = lane >> 3;
        int epi_chunk = 0;  // TMA-store slabs used by this warp (double-buffered)
        int acc = 0;
        uint32_t acc_phase = 0;
        const int nseg = num_segments<CS>(P);
        for (int si = 0; si < nseg; ++si) {
            const Tile T = segment<CS>(P, si, BN, crank);
            if (T.skip) continue;
            mbar_wait_hint(smem_u32(&tfull[acc]), acc_phase, 0u);
            tc_fence_after();
            if (T.role == 2) {  // stream-K suffix: wait for the previous CTA's partial of this tile
                if (warp == 0 && lane == 0) {
                    unsigned f = 0;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(P.sk_flags + blockIdx.x - CS) : "memory");
                        if (f != P.sk_epoch) __nanosleep(64);
                    } while (f != P.sk_epoch);
                }
                asm volatile("bar.sync 1, %0;" ::"r"(kEpiWarps * 32) : "memory");
            }
            const int m_base = T.tm * BM + q * 32;
            const long long zc = (long long)T.z1 * P.c_s1 + (long long)T.z2 * P.c_s2;
            const long long zr = (long long)T.z1 * P.res_s1 + (long long)T.z2 * P.res_s2;
            const long long za = (long long)T.z1 * P.aux_s1 + (long long)T.z2 * P.aux_s2;
            const int rows = min(32, P.M - m_base);
#pragma unroll 1
            for (int c = half; c < BN / 32; c += 2) {
                float v[32];
                tmem_ld32(tmem_base + (uint32_t(q * 32) << 16) + acc * BN + c * 32, v);
                const int n0 = T.tn * BN + c * 32;
                if (rows <= 0 || n0 >= P.N) continue;  // warp-uniform
                if (T.role != 0) {  // stream-K: raw fp32 accumulator row chunk <-> workspace slot
                    const unsigned slot_cta = T.role == 1 ? blockIdx.x : blockIdx.x - CS;  // same rank, previous cluster
                    float4* s4 = reinterpret_cast<float4*>(P.sk_ws + ((size_t)slot_cta * BM + q * 32 + lane) * BN + c * 32);
                    if (T.role == 1) {
#pragma unroll
                        for (int w = 0; w < 8; ++w) s4[w] = make_float4(v[4 * w], v[4 * w + 1], v[4 * w + 2], v[4 * w + 3]);
                        continue;
                    }
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        const float4 x = s4[w];
                        v[4 * w] += x.x;
                        v[4 * w + 1] += x.y;
                        v[4 * w + 2] += x.z;
                        v[4 * w + 3] += x.w;
                    }
                }
                if (P.fast && rows == 32) {
                    // Lean path for whole 32 x 32 chunks: vector operand loads, hardware bf16
                    // packs, one TMA store. (Its instruction count paces the MMAs: every issue
                    // slot spent here is shared with the single-thread MMA issuer.)
                    const int m = m_base + lane;
                    if (P.epi & kEpiBias) {
                        const uint4* b4 = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(P.bias) + n0);
#pragma unroll
                        for (int w = 0; w < 4; ++w) add8(v, 8 * w, b4[w]);
                    }
                    if (P.epi & (kEpiAux | kEpiGeluBwd)) {
                        uint4* a4 = reinterpret_cast<uint4*>(P.aux + za + (long long)m * P.ld_aux + n0);
                        if (P.epi & kEpiGeluBwd) {
#pragma unroll
                            for (int w = 0; w < 4; ++w) {
                                const uint4 q4 = a4[w];
                                const uint32_t u[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e)
                                    mul_gelu_grad2(v[8 * w + 2 * e], v[8 * w + 2 * e + 1], __uint_as_float(u[e] << 16),
                                                   __uint_as_float(u[e] & 0xffff0000u));
                            }
                        } else {
#pragma unroll
                            for (int w = 0; w < 4; ++w)
                                a4[w] = make_uint4(pack_bf16x2_rn(v[8 * w], v[8 * w + 1]), pack_bf16x2_rn(v[8 * w + 2], v[8 * w + 3]),
                                                   pack_bf16x2_rn(v[8 * w + 4], v[8 * w + 5]), pack_bf16x2_rn(v[8 * w + 6], v[8 * w + 7]));
                        }
                    }
                    if ((P.epi & kEpiGelu) && !(P.epi & kEpiGeluBwd)) {
#pragma unroll
                        for (int j = 0; j < 32; j += 2) gelu_tanh2(v[j], v[j + 1]);
                    }
                    if (P.epi & kEpiResidual) {
                        const uint4* r4 = reinterpret_cast<const uint4*>(P.res + zr + (long long)m * P.ld_res + n0);
#pragma unroll
                        for (int w = 0; w < 4; ++w) add8(v, 8 * w, r4[w]);
                    }
                    uint8_t* slab = cstage + (warp * 2 + (epi_chunk & 1)) * 2048;
                    if (epi_chunk >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    __syncwarp();
#pragma unroll
                    for (int w = 0; w < 4; ++w)
                        *reinterpret_cast<uint4*>(slab + lane * 64 + ((w ^ ((lane >> 1) & 3)) << 4)) =
                            make_uint4(pack_bf16x2_rn(v[8 * w], v[8 * w + 1]), pack_bf16x2_rn(v[8 * w + 2], v[8 * w + 3]),
                                       pack_bf16x2_rn(v[8 * w + 4], v[8 * w + 5]), pack_bf16x2_rn(v[8 * w + 6], v[8 * w + 7]));
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile(
                            "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                                reinterpret_cast<uint64_t>(&tmC)),
                            "r"(smem_u32(slab)), "r"(n0), "r"(m_base), "r"(T.z1), "r"(T.z2)
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    ++epi_chunk;
                    continue;
                }
                if (!P.staged) {  // bf16 output: each thread owns its row's 32 columns
                    const int m = m_base + lane;
                    const bool row_live = m < P.M;
                    if (!row_live && !P.tma_c) continue;
                    const long long c_off = zc + (long long)m * P.ldc;
                const bool full_chunk = n0 + 32 <= P.N;
                if (!row_live) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = 0.f;
                } else {
                if (P.alpha != 1.f) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] *= P.alpha;
                }
                if (P.beta != 0.f) {
                    if (P.c_f32) {
                        const float* cp = static_cast<const float*>(P.C) + c_off + n0;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (full_chunk || n0 + j < P.N) v[j] += P.beta * cp[j];
                    } else {
                        const uint16_t* cp = static_cast<const uint16_t*>(P.C) + c_off + n0;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (full_chunk || n0 + j < P.N) v[j] += P.beta * bf16_bits_to_f32(cp[j]);
                    }
                }
                if (P.epi & kEpiBias) {
                    if (full_chunk && P.vec_bias) {  // same 64 B for every row: 4 x 16 B broadcast loads
                        const uint4* b4 = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(P.bias) + n0);
#pragma unroll
                        for (int w = 0; w < 4; ++w) add8(v, 8 * w, b4[w]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            if (!full_chunk && n0 + j >= P.N) continue;
                            v[j] += P.bias_f32 ? static_cast<const float*>(P.bias)[n0 + j]
                                               : bf16_bits_to_f32(static_cast<const uint16_t*>(P.bias)[n0 + j]);
                        }
                    }
                }
                if (P.epi & kEpiGeluBwd) {
                    const uint16_t* ap = P.aux + (long long)T.z1 * P.aux_s1 + (long long)T.z2 * P.aux_s2 +
                                         (long long)m * P.ld_aux + n0;
                    if (full_chunk && P.vec16_aux) {
                        const uint4* a4 = reinterpret_cast<const uint4*>(ap);
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            const uint4 q4 = a4[w];
                            const uint32_t u[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                            for (int e = 0; e < 8; ++e)
                                v[8 * w + e] *= gelu_grad(bf16_bits_to_f32((e & 1) ? (u[e >> 1] >> 16) : (u[e >> 1] & 0xffffu)));
                        }
                    } else {
                        for (int j = 0; j < 32; ++j)
                            if (full_chunk || n0 + j < P.N) v[j] *= gelu_grad(bf16_bits_to_f32(ap[j]));
                    }
                }
                if ((P.epi & kEpiAux) && !(P.epi & kEpiGeluBwd)) {
                    uint16_t* ap = P.aux + (long long)T.z1 * P.aux_s1 + (long long)T.z2 * P.aux_s2 +
                                   (long long)m * P.ld_aux + n0;
                    if (full_chunk && P.vec16_aux) {
                        uint4* a4 = reinterpret_cast<uint4*>(ap);
#pragma unroll
                        for (int w = 0; w < 4; ++w)
                            a4[w] = make_uint4(pack_bf16x2_rn(v[8 * w], v[8 * w + 1]), pack_bf16x2_rn(v[8 * w + 2], v[8 * w + 3]),
                                               pack_bf16x2_rn(v[8 * w + 4], v[8 * w + 5]), pack_bf16x2_rn(v[8 * w + 6], v[8 * w + 7]));
                    } else {
                        #pragma unroll
                        for (int j = 0; j < 32; ++j) if (n0 + j < P.N) ap[j] = (uint16_t)f32_to_bf16_bits(v[j]);
                    }
                }
                if ((P.epi & kEpiGelu) && !(P.epi & kEpiGeluBwd)) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = gelu_tanh(v[j]);
                }
                if (P.epi & kEpiResidual) {
                    const uint16_t* rp = P.res + (long long)T.z1 * P.res_s1 + (long long)T.z2 * P.res_s2 +
                                         (long long)m * P.ld_res + n0;
                    if (full_chunk && P.vec16_res) {
                        const uint4* r4 = reinterpret_cast<const uint4*>(rp);
#pragma unroll
                        for (int w = 0; w < 4; ++w) add8(v, 8 * w, r4[w]);
                    } else {
                        for (int j = 0; j < 32; ++j)
                            if (full_chunk || n0 + j < P.N) v[j] += bf16_bits_to_f32(rp[j]);
                    }
                }
                }  // row_live
                if (P.tma_c) {  // registers -> swizzled smem slab -> one TMA bulk store per chunk
                    uint8_t* slab = cstage + (warp * 2 + (epi_chunk & 1)) * 2048;
                    if (epi_chunk >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    __syncwarp();
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const int chunk = w ^ ((lane >> 1) & 3);
                        *reinterpret_cast<uint4*>(slab + lane * 64 + chunk * 16) =
                            make_uint4(pack_bf16x2_rn(v[8 * w], v[8 * w + 1]), pack_bf16x2_rn(v[8 * w + 2], v[8 * w + 3]),
                                       pack_bf16x2_rn(v[8 * w + 4], v[8 * w + 5]), pack_bf16x2_rn(v[8 * w + 6], v[8 * w + 7]));
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile(
                            "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                                reinterpret_cast<uint64_t>(&tmC)),
                            "r"(smem_u32(slab)), "r"(n0), "r"(m_base), "r"(T.z1), "r"(T.z2)
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    ++epi_chunk;
                    continue;
                }
                if (P.c_f32) {
                    float* cp = static_cast<float*>(P.C) + c_off + n0;
                    if (full_chunk && P.vec16_c) {
                        float4* c4 = reinterpret_cast<float4*>(cp);
#pragma unroll
                        for (int w = 0; w < 8; ++w) c4[w] = make_float4(v[4 * w], v[4 * w + 1], v[4 * w + 2], v[4 * w + 3]);
                    } else {
                        #pragma unroll
                        for (int j = 0; j < 32; ++j) if (n0 + j < P.N) cp[j] = v[j];
                    }
                } else {
                    uint16_t* cp = static_cast<uint16_t*>(P.C) + c_off + n0;
                    if (full_chunk && P.vec16_c) {
                        uint4* c4 = reinterpret_cast<uint4*>(cp);
#pragma unroll
                        for (int w = 0; w < 4; ++w)
                            c4[w] = make_uint4(pack_bf16x2_rn(v[8 * w], v[8 * w + 1]), pack_bf16x2_rn(v[8 * w + 2], v[8 * w + 3]),
                                               pack_bf16x2_rn(v[8 * w + 4], v[8 * w + 5]), pack_bf16x2_rn(v[8 * w + 6], v[8 * w + 7]));
                    } else {
                        #pragma unroll
                        for (int j = 0; j < 32; ++j) if (n0 + j < P.N) cp[j] = (uint16_t)f32_to_bf16_bits(v[j]);
                    }
                }
                    continue;
                }
                float4* srow = reinterpret_cast<float4*>(stage + lane * 36);
#pragma unroll
                for (int j = 0; j < 8; ++j) srow[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                __syncwarp();
                const int n = n0 + sub * 4;
                const int ncols = min(4, P.N - n);  // <= 0: lane idle
                float bias[4] = {0.f, 0.f, 0.f, 0.f};
                if ((P.epi & kEpiBias) && ncols > 0) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (k < ncols)
                            bias[k] = P.bias_f32 ? static_cast<const float*>(P.bias)[n + k]
                                                 : bf16_bits_to_f32(static_cast<const uint16_t*>(P.bias)[n + k]);
                }
                const bool vec = ncols == 4 && P.vec_c;
#pragma unroll 2
                for (int pass = 0; pass < 8; ++pass) {
                    const int rr = pass * 4 + rsub;
                    if (rr >= rows || ncols <= 0) continue;
                    const long long m = m_base + rr;
                    const float4 s4 = *reinterpret_cast<const float4*>(stage + rr * 36 + sub * 4);
                    float x[4] = {s4.x * P.alpha, s4.y * P.alpha, s4.z * P.alpha, s4.w * P.alpha};
                    const long long ci = zc + m * P.ldc + n;
                    if (P.beta != 0.f) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (k < ncols)
                                x[k] += P.beta * (P.c_f32 ? static_cast<const float*>(P.C)[ci + k]
                                                          : bf16_bits_to_f32(static_cast<const uint16_t*>(P.C)[ci + k]));
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) x[k] += bias[k];
                    if (P.epi & (kEpiGeluBwd | kEpiAux)) {
                        uint16_t* ap = P.aux + za + m * P.ld_aux + n;
                        if (P.epi & kEpiGeluBwd) {
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                if (k < ncols) x[k] *= gelu_grad(bf16_bits_to_f32(ap[k]));
                        } else if (vec && P.vec_aux) {
                            *reinterpret_cast<uint2*>(ap) = make_uint2(pack_bf16x2_rn(x[0], x[1]), pack_bf16x2_rn(x[2], x[3]));
                        } else {
                            for (int k = 0; k < ncols; ++k) ap[k] = (uint16_t)f32_to_bf16_bits(x[k]);
                        }
                    }
                    if ((P.epi & kEpiGelu) && !(P.epi & kEpiGeluBwd)) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) x[k] = gelu_tanh(x[k]);
                    }
                    if (P.epi & kEpiResidual) {
                        const uint16_t* rp = P.res + zr + m * P.ld_res + n;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (k < ncols) x[k] += bf16_bits_to_f32(rp[k]);
                    }
                    if (P.c_f32) {
                        float* cp = static_cast<float*>(P.C) + ci;
                        if (vec)
                            *reinterpret_cast<float4*>(cp) = make_float4(x[0], x[1], x[2], x[3]);
                        else
                            for (int k = 0; k < ncols; ++k) cp[k] = x[k];
                    } else {
                        uint16_t* cp = static_cast<uint16_t*>(P.C) + ci;
                        if (vec)
                            *reinterpret_cast<uint2*>(cp) = make_uint2(pack_bf16x2_rn(x[0], x[1]), pack_bf16x2_rn(x[2], x[3]));
                        else
                            for (int k = 0; k < ncols; ++k) cp[k] = (uint16_t)f32_to_bf16_bits(x[k]);
                    }
                }
                __syncwarp();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (kPair)
                    mbar_arrive_cluster(mapa_rank(smem_u32(&tempty[acc]), 0));
                else
                    mbar_arrive(smem_u32(&tempty[acc]));
            }
            if (T.role == 1) {  // publish the prefix partial for the next CTA
                asm volatile("bar.sync 1, %0;" ::"r"(kEpiWarps * 32) : "memory");
                if (warp == 0 && lane == 0) {
                    __threadfence();
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.sk_flags + blockIdx.x), "r"(P.sk_epoch) : "memory");
                }
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (P.tma_c && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // slabs stay live until read
    }
    if (CS > 1)
        cluster_sync_all();  // no peer may still multicast into / arrive on this CTA
    else
        __syncthreads();
    if (warp == kWarpAlloc) {
        tc_fence_after();
        if (kPair)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * BN));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * BN));
    }
}

// ---------------------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
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

// 4-D map over a bf16 operand: dims {inner, outer, b1, b2} with element strides.
static bool make_map(CUtensorMap* map, const void* base, long long inner, long long outer, long long ld,
                     int b1, long long s1, int b2, long long s2, int box_inner, int box_outer) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    const long long plane = ld * outer;
    if (b1 <= 1 || s1 == 0) s1 = plane;
    if (b2 <= 1 || s2 == 0) s2 = s1 * (b1 > 0 ? b1 : 1);
    cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)(b1 > 0 ? b1 : 1), (cuuint64_t)(b2 > 0 ? b2 : 1)};
    cuuint64_t strides[3] = {(cuuint64_t)(ld * 2), (cuuint64_t)(s1 * 2), (cuuint64_t)(s2 * 2)};
    cuuint32_t box[4] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static bool make_map_sw(CUtensorMap* map, const void* base, long long inner, long long outer, long long ld, int b1,
                        long long s1, int b2, long long s2, int box_inner, int box_outer, CUtensorMapSwizzle sw) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    const long long plane = ld * outer;
    if (b1 <= 1 || s1 == 0) s1 = plane;
    if (b2 <= 1 || s2 == 0) s2 = s1 * (b1 > 0 ? b1 : 1);
    cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)(b1 > 0 ? b1 : 1), (cuuint64_t)(b2 > 0 ? b2 : 1)};
    cuuint64_t strides[3] = {(cuuint64_t)(ld * 2), (cuuint64_t)(s1 * 2), (cuuint64_t)(s2 * 2)};
    cuuint32_t box[4] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

template <int BN, int STAGES, int CS>
static size_t smem_bytes() {
    return 1024 + STAGES * (size_t)(BM * BK * 2 + (BN / CS) * BK * 2) + (2 * STAGES + 4) * 8 + 16 + kStagedSmem + 1024 + kEpiWarps * 2 * 2048;
}

template <int BN, int STAGES, int CS>
static cudaError_t launch_cfg(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const Params& P, int grid,
                              cudaStream_t stream) {
    const size_t sm = smem_bytes<BN, STAGES, CS>();
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN, STAGES, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const cudaError_t e = launch_ex(gemm_kernel<BN, STAGES, CS>, dim3(grid), dim3(kThreads), sm, stream, CS, a, b, c, P);
    launched(1);
    return e != cudaSuccess ? e : cudaGetLastError();
}

struct TimingState {
    std::mutex mu;
    bool on = false;
    struct Rec {
        cudaEvent_t a, b;
        double flops;
        std::string shape;  // for the per-shape dump (AH_GEMM_TIMING_DUMP)
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;  // pre-created timing events: no cudaEventCreate on the launch path
    cudaEvent_t take() {
        if (pool.empty()) {
            cudaEvent_t e = nullptr;
            cudaEventCreate(&e);
            return e;
        }
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
};
static TimingState& timing() {
    static TimingState t;
    return t;
}

void timing_enable(bool on) {
    std::lock_guard<std::mutex> lk(timing().mu);
    timing().on = on;
    while (on && timing().pool.size() < 16384) {  // enough for a timed bench region
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) break;
        timing().pool.push_back(e);
    }
}

void timing_collect(double* total_ms, double* total_flops, long long* launches) {
    std::lock_guard<std::mutex> lk(timing().mu);
    double ms = 0.0, fl = 0.0;
    long long n = 0;
    std::map<std::string, std::tuple<long long, double, double>> by_shape;
    for (auto& r : timing().recs) {
        float t = 0.f;
        cudaEventSynchronize(r.b);
        if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) {
            ms += t;
            fl += r.flops;
            ++n;
            auto& a = by_shape[r.shape];
            std::get<0>(a) += 1;
            std::get<1>(a) += t;
            std::get<2>(a) += r.flops;
        }
        timing().pool.push_back(r.a);
        timing().pool.push_back(r.b);
    }
    timing().recs.clear();
    if (const char* path = std::getenv("AH_GEMM_TIMING_DUMP"); path && n > 0) {
        if (FILE* f = std::fopen(path, "a")) {  // one line per shape: launches, ms, TFLOP/s
            for (auto& [k, a] : by_shape)
                std::fprintf(f, "%s n=%lld ms=%.3f tflops=%.1f\n", k.c_str(), std::get<0>(a), std::get<1>(a),
                             std::get<2>(a) / (std::get<1>(a) * 1e-3) / 1e12);
            std::fclose(f);
        }
    }
    if (total_ms) *total_ms = ms;
    if (total_flops) *total_flops = fl;
    if (launches) *launches = n;
}

double executed_flops(const GemmArgs& g) {
    int BN = g.block_n;
    if (BN == 0) BN = g.N >= 256 ? 256 : (g.N > 64 ? 128 : 64);
    const long long tiles_m = (g.M + BM - 1) / BM, tiles_n = (g.N + BN - 1) / BN, kb = (g.K + BK - 1) / BK;
    double f = 0.0;
    for (long long tm = 0; tm < tiles_m; ++tm) {
        const long long m0 = tm * BM, mrows = std::min<long long>(BM, g.M - m0);
        long long k0 = 0, k1 = kb;
        if (g.causal == kCausalKUptoM) k1 = std::min<long long>(kb, (m0 + BM + BK - 1) / BK);
        if (g.causal == kCausalKFromM) k0 = m0 / BK;
        if (k0 >= k1) continue;
        const long long kl = std::min<long long>(g.K, k1 * BK) - k0 * BK;
        for (long long tn = 0; tn < tiles_n; ++tn) {
            if (g.causal == kCausalSkipUpper && tn * BN > m0 + BM - 1) continue;
            f += 2.0 * mrows * std::min<long long>(BN, g.N - tn * BN) * kl;
        }
    }
    return f * std::max(1, g.batch1) * std::max(1, g.batch2);
}

cudaError_t run(const GemmArgs& g, cudaStream_t stream, int max_ctas) {
    if (g.M <= 0 || g.N <= 0 || g.K <= 0) return cudaErrorInvalidValue;
    if (g.K % 8 != 0) return cudaErrorInvalidValue;  // TMA: 16-byte strides
    int BN = g.block_n;
    if (BN == 0) BN = g.N >= 256 ? 256 : (g.N > 64 ? 128 : 64);
    if (BN != 256 && BN != 128 && BN != 64) return cudaErrorInvalidValue;
    Params P{};
    P.M = (int)g.M;
    P.N = (int)g.N;
    P.K = (int)g.K;
    P.batch1 = g.batch1 > 0 ? g.batch1 : 1;
    P.batch2 = g.batch2 > 0 ? g.batch2 : 1;
    P.tiles_m = (P.M + BM - 1) / BM;
    P.tiles_n = (P.N + BN - 1) / BN;
    P.num_tiles = P.tiles_m * P.tiles_n * P.batch1 * P.batch2;
    P.k_blocks = (P.K + BK - 1) / BK;
    P.a_mn = g.a_mn_major;
    P.b_mn = g.b_mn_major;
    P.C = g.C;
    P.c_f32 = g.c_f32;
    P.ldc = g.ldc;
    P.c_s1 = g.c_s1;
    P.c_s2 = g.c_s2;
    P.bias = g.bias;
    P.bias_f32 = g.bias_f32;
    P.res = static_cast<const uint16_t*>(g.residual);
    P.ld_res = g.ld_res;
    P.res_s1 = g.res_s1;
    P.res_s2 = g.res_s2;
    P.aux = static_cast<uint16_t*>(g.aux);
    P.ld_aux = g.ld_aux;
    P.aux_s1 = g.aux_s1;
    P.aux_s2 = g.aux_s2;
    P.alpha = g.alpha;
    P.beta = g.beta;
    P.epi = g.epilogue;
    P.causal = g.causal;
    {
        const long long align = 4;  // 4-element vectors: 16 B fp32 / 8 B bf16
        P.vec_c = (reinterpret_cast<uintptr_t>(g.C) % (g.c_f32 ? 16 : 8) == 0) && g.ldc % align == 0 && g.c_s1 % align == 0 &&
                  g.c_s2 % align == 0;
        P.vec_aux = (reinterpret_cast<uintptr_t>(g.aux) % 8 == 0) && g.ld_aux % 4 == 0 && g.aux_s1 % 4 == 0 &&
                    g.aux_s2 % 4 == 0;
        const long long e16 = g.c_f32 ? 4 : 8;
        P.vec16_c = (reinterpret_cast<uintptr_t>(g.C) % 16 == 0) && g.ldc % e16 == 0 && g.c_s1 % e16 == 0 &&
                    g.c_s2 % e16 == 0;
        P.vec16_aux = (reinterpret_cast<uintptr_t>(g.aux) % 16 == 0) && g.ld_aux % 8 == 0 && g.aux_s1 % 8 == 0 &&
                      g.aux_s2 % 8 == 0;
        P.staged = 0;
        P.vec_bias = !g.bias_f32 && (reinterpret_cast<uintptr_t>(g.bias) % 16 == 0);
        P.vec16_res = (reinterpret_cast<uintptr_t>(g.residual) % 16 == 0) && g.ld_res % 8 == 0 && g.res_s1 % 8 == 0 &&
                      g.res_s2 % 8 == 0;
    }

    // CTA pairs (cta_group::2, M = 256 over two adjacent M tiles sharing the B tile): each SM
    // stages and the MMA reads half of B, so smem traffic per k-block drops from 48 to 32 KB
    // and L2 -> SM traffic for B halves. Causal tiles have per-tile K ranges: unpaired.
    const int CS = (BN == 256 && g.causal == kCausalNone && P.tiles_m >= 2) ? 2 : 1;
    if (CS > 1) P.num_tiles = ((P.tiles_m + CS - 1) / CS) * P.tiles_n * P.batch1 * P.batch2;
    {
        const int G = kNumSMs / CS;  // clusters
        const int waves = (P.num_tiles + G - 1) / G;
        const double eff = (double)P.num_tiles / ((double)waves * G);
        const int tail = P.num_tiles - (P.num_tiles / G) * G;
        // Stream-K when the data-parallel tile count fills the last wave poorly (e.g. 512 tiles on
        // 148 SMs -> 86 % of 4 waves): every CTA then gets the same number of k-block iterations.
        P.sk = ((max_ctas <= 0 || max_ctas >= kNumSMs) && g.causal == kCausalNone && P.num_tiles >= G && eff < 0.9 && BN == 256 && tail > 0 &&
                2 * tail <= G && P.k_blocks >= 64) ? 1 : 0;  // measured: +4% at K=8192, -2% at K=2048
    }
    if (P.sk) {
        // partial-tile workspace + hand-off flags, one set per (device, stream): GEMMs on
        // different streams (e.g. in-process DP ranks) may run concurrently; on one stream they
        // are ordered, so the epoch counter tells consecutive launches apart
        struct SkState {
            float* ws = nullptr;
            unsigned* flags = nullptr;
            unsigned epoch = 0;
        };
        static std::mutex mu;
        static std::map<std::pair<int, cudaStream_t>, SkState> states;
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(mu);
        SkState& S = states[{dev, stream}];
        if (!S.ws) {
            if (cudaMalloc(&S.ws, (size_t)kNumSMs * BM * 256 * 4) != cudaSuccess ||
                cudaMalloc(&S.flags, kNumSMs * sizeof(unsigned)) != cudaSuccess ||
                cudaMemsetAsync(S.flags, 0, kNumSMs * sizeof(unsigned), stream) != cudaSuccess)
                return cudaErrorMemoryAllocation;
        }
        P.sk_ws = S.ws;
        P.sk_flags = S.flags;
        P.sk_epoch = ++S.epoch;
        if (P.sk_epoch == 0) P.sk_epoch = ++S.epoch;  // flags start at 0
    }
    CUtensorMap ma, mb;
    const bool ok_a = g.a_mn_major
                          ? make_map(&ma, g.A, g.M, g.K, g.lda, P.batch1, g.a_s1, P.batch2, g.a_s2, 64, 64)
                          : make_map(&ma, g.A, g.K, g.M, g.lda, P.batch1, g.a_s1, P.batch2, g.a_s2, 64, BM);
    const bool ok_b = g.b_mn_major
                          ? make_map(&mb, g.B, g.N, g.K, g.ldb, P.batch1, g.b_s1, P.batch2, g.b_s2, 64, 64)
                          : make_map(&mb, g.B, g.K, g.N, g.ldb, P.batch1, g.b_s1, P.batch2, g.b_s2, 64, BN / CS);
    if (!ok_a || !ok_b) return cudaErrorInvalidValue;
    // bf16 C through TMA bulk stores (16-byte aligned base and strides; OOB rows/cols clipped)
    CUtensorMap mc;
    std::memset(&mc, 0, sizeof(mc));
    P.tma_c = 0;
    if (!g.c_f32 && (reinterpret_cast<uintptr_t>(g.C) % 16 == 0) && g.ldc % 8 == 0 && (P.batch1 == 1 || g.c_s1 % 8 == 0) &&
        (P.batch2 == 1 || g.c_s2 % 8 == 0))
        P.tma_c = make_map_sw(&mc, g.C, g.N, g.M, g.ldc, P.batch1, g.c_s1, P.batch2, g.c_s2, 32, 32,
                              CU_TENSOR_MAP_SWIZZLE_64B) ? 1 : 0;
    P.fast = P.tma_c && g.alpha == 1.f && g.beta == 0.f && P.N % BN == 0 &&
             (!(g.epilogue & kEpiBias) || P.vec_bias) && (!(g.epilogue & kEpiResidual) || P.vec16_res) &&
             (!(g.epilogue & (kEpiAux | kEpiGeluBwd)) || P.vec16_aux);
    const int max_clusters = kNumSMs / CS;
    int grid = P.sk ? kNumSMs : (P.num_tiles < max_clusters ? P.num_tiles : max_clusters) * CS;
    if (max_ctas > 0 && grid > max_ctas) grid = (max_ctas / CS) * CS;
    cudaEvent_t ta = nullptr, tb = nullptr;
    bool timed = false;
    {
        std::lock_guard<std::mutex> lk(timing().mu);
        timed = timing().on;
        if (timed) {
            ta = timing().take();
            tb = timing().take();
        }
    }
    if (timed) cudaEventRecord(ta, stream);
    cudaError_t e;
    if (BN == 256)
        e = CS == 2 ? launch_cfg<256, 6, 2>(ma, mb, mc, P, grid, stream) : launch_cfg<256, 4, 1>(ma, mb, mc, P, grid, stream);
    else if (BN == 128)
        e = launch_cfg<128, 6, 1>(ma, mb, mc, P, grid, stream);
    else
        e = launch_cfg<64, 8, 1>(ma, mb, mc, P, grid, stream);
    if (timed) {
        cudaEventRecord(tb, stream);
        std::lock_guard<std::mutex> lk(timing().mu);
        char shape[160];
        std::snprintf(shape, sizeof shape, "M=%lld N=%lld K=%lld z=%d a_mn=%d b_mn=%d causal=%d epi=%d f32=%d BN=%d CS=%d sk=%d grid=%d",
                      g.M, g.N, g.K, g.batch1 * (g.batch2 > 0 ? g.batch2 : 1), g.a_mn_major, g.b_mn_major, g.causal,
                      g.epilogue, g.c_f32, BN, CS, (int)P.sk, grid);
        timing().recs.push_back({ta, tb, executed_flops(g), shape});
    }
    return e;
}

}  // namespace gemm
}  // namespace ah
