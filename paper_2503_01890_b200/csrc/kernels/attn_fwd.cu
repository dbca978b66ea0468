// Fused causal attention forward on tcgen05 (sm_100a): S = Q K^T, softmax, O = P V in one
// kernel per (128-query tile, head, sequence), S and O accumulated in TMEM, Q/K/V staged by TMA.
//
// Two passes over the key tiles: pass 1 computes the exact row max / sum, pass 2 recomputes
// S and emits the final normalised P (bf16) both to shared memory (the A operand of P·V) and
// to HBM (the backward consumes it: same layout and zero-fill contract as softmax_fwd), so the
// O accumulator never needs the online-softmax rescale. Compared with GEMM(S fp32) + softmax +
// GEMM(P V) this removes the fp32 score round trip through HBM.
//
// Warp roles (384 threads): 0 TMA producer, 1 MMA issuer (single thread), 2 TMEM allocator,
// 4-11 softmax / epilogue (thread = query row, two warps per row quarter splitting the keys;
// warp w reads TMEM lanes 32*(w%4)...).
// TMEM: S double buffer (2 x 128 fp32 columns) + O (128 columns).
// Shapes: head_dim = 128, seq_len % 128 == 0.
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "gpt_kernels.h"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace ah {
namespace gpt {
namespace {

using namespace ah::tc;

constexpr int kHD = 128, kBQ = 128, kBK = 128;
constexpr uint32_t kTile = kBQ * kHD * 2;  // 32 KB: one 128 x 128 bf16 operand tile
constexpr int kThreads = 384;  // + 8 softmax warps (4..11)

struct AttnParams {
    int s, nh, B, h;
    float scale_log2;  // softmax scale * log2(e)
    uint16_t* P;       // [B][nh][s][s]
    uint16_t* O;       // [B][s][h], head slice at head * hd
};

__global__ void __launch_bounds__(kThreads, 1)
attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnParams A) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;
    uint8_t* sK = sm + kTile;          // 2 stages
    uint8_t* sV = sm + 3 * kTile;      // 2 stages
    uint8_t* sP = sm + 5 * kTile;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 6 * kTile);
    uint64_t* bar_q = bar;
    uint64_t* kv_full = bar + 1;   // [2]
    uint64_t* kv_empty = bar + 3;  // [2]
    uint64_t* s_full = bar + 5;    // [2]
    uint64_t* s_free = bar + 7;    // [2]
    uint64_t* p_full = bar + 9;
    uint64_t* p_free = bar + 10;
    uint64_t* o_full = bar + 11;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bar + 12);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqt = A.s / kBQ;
    const int qt = nqt - 1 - (int)blockIdx.x;  // heavy (long causal) tiles first
    const int head = blockIdx.y, b = blockIdx.z;
    const int n = qt + 1;                      // key tiles 0..qt

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmV)) : "memory");
        mbar_init(smem_u32(bar_q), 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&kv_full[i]), 1);
            mbar_init(smem_u32(&kv_empty[i]), 1);
            mbar_init(smem_u32(&s_full[i]), 1);
            mbar_init(smem_u32(&s_free[i]), 8);
        }
        mbar_init(smem_u32(p_full), 8);
        mbar_init(smem_u32(p_free), 1);
        mbar_init(smem_u32(o_full), 1);
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

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer =====
            const uint32_t bq = smem_u32(bar_q);
            mbar_expect_tx(bq, kTile);
            tma_load_4d(smem_u32(sQ), &tmQ, bq, 0, qt * kBQ, head, b);
            tma_load_4d(smem_u32(sQ) + kTile / 2, &tmQ, bq, 64, qt * kBQ, head, b);
            for (int k = 0; k < 2 * n; ++k) {  // ring items: pass 1 (K only), pass 2 (K + V)
                const int st = k & 1, j = k < n ? k : k - n;
                mbar_wait(smem_u32(&kv_empty[st]), ((k >> 1) & 1) ^ 1);
                const uint32_t fb = smem_u32(&kv_full[st]);
                const bool with_v = k >= n;
                mbar_expect_tx(fb, with_v ? 2 * kTile : kTile);
                const uint32_t dk = smem_u32(sK + st * kTile);
                tma_load_4d(dk, &tmK, fb, 0, j * kBK, head, b);
                tma_load_4d(dk + kTile / 2, &tmK, fb, 64, j * kBK, head, b);
                if (with_v) {
                    const uint32_t dv = smem_u32(sV + st * kTile);
#pragma unroll
                    for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                        for (int c = 0; c < 2; ++c)
                            tma_load_4d(dv + kb * (kTile / 2) + c * (kTile / 4), &tmV, fb, c * 64, j * kBK + kb * 64,
                                        head, b);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer =====
            constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);
            constexpr uint32_t idO = idesc_bf16(128, 128, 0, 1);
            mbar_wait(smem_u32(bar_q), 0);
            auto issue_S = [&](int k, int g) {  // ring item k -> S buffer g & 1
                const int st = k & 1, buf = g & 1, u = g >> 1;
                mbar_wait(smem_u32(&kv_full[st]), (k >> 1) & 1);
                mbar_wait(smem_u32(&s_free[buf]), (u & 1) ^ 1);
                fence_after();
                const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK + st * kTile);
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const uint32_t off = (t >> 2) * (kTile / 2) + (t & 3) * 32;
                    mma_f16(tmem + buf * 128, sdesc(qa + off, 16, 1024), sdesc(ka + off, 16, 1024), idS, t > 0);
                }
                commit(smem_u32(&s_full[buf]));
            };
            for (int j = 0; j < n; ++j) {  // pass 1: scores only
                issue_S(j, j);
                commit(smem_u32(&kv_empty[j & 1]));
            }
            issue_S(n, n);
            for (int j = 0; j < n; ++j) {  // pass 2: scores of j+1 overlap the softmax of j
                const int k = n + j;
                if (j + 1 < n) issue_S(k + 1, n + j + 1);
                mbar_wait(smem_u32(p_full), j & 1);
                fence_after();
                const uint32_t pa = smem_u32(sP), va = smem_u32(sV + (k & 1) * kTile);
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const uint64_t ad = sdesc(pa + (t >> 2) * (kTile / 2) + (t & 3) * 32, 16, 1024);
                    const uint64_t bd = sdesc(va + (t >> 2) * (kTile / 2) + (t & 3) * 2048, kTile / 4, 1024);
                    mma_f16(tmem + 256, ad, bd, idO, (j > 0 || t > 0) ? 1u : 0u);
                }
                commit(smem_u32(p_free));
                commit(smem_u32(&kv_empty[k & 1]));
            }
            commit(smem_u32(o_full));
        }
    } else if (warp >= 4) {  // ===== softmax / epilogue: thread = query row, one half of the keys =====
        // 8 warps: two per TMEM lane quarter, each owning 64 of a tile's 128 key columns, so
        // each SM sub-partition runs two independent exp2 streams.
        const int half = (warp - 4) >> 2;
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
        const int q = qt * kBQ + r;
        float* red = reinterpret_cast<float*>(tmem_holder + 4);  // [2 halves][2 (m, l)][128 rows]
        // Work in the log2 domain on raw scores: max over raw S (the scale is positive), then
        // p = 2^(S * scale_log2 - m * scale_log2). Only the diagonal tile (j == qt) is masked.
        const float sl2 = A.scale_log2;
        float m = -INFINITY, l = 0.f;  // m: raw-score max of this half's keys
        for (int j = 0; j < n; ++j) {  // pass 1: exact row max and sum over this half's keys
            const int buf = j & 1, u = j >> 1;
            mbar_wait(smem_u32(&s_full[buf]), u & 1);
            fence_after();
            float v[64];
            ld32(tmem + lane_base + buf * 128 + half * 64, *reinterpret_cast<float(*)[32]>(v));
            ld32(tmem + lane_base + buf * 128 + half * 64 + 32, *reinterpret_cast<float(*)[32]>(v + 32));
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&s_free[buf]));  // scores are in registers now
            if (j == qt) {
                const int lim = q - j * kBK - half * 64;  // keys <= q stay
#pragma unroll
                for (int i = 0; i < 64; ++i) v[i] = i <= lim ? v[i] : -INFINITY;
            }
            float cm = v[0];
#pragma unroll
            for (int i = 1; i < 64; ++i) cm = fmaxf(cm, v[i]);
            if (cm == -INFINITY) continue;  // fully masked half row
            const float mn = fmaxf(m, cm);
            const float mb = mn * sl2;
            float add = 0.f;
#pragma unroll
            for (int i = 0; i < 64; ++i) add += ex2_approx(fmaf(v[i], sl2, -mb));
            l = (m == -INFINITY ? 0.f : l * ex2_approx((m - mn) * sl2)) + add;
            m = mn;
        }
        red[(half * 2 + 0) * 128 + r] = m;
        red[(half * 2 + 1) * 128 + r] = l;
        asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 softmax warps only
        {
            const float mo = red[((half ^ 1) * 2 + 0) * 128 + r], lo = red[((half ^ 1) * 2 + 1) * 128 + r];
            const float mt = fmaxf(m, mo);
            l = (m == -INFINITY ? 0.f : l * ex2_approx((m - mt) * sl2)) + (mo == -INFINITY ? 0.f : lo * ex2_approx((mo - mt) * sl2));
            m = mt;
        }
        // p = 2^(S * sl2 - (m * sl2 + log2 l)): normalisation folded into the exponent
        const float off = fmaf(m, sl2, __log2f(l));
        uint16_t* prow = A.P + (((size_t)b * A.nh + head) * A.s + q) * (size_t)A.s;
        for (int j = 0; j < n; ++j) {  // pass 2: normalised P -> smem (A operand) + HBM
            const int g = n + j, buf = g & 1, u = g >> 1;
            mbar_wait(smem_u32(&s_full[buf]), u & 1);
            fence_after();
            float v[64];
            ld32(tmem + lane_base + buf * 128 + half * 64, *reinterpret_cast<float(*)[32]>(v));
            ld32(tmem + lane_base + buf * 128 + half * 64 + 32, *reinterpret_cast<float(*)[32]>(v + 32));
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&s_free[buf]));
            uint32_t w[32];
#pragma unroll
            for (int i = 0; i < 32; ++i)
                w[i] = pack_bf16x2_rn(ex2_approx(fmaf(v[2 * i], sl2, -off)), ex2_approx(fmaf(v[2 * i + 1], sl2, -off)));
            if (j == qt) {  // causal mask of the diagonal tile: zero keys > q
                const int lim = q - j * kBK - half * 64;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const uint32_t keep = (2 * i <= lim ? 0x0000ffffu : 0u) | (2 * i + 1 <= lim ? 0xffff0000u : 0u);
                    w[i] &= keep;
                }
            }
            if (j > 0) mbar_wait(smem_u32(p_free), (j - 1) & 1);
            // smem: K-major SWIZZLE_128B tile; this half's 64 keys are atom `half`
            uint8_t* rowp = sP + half * (kTile / 2) + r * 128;
#pragma unroll
            for (int k8 = 0; k8 < 8; ++k8)
                *reinterpret_cast<uint4*>(rowp + ((k8 ^ (r & 7)) << 4)) = make_uint4(w[4 * k8], w[4 * k8 + 1], w[4 * k8 + 2], w[4 * k8 + 3]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P visible to the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(p_full));
            uint4* gp = reinterpret_cast<uint4*>(prow + j * kBK + half * 64);
#pragma unroll
            for (int k8 = 0; k8 < 8; ++k8) gp[k8] = make_uint4(w[4 * k8], w[4 * k8 + 1], w[4 * k8 + 2], w[4 * k8 + 3]);
        }
        mbar_wait(smem_u32(o_full), 0);
        fence_after();
        uint16_t* orow = A.O + ((size_t)b * A.s + q) * A.h + (size_t)head * kHD;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
            float v[32];
            const int col0 = half * 64 + c * 32;
            ld32(tmem + lane_base + 256 + col0, v);
            uint4* op = reinterpret_cast<uint4*>(orow + col0);
#pragma unroll
            for (int k8 = 0; k8 < 4; ++k8)
                op[k8] = make_uint4(pack_bf16x2_rn(v[8 * k8], v[8 * k8 + 1]), pack_bf16x2_rn(v[8 * k8 + 2], v[8 * k8 + 3]),
                                    pack_bf16x2_rn(v[8 * k8 + 4], v[8 * k8 + 5]), pack_bf16x2_rn(v[8 * k8 + 6], v[8 * k8 + 7]));
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
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

// Head view of the [B, s, 3h] qkv buffer: dims {hd, s, nh, B}.
bool head_map(CUtensorMap* m, const uint16_t* base, int s, int nh, int B, int h, int box_inner, int box_rows) {
    EncodeFn fn = encode();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)kHD, (cuuint64_t)s, (cuuint64_t)nh, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)3 * h * 2, (cuuint64_t)kHD * 2, (cuuint64_t)s * 3 * h * 2};
    cuuint32_t box[4] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool attn_fwd_supported(int hd, int s) { return hd == kHD && s % kBQ == 0; }

cudaError_t attn_fwd(const uint16_t* qkv, uint16_t* P, uint16_t* O, int B, int s, int nh, int hd, float scale,
                     cudaStream_t st) {
    if (!attn_fwd_supported(hd, s)) return cudaErrorInvalidValue;
    const int h = nh * hd;
    CUtensorMap mq, mk, mv;
    if (!head_map(&mq, qkv, s, nh, B, h, 64, 128) || !head_map(&mk, qkv + h, s, nh, B, h, 64, 128) ||
        !head_map(&mv, qkv + 2 * h, s, nh, B, h, 64, 64))
        return cudaErrorInvalidValue;
    AttnParams a;
    a.s = s;
    a.nh = nh;
    a.B = B;
    a.h = h;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.P = P;
    a.O = O;
    const size_t smem = 1024 + 6 * (size_t)kTile + 16 * 8 + 4 * 128 * 4;
    static bool cfg = false;
    if (!cfg) {
        cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        cfg = true;
    }
    attn_fwd_kernel<<<dim3(s / kBQ, nh, B), kThreads, smem, st>>>(mq, mk, mv, a);
    return launched(1);
}

}  // namespace gpt
}  // namespace ah
