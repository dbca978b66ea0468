// Fused causal attention backward on tcgen05 (sm_100a), one CTA per (128-key tile, head, seq).
//
// For every query tile i >= key tile kt (causal), with P saved by the forward:
//   dP_i = dO_i V^T                (TMEM, double-buffered)
//   dV  += P_i^T dO_i              (TMEM accumulator)
//   dS_i = P_i * (dP_i - D_i)      (softmax warps; D = rowsum(dO * O) precomputed)
//   dK  += dS_i^T Q_i              (TMEM accumulator)
// dS_i also goes to HBM for the dQ = dS K GEMM (K_UPTO_M), which keeps dQ deterministic
// without cross-CTA accumulation. Replaces GEMM(dP fp32) + softmax_bwd + GEMM(dV) + GEMM(dK):
// the fp32 dP round trip through HBM disappears.
//
// Shared-memory trick: a SWIZZLE_128B tile loaded K-major ([rows][64-col atoms]) is byte-for-
// byte the MN-major operand layout of its transpose (8 KB per 64-row box), so dO, Q, P and dS
// are each staged once and read by the tensor core in both orientations.
// Warp roles (384 threads): 0 TMA, 1 MMA issuer, 2 TMEM allocator, 4-11 softmax / epilogue.
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

constexpr int kHD = 128, kT = 128;
constexpr uint32_t kTile = kT * 128 * 2;  // 32 KB
constexpr int kThreads = 384;

struct BwdParams {
    int s, nh, B, h;
    float scale;          // softmax scale (dK, dQ factor)
    const float* D;       // [B][nh][s]
    uint16_t* dS;         // [B][nh][s][s]
    uint16_t* dqkv;       // [B][s][3h]
};

// K-major SWIZZLE_128B view as the MN-major operand of the transpose: LBO = atom stride.
__device__ __forceinline__ uint64_t mn_desc(uint32_t base, int t) { return sdesc(base + t * 2048, kTile / 2, 1024); }
__device__ __forceinline__ uint64_t k_desc(uint32_t base, int t) {
    return sdesc(base + (t >> 2) * (kTile / 2) + (t & 3) * 32, 16, 1024);
}

__global__ void __launch_bounds__(kThreads, 1)
attn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmV,
                const __grid_constant__ CUtensorMap tmdO, const __grid_constant__ CUtensorMap tmP, const BwdParams A) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sV = sm;                   // keys x hd, K-major
    uint8_t* sQ = sm + kTile;           // q x hd (single buffer)
    uint8_t* sdS = sm + 2 * kTile;      // q x keys
    uint8_t* sdO = sm + 3 * kTile;      // [2] q x hd
    uint8_t* sP = sm + 5 * kTile;       // [2] q x keys
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 7 * kTile);
    uint64_t* v_full = bar;
    uint64_t* st_full = bar + 1;   // [2]
    uint64_t* st_empty = bar + 3;  // [2]
    uint64_t* q_full = bar + 5;
    uint64_t* q_empty = bar + 6;
    uint64_t* dp_full = bar + 7;   // [2]
    uint64_t* dp_free = bar + 9;   // [2]
    uint64_t* ds_full = bar + 11;
    uint64_t* ds_free = bar + 12;
    uint64_t* acc_full = bar + 13;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bar + 14);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt = A.s / kT;
    const int kt = (int)blockIdx.x;  // 0 = longest (most query tiles) first
    const int head = blockIdx.y, b = blockIdx.z;
    const int nq = nt - kt;          // query tiles kt .. nt-1

    if (warp == 0 && lane == 0) {
        for (const CUtensorMap* m : {&tmQ, &tmV, &tmdO, &tmP})
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
        mbar_init(smem_u32(v_full), 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&st_full[i]), 1);
            mbar_init(smem_u32(&st_empty[i]), 1 + 8);  // dV MMA commit + 8 softmax warps (read P)
            mbar_init(smem_u32(&dp_full[i]), 1);
            mbar_init(smem_u32(&dp_free[i]), 8);
        }
        mbar_init(smem_u32(q_full), 1);
        mbar_init(smem_u32(q_empty), 1);
        mbar_init(smem_u32(ds_full), 8);
        mbar_init(smem_u32(ds_free), 1);
        mbar_init(smem_u32(acc_full), 1);
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
    const uint32_t tmem = *tmem_holder;  // dP[0] 0-127, dP[1] 128-255, dV 256-383, dK 384-511

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer =====
            const uint32_t vb = smem_u32(v_full);
            mbar_expect_tx(vb, kTile);
            tma_load_4d(smem_u32(sV), &tmV, vb, 0, kt * kT, head, b);
            tma_load_4d(smem_u32(sV) + kTile / 2, &tmV, vb, 64, kt * kT, head, b);
            for (int i = 0; i < nq; ++i) {
                const int qi = kt + i, st = i & 1;
                mbar_wait(smem_u32(&st_empty[st]), ((i >> 1) & 1) ^ 1);
                const uint32_t fb = smem_u32(&st_full[st]);
                mbar_expect_tx(fb, 2 * kTile);
                const uint32_t dd = smem_u32(sdO + st * kTile), dp = smem_u32(sP + st * kTile);
                tma_load_4d(dd, &tmdO, fb, 0, qi * kT, head, b);
                tma_load_4d(dd + kTile / 2, &tmdO, fb, 64, qi * kT, head, b);
                tma_load_4d(dp, &tmP, fb, kt * kT, qi * kT, head, b);
                tma_load_4d(dp + kTile / 2, &tmP, fb, kt * kT + 64, qi * kT, head, b);
                mbar_wait(smem_u32(q_empty), (i & 1) ^ 1);
                const uint32_t qb = smem_u32(q_full);
                mbar_expect_tx(qb, kTile);
                tma_load_4d(smem_u32(sQ), &tmQ, qb, 0, qi * kT, head, b);
                tma_load_4d(smem_u32(sQ) + kTile / 2, &tmQ, qb, 64, qi * kT, head, b);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer =====
            constexpr uint32_t idDP = idesc_bf16(128, 128, 0, 0);  // dO (K-major) x V^T (K-major)
            constexpr uint32_t idACC = idesc_bf16(128, 128, 1, 1); // X^T (MN-major) x Y (MN-major)
            mbar_wait(smem_u32(v_full), 0);
            auto stage_mmas = [&](int i) {  // dP_i and dV += P_i^T dO_i
                const int st = i & 1, buf = i & 1;
                mbar_wait(smem_u32(&st_full[st]), (i >> 1) & 1);
                mbar_wait(smem_u32(&dp_free[buf]), ((i >> 1) & 1) ^ 1);
                fence_after();
                const uint32_t dd = smem_u32(sdO + st * kTile), pp = smem_u32(sP + st * kTile), vv = smem_u32(sV);
#pragma unroll
                for (int t = 0; t < 8; ++t) mma_f16(tmem + buf * 128, k_desc(dd, t), k_desc(vv, t), idDP, t > 0);
                commit(smem_u32(&dp_full[buf]));
#pragma unroll
                for (int t = 0; t < 8; ++t) mma_f16(tmem + 256, mn_desc(pp, t), mn_desc(dd, t), idACC, (i > 0 || t > 0));
                commit(smem_u32(&st_empty[st]));
            };
            stage_mmas(0);
            for (int i = 0; i < nq; ++i) {
                if (i + 1 < nq) stage_mmas(i + 1);
                mbar_wait(smem_u32(ds_full), i & 1);
                mbar_wait(smem_u32(q_full), i & 1);
                fence_after();
                const uint32_t ds = smem_u32(sdS), qq = smem_u32(sQ);
#pragma unroll
                for (int t = 0; t < 8; ++t) mma_f16(tmem + 384, mn_desc(ds, t), mn_desc(qq, t), idACC, (i > 0 || t > 0));
                commit(smem_u32(ds_free));
                commit(smem_u32(q_empty));
            }
            commit(smem_u32(acc_full));
        }
    } else if (warp >= 4) {  // ===== dS = P (dP - D); epilogue =====
        const int half = (warp - 4) >> 2;  // key columns [64*half, 64*half + 64)
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
        for (int i = 0; i < nq; ++i) {
            const int qi = kt + i, st = i & 1, buf = i & 1;
            const int q = qi * kT + r;
            const float Dq = A.D[((size_t)b * A.nh + head) * A.s + q];
            mbar_wait(smem_u32(&dp_full[buf]), (i >> 1) & 1);
            fence_after();
            if (i > 0) mbar_wait(smem_u32(ds_free), (i - 1) & 1);
            const uint8_t* prow = sP + st * kTile + half * (kTile / 2) + r * 128;
            uint8_t* drow = sdS + half * (kTile / 2) + r * 128;
            uint16_t* grow = A.dS + (((size_t)b * A.nh + head) * A.s + q) * (size_t)A.s + kt * kT + half * 64;
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                float v[32];
                ld32(tmem + lane_base + buf * 128 + half * 64 + c * 32, v);
#pragma unroll
                for (int k8 = 0; k8 < 4; ++k8) {
                    const int chunk = (c * 4 + k8) ^ (r & 7);
                    const uint4 pw = *reinterpret_cast<const uint4*>(prow + chunk * 16);
                    const uint32_t pu[4] = {pw.x, pw.y, pw.z, pw.w};
                    uint32_t o[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float p0 = bf16_bits_to_f32(pu[e] & 0xffffu), p1 = bf16_bits_to_f32(pu[e] >> 16);
                        o[e] = pack_bf16x2(p0 * (v[8 * k8 + 2 * e] - Dq), p1 * (v[8 * k8 + 2 * e + 1] - Dq));
                    }
                    const uint4 ow = make_uint4(o[0], o[1], o[2], o[3]);
                    *reinterpret_cast<uint4*>(drow + chunk * 16) = ow;
                    *reinterpret_cast<uint4*>(grow + c * 32 + k8 * 8) = ow;
                }
            }
            fence_before();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(smem_u32(&dp_free[buf]));
                mbar_arrive(smem_u32(&st_empty[st]));
                mbar_arrive(smem_u32(ds_full));
            }
        }
        mbar_wait(smem_u32(acc_full), 0);
        fence_after();
        // thread r = key row of the tile: dV, dK (x scale) -> dqkv
        uint16_t* base = A.dqkv + ((size_t)b * A.s + (size_t)kt * kT + r) * 3 * A.h + (size_t)head * kHD + half * 64;
#pragma unroll 1
        for (int which = 0; which < 2; ++which) {  // 0: dV (col 256), 1: dK (col 384)
            uint16_t* dst = base + (which == 0 ? 2 * A.h : A.h);
            const float f = which == 0 ? 1.f : A.scale;
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                float v[32];
                ld32(tmem + lane_base + 256 + which * 128 + half * 64 + c * 32, v);
                uint4* op = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
                for (int k8 = 0; k8 < 4; ++k8)
                    op[k8] = make_uint4(pack_bf16x2(v[8 * k8] * f, v[8 * k8 + 1] * f), pack_bf16x2(v[8 * k8 + 2] * f, v[8 * k8 + 3] * f),
                                        pack_bf16x2(v[8 * k8 + 4] * f, v[8 * k8 + 5] * f), pack_bf16x2(v[8 * k8 + 6] * f, v[8 * k8 + 7] * f));
            }
        }
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

bool map4(CUtensorMap* m, const void* base, cuuint64_t d0, cuuint64_t d1, cuuint64_t d2, cuuint64_t d3, cuuint64_t s1,
          cuuint64_t s2, cuuint64_t s3) {
    EncodeFn fn = encode();
    if (!fn) return false;
    cuuint64_t dims[4] = {d0, d1, d2, d3};
    cuuint64_t strides[3] = {s1 * 2, s2 * 2, s3 * 2};
    cuuint32_t box[4] = {64, 128, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool attn_bwd_supported(int hd, int s) { return hd == kHD && s % kT == 0; }

cudaError_t attn_rowdot(const uint16_t* dO, const uint16_t* O, float* D, int B, int s, int nh, cudaStream_t st) {
    launch_ex(attn_bwd_dot_kernel, dim3(kNumSMs * 8), dim3(256), 0, st, 1, dO, O, D, B, s, nh);
    return launched(1);
}

cudaError_t attn_bwd(const uint16_t* qkv, const uint16_t* O, const uint16_t* dO, const uint16_t* P, float* D,
                     uint16_t* dS, uint16_t* dqkv, int B, int s, int nh, int hd, float scale, cudaStream_t st) {
    if (!attn_bwd_supported(hd, s)) return cudaErrorInvalidValue;
    const int h = nh * hd;
    launch_ex(attn_bwd_dot_kernel, dim3(kNumSMs * 8), dim3(256), 0, st, 1, dO, O, D, B, s, nh);
    launched(1);
    CUtensorMap mq, mv, mdo, mp;
    const cuuint64_t row3 = 3ull * h;
    if (!map4(&mq, qkv, hd, s, nh, B, row3, hd, (cuuint64_t)s * row3) ||
        !map4(&mv, qkv + 2 * h, hd, s, nh, B, row3, hd, (cuuint64_t)s * row3) ||
        !map4(&mdo, dO, hd, s, nh, B, h, hd, (cuuint64_t)s * h) ||
        !map4(&mp, P, s, s, nh, B, s, (cuuint64_t)s * s, (cuuint64_t)nh * s * s))
        return cudaErrorInvalidValue;
    BwdParams a;
    a.s = s;
    a.nh = nh;
    a.B = B;
    a.h = h;
    a.scale = scale;
    a.D = D;
    a.dS = dS;
    a.dqkv = dqkv;
    const size_t smem = 1024 + 7 * (size_t)kTile + 16 * 8;
    static bool cfg = false;
    if (!cfg) {
        cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        cfg = true;
    }
    attn_bwd_kernel<<<dim3(s / kT, nh, B), kThreads, smem, st>>>(mq, mv, mdo, mp, a);
    return launched(1);
}

}  // namespace gpt
}  // namespace ah
