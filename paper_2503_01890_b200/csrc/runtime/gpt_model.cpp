// GPT-2 block forward / backward as sequences of tcgen05 GEMMs + HBM-bound kernels.
// Attention is computed per (head, sequence) with batched GEMMs over strided views of the
// [T, 3h] qkv buffer; causal structure is exploited by the GEMM's tile skipping.
#include "gpt_model.h"

#include <cmath>
#include <cstdlib>
#include <string>

#include "../kernels/gemm.h"
#include "../kernels/gpt_kernels.h"

namespace ah {

using gemm::GemmArgs;

namespace {

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

#define AH_TRY(expr)                               \
    do {                                           \
        const cudaError_t ah_e = (expr);           \
        if (ah_e != cudaSuccess) return ah_e;      \
    } while (0)

// Row-major activation X[T][K] times weight W[N][K]^T -> Y[T][N]  (forward, TN)
GemmArgs linear_fwd(const GptDims& d, const uint16_t* X, int K, const uint16_t* W, int N, void* Y) {
    GemmArgs g;
    g.M = d.T();
    g.N = N;
    g.K = K;
    g.A = X;
    g.lda = K;
    g.B = W;
    g.ldb = K;
    g.C = Y;
    g.ldc = N;
    return g;
}

// dX[T][K] = dY[T][N] . W[N][K]  (dgrad: B is W read MN-major)
GemmArgs linear_dgrad(const GptDims& d, const uint16_t* dY, int N, const uint16_t* W, int K, void* dX) {
    GemmArgs g;
    g.M = d.T();
    g.N = K;
    g.K = N;
    g.A = dY;
    g.lda = N;
    g.B = W;
    g.b_mn_major = 1;
    g.ldb = K;
    g.C = dX;
    g.ldc = K;
    return g;
}

// dW[N][K] = dY[T][N]^T . X[T][K]  (wgrad: both operands MN-major, reduction over tokens)
GemmArgs linear_wgrad(const GptDims& d, const uint16_t* dY, int N, const uint16_t* X, int K, void* dW) {
    GemmArgs g;
    g.M = N;
    g.N = K;
    g.K = d.T();
    g.A = dY;
    g.a_mn_major = 1;
    g.lda = N;
    g.B = X;
    g.b_mn_major = 1;
    g.ldb = K;
    g.C = dW;
    g.ldc = K;
    return g;
}

// Per-(head, sequence) view helpers: z1 = head, z2 = sequence.
void heads(GemmArgs& g, const GptDims& d) {
    g.batch1 = d.nh;
    g.batch2 = d.B;
}

}  // namespace

// head_dim 128 and s % 128 == 0 run the flash tcgen05 kernels; other shapes (e.g. head_dim 64)
// take the unfused path: S GEMM, softmax kernel, P V GEMM, with P kept for the backward.
AttnMode attention_mode(const GptDims& d) {
    return gpt::flash_supported(d.hd, d.s) ? AttnMode::Flash : AttnMode::Unfused;
}

namespace {
size_t saved_probs_bytes(const GptDims& d) {  // P (bf16, s x s per head) or lse2 (fp32 per row)
    const size_t rows = (size_t)d.B * d.nh * d.s;
    return attention_mode(d) == AttnMode::Flash ? rows * 4 : rows * d.s * 2;
}
}  // namespace

size_t BlockActs::bytes(const GptDims& d) {
    const size_t T = d.T(), h = d.h;
    size_t b = 0;
    b += align_up(T * h * 2);                        // ln1
    b += align_up(T * 3 * h * 2);                    // qkv
    b += align_up(saved_probs_bytes(d));             // P or lse2
    b += align_up(T * h * 2);                        // att
    b += align_up(T * h * 2);                        // x2
    b += align_up(T * h * 2);                        // ln2
    b += 2 * align_up(T * 4 * h * 2);                // fc_pre, gelu
    b += 4 * align_up(T * 4);                        // LN stats
    return b;
}

BlockActs BlockActs::carve(const GptDims& d, void* base) {
    const size_t T = d.T(), h = d.h;
    uint8_t* p = static_cast<uint8_t*>(base);
    auto take = [&](size_t n) {
        uint8_t* r = p;
        p += align_up(n);
        return r;
    };
    BlockActs a;
    a.ln1 = reinterpret_cast<uint16_t*>(take(T * h * 2));
    a.qkv = reinterpret_cast<uint16_t*>(take(T * 3 * h * 2));
    {
        uint8_t* pr = take(saved_probs_bytes(d));
        if (attention_mode(d) == AttnMode::Flash) {
            a.P = nullptr;
            a.lse2 = reinterpret_cast<float*>(pr);
        } else {
            a.P = reinterpret_cast<uint16_t*>(pr);
        }
    }
    a.att = reinterpret_cast<uint16_t*>(take(T * h * 2));
    a.x2 = reinterpret_cast<uint16_t*>(take(T * h * 2));
    a.ln2 = reinterpret_cast<uint16_t*>(take(T * h * 2));
    a.fc_pre = reinterpret_cast<uint16_t*>(take(T * 4 * h * 2));
    a.gelu = reinterpret_cast<uint16_t*>(take(T * 4 * h * 2));
    a.mean1 = reinterpret_cast<float*>(take(T * 4));
    a.rstd1 = reinterpret_cast<float*>(take(T * 4));
    a.mean2 = reinterpret_cast<float*>(take(T * 4));
    a.rstd2 = reinterpret_cast<float*>(take(T * 4));
    return a;
}

namespace {
size_t ws_s_bytes(const GptDims& d) {  // fp32 scores (unfused) or the row dot D (fused)
    const size_t rows = (size_t)d.B * d.nh * d.s;
    return attention_mode(d) == AttnMode::Unfused ? rows * d.s * 4 : rows * 4;
}
}  // namespace

size_t Workspace::bytes(const GptDims& d) {
    const size_t T = d.T(), h = d.h, Z = (size_t)d.B * d.nh;
    const size_t part_rows = (size_t)std::max(gpt::ln_bwd_ctas(d.T()), gpt::colsum_rows(d.T()));
    return align_up(ws_s_bytes(d)) + align_up(Z * d.s * d.s * 2) + align_up(T * 4 * h * 2) +
           align_up(T * 3 * h * 2) + 3 * align_up(T * h * 2) + align_up(part_rows * 4 * h * 4);
}

Workspace Workspace::carve(const GptDims& d, void* base) {
    const size_t T = d.T(), h = d.h, Z = (size_t)d.B * d.nh;
    const size_t part_rows = (size_t)std::max(gpt::ln_bwd_ctas(d.T()), gpt::colsum_rows(d.T()));
    uint8_t* p = static_cast<uint8_t*>(base);
    auto take = [&](size_t n) {
        uint8_t* r = p;
        p += align_up(n);
        return r;
    };
    Workspace w;
    w.S = reinterpret_cast<float*>(take(ws_s_bytes(d)));
    w.dS = reinterpret_cast<uint16_t*>(take(Z * d.s * d.s * 2));
    w.d4h = reinterpret_cast<uint16_t*>(take(T * 4 * h * 2));
    w.dqkv = reinterpret_cast<uint16_t*>(take(T * 3 * h * 2));
    w.dln = reinterpret_cast<uint16_t*>(take(T * h * 2));
    w.datt = reinterpret_cast<uint16_t*>(take(T * h * 2));
    w.dx2 = reinterpret_cast<uint16_t*>(take(T * h * 2));
    w.part = reinterpret_cast<float*>(take(part_rows * 4 * h * 4));
    return w;
}

cudaError_t block_forward(const GptDims& d, const uint16_t* W, const uint16_t* x_in, uint16_t* x_out,
                          const BlockActs& a, const Workspace& ws, cudaStream_t st) {
    const BlockLayout o = BlockLayout::make(d.h);
    const int h = d.h, T = d.T(), s = d.s, hd = d.hd;
    AH_TRY(gpt::ln_fwd(x_in, W + o.ln1_g, W + o.ln1_b, a.ln1, a.mean1, a.rstd1, T, h, st));
    {  // qkv = ln1 Wqkv^T + b
        GemmArgs g = linear_fwd(d, a.ln1, h, W + o.w_qkv, 3 * h, a.qkv);
        g.epilogue = gemm::kEpiBias;
        g.bias = W + o.b_qkv;
        AH_TRY(gemm::run(g, st));
    }
    const AttnMode mode = attention_mode(d);
    if (mode == AttnMode::Flash) {  // one tcgen05 kernel: S, online softmax, P V; keeps O and lse
        AH_TRY(gpt::flash_fwd(a.qkv, a.att, a.lse2, d.B, s, d.nh, hd, 1.0f / std::sqrt((float)hd), st));
    } else {
    {  // S = Q K^T / sqrt(hd), causal tiles only, fp32
        GemmArgs g;
        heads(g, d);
        g.M = s; g.N = s; g.K = hd;
        g.A = a.qkv; g.lda = 3 * h; g.a_s1 = hd; g.a_s2 = (long long)s * 3 * h;
        g.B = a.qkv + h; g.ldb = 3 * h; g.b_s1 = hd; g.b_s2 = (long long)s * 3 * h;
        g.C = ws.S; g.c_f32 = 1; g.ldc = s; g.c_s1 = (long long)s * s; g.c_s2 = (long long)d.nh * s * s;
        g.alpha = 1.0f / std::sqrt((float)hd);
        g.causal = gemm::kCausalSkipUpper;
        AH_TRY(gemm::run(g, st));
    }
    AH_TRY(gpt::softmax_fwd2(ws.S, a.P, (long long)d.B * d.nh * s, s, st));
    {  // att[b, t, head*hd + j] = sum_k P[t][k] V[k][j]
        GemmArgs g;
        heads(g, d);
        g.M = s; g.N = hd; g.K = s;
        g.A = a.P; g.lda = s; g.a_s1 = (long long)s * s; g.a_s2 = (long long)d.nh * s * s;
        g.B = a.qkv + 2 * h; g.b_mn_major = 1; g.ldb = 3 * h; g.b_s1 = hd; g.b_s2 = (long long)s * 3 * h;
        g.C = a.att; g.ldc = h; g.c_s1 = hd; g.c_s2 = (long long)s * h;
        g.causal = gemm::kCausalKUptoM;
        AH_TRY(gemm::run(g, st));
    }
    }  // unfused attention
    {  // x2 = x_in + att Wproj^T + b
        GemmArgs g = linear_fwd(d, a.att, h, W + o.w_proj, h, a.x2);
        g.epilogue = gemm::kEpiBias | gemm::kEpiResidual;
        g.bias = W + o.b_proj;
        g.residual = x_in;
        g.ld_res = h;
        AH_TRY(gemm::run(g, st));
    }
    AH_TRY(gpt::ln_fwd(a.x2, W + o.ln2_g, W + o.ln2_b, a.ln2, a.mean2, a.rstd2, T, h, st));
    {  // gelu = GELU(ln2 Wfc^T + b), pre-activation kept
        GemmArgs g = linear_fwd(d, a.ln2, h, W + o.w_fc, 4 * h, a.gelu);
        g.epilogue = gemm::kEpiBias | gemm::kEpiGelu | gemm::kEpiAux;
        g.bias = W + o.b_fc;
        g.aux = a.fc_pre;
        g.ld_aux = 4 * h;
        AH_TRY(gemm::run(g, st));
    }
    if (x_out) {  // x_out = x2 + gelu Wfc2^T + b   (skipped by a recompute: not saved)
        GemmArgs g = linear_fwd(d, a.gelu, 4 * h, W + o.w_fc2, h, x_out);
        g.epilogue = gemm::kEpiBias | gemm::kEpiResidual;
        g.bias = W + o.b_fc2;
        g.residual = a.x2;
        g.ld_res = h;
        AH_TRY(gemm::run(g, st));
    }
    return cudaSuccess;
}

cudaError_t block_backward(const GptDims& d, uint16_t* W, const uint16_t* x_in, const BlockActs& a,
                           const uint16_t* dy, uint16_t* dx, const Workspace& ws, cudaStream_t st) {
    const BlockLayout o = BlockLayout::make(d.h);
    const int h = d.h, T = d.T(), s = d.s, hd = d.hd;
    const float scale = 1.0f / std::sqrt((float)hd);

    // ---- MLP out: x_out = x2 + gelu Wfc2^T + b_fc2
    {  // dfc_pre = (dy Wfc2) * GELU'(fc_pre): GELU backward fused into the dgrad epilogue
        GemmArgs g = linear_dgrad(d, dy, h, W + o.w_fc2, 4 * h, ws.d4h);
        g.epilogue = gemm::kEpiGeluBwd;
        g.aux = a.fc_pre;
        g.ld_aux = 4 * h;
        AH_TRY(gemm::run(g, st));
    }
    AH_TRY(gemm::run(linear_wgrad(d, dy, h, a.gelu, 4 * h, W + o.w_fc2), st));  // dWfc2 -> slot
    const bool ln_fused = gpt::ln_rows_enabled(h);  // b_fc2 / b_proj grads come out of the LN2 backward
    if (!ln_fused) AH_TRY(gpt::colsum(dy, T, h, h, ws.part, W + o.b_fc2, 0, st));
    // ---- MLP in: fc_pre = ln2 Wfc^T + b_fc
    AH_TRY(gemm::run(linear_dgrad(d, ws.d4h, 4 * h, W + o.w_fc, h, ws.dln), st));
    AH_TRY(gemm::run(linear_wgrad(d, ws.d4h, 4 * h, a.ln2, h, W + o.w_fc), st));
    AH_TRY(gpt::colsum(ws.d4h, T, 4 * h, 4 * h, ws.part, W + o.b_fc, 0, st));
    // ---- LN2 (+ residual path dy)
    if (ln_fused)  // dx2 = LN2'(dln) + dy; dgamma/dbeta; b_fc2 grad = colsum(dy); b_proj grad = colsum(dx2)
        AH_TRY(gpt::ln_bwd_rows(ws.dln, a.x2, a.mean2, a.rstd2, W + o.ln2_g, dy, ws.dx2, W + o.ln2_g, W + o.b_fc2,
                                W + o.b_proj, ws.part, T, h, st));
    else
        AH_TRY(gpt::ln_bwd2(ws.dln, a.x2, a.mean2, a.rstd2, W + o.ln2_g, dy, ws.dx2, W + o.ln2_g, ws.part, T, h, st));
    // ---- attention out-projection: x2 = x_in + att Wproj^T + b_proj
    AH_TRY(gemm::run(linear_dgrad(d, ws.dx2, h, W + o.w_proj, h, ws.datt), st));
    AH_TRY(gemm::run(linear_wgrad(d, ws.dx2, h, a.att, h, W + o.w_proj), st));
    if (!ln_fused) AH_TRY(gpt::colsum(ws.dx2, T, h, h, ws.part, W + o.b_proj, 0, st));
    // ---- attention core, per (head, sequence)
    const bool fused = attention_mode(d) == AttnMode::Flash;
    if (fused) {  // P recomputed from lse; dS^T (-> HBM for dQ), dV, dK
        AH_TRY(gpt::flash_bwd(a.qkv, a.att, ws.datt, a.lse2, ws.S, ws.dS, ws.dqkv, d.B, s, d.nh, hd, scale, st));
    } else {
    {  // dP = dO V^T (fp32, lower tiles)
        GemmArgs g;
        heads(g, d);
        g.M = s; g.N = s; g.K = hd;
        g.A = ws.datt; g.lda = h; g.a_s1 = hd; g.a_s2 = (long long)s * h;
        g.B = a.qkv + 2 * h; g.ldb = 3 * h; g.b_s1 = hd; g.b_s2 = (long long)s * 3 * h;
        g.C = ws.S; g.c_f32 = 1; g.ldc = s; g.c_s1 = (long long)s * s; g.c_s2 = (long long)d.nh * s * s;
        g.causal = gemm::kCausalSkipUpper;
        AH_TRY(gemm::run(g, st));
    }
    AH_TRY(gpt::softmax_bwd2(a.P, ws.S, ws.dS, (long long)d.B * d.nh * s, s, st));
    {  // dV = P^T dO
        GemmArgs g;
        heads(g, d);
        g.M = s; g.N = hd; g.K = s;
        g.A = a.P; g.a_mn_major = 1; g.lda = s; g.a_s1 = (long long)s * s; g.a_s2 = (long long)d.nh * s * s;
        g.B = ws.datt; g.b_mn_major = 1; g.ldb = h; g.b_s1 = hd; g.b_s2 = (long long)s * h;
        g.C = ws.dqkv + 2 * h; g.ldc = 3 * h; g.c_s1 = hd; g.c_s2 = (long long)s * 3 * h;
        g.causal = gemm::kCausalKFromM;
        AH_TRY(gemm::run(g, st));
    }
    }  // unfused dP / softmax backward / dV
    {  // dQ = dS K * scale
        GemmArgs g;
        heads(g, d);
        g.M = s; g.N = hd; g.K = s;
        g.A = ws.dS; g.lda = s; g.a_s1 = (long long)s * s; g.a_s2 = (long long)d.nh * s * s;
        // the flash backward stores dS^T [key][query]: read it as an MN-major A
        g.a_mn_major = fused ? 1 : 0;
        g.B = a.qkv + h; g.b_mn_major = 1; g.ldb = 3 * h; g.b_s1 = hd; g.b_s2 = (long long)s * 3 * h;
        g.C = ws.dqkv; g.ldc = 3 * h; g.c_s1 = hd; g.c_s2 = (long long)s * 3 * h;
        g.alpha = scale;
        g.causal = gemm::kCausalKUptoM;
        AH_TRY(gemm::run(g, st));
    }
    if (!fused) {  // dK = dS^T Q * scale
        GemmArgs g;
        heads(g, d);
        g.M = s; g.N = hd; g.K = s;
        g.A = ws.dS; g.a_mn_major = 1; g.lda = s; g.a_s1 = (long long)s * s; g.a_s2 = (long long)d.nh * s * s;
        g.B = a.qkv; g.b_mn_major = 1; g.ldb = 3 * h; g.b_s1 = hd; g.b_s2 = (long long)s * 3 * h;
        g.C = ws.dqkv + h; g.ldc = 3 * h; g.c_s1 = hd; g.c_s2 = (long long)s * 3 * h;
        g.alpha = scale;
        g.causal = gemm::kCausalKFromM;
        AH_TRY(gemm::run(g, st));
    }
    // ---- qkv projection: qkv = ln1 Wqkv^T + b_qkv
    AH_TRY(gemm::run(linear_dgrad(d, ws.dqkv, 3 * h, W + o.w_qkv, h, ws.dln), st));
    AH_TRY(gemm::run(linear_wgrad(d, ws.dqkv, 3 * h, a.ln1, h, W + o.w_qkv), st));
    AH_TRY(gpt::colsum(ws.dqkv, T, 3 * h, 3 * h, ws.part, W + o.b_qkv, 0, st));
    // ---- LN1 (+ residual path dx2)
    AH_TRY(gpt::ln_bwd2(ws.dln, x_in, a.mean1, a.rstd1, W + o.ln1_g, ws.dx2, dx, W + o.ln1_g, ws.part, T, h, st));
    return cudaSuccess;
}

}  // namespace ah
