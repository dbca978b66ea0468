// GPT-2 block compute on B200: the work behind OpKind::Forward / Backward / Recompute
// (reference: modelled only as t_fp / t_bp, proj/core/src/workload.cpp:55-67; block shape
// 12h^2+13h params, workload.cpp:41-44). Weights and activations are bf16, reductions fp32.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ah {

struct GptDims {
    int L = 0, h = 0, nh = 0, hd = 0, s = 0, B = 0, V = 0, Vp = 0;
    int T() const { return B * s; }
    size_t m_p() const { return 12ull * h * h + 13ull * h; }
};

// Offsets (elements) into one block's flat parameter / gradient vector. Matrices first, so
// every offset is a multiple of h (16-byte aligned for h % 8 == 0). Weights are [out][in].
struct BlockLayout {
    size_t w_qkv, w_proj, w_fc, w_fc2, b_qkv, b_proj, b_fc, b_fc2, ln1_g, ln1_b, ln2_g, ln2_b, total;
    static BlockLayout make(size_t h) {
        BlockLayout o{};
        size_t at = 0;
        o.w_qkv = at; at += 3 * h * h;
        o.w_proj = at; at += h * h;
        o.w_fc = at; at += 4 * h * h;
        o.w_fc2 = at; at += 4 * h * h;
        o.b_qkv = at; at += 3 * h;
        o.b_proj = at; at += h;
        o.b_fc = at; at += 4 * h;
        o.b_fc2 = at; at += h;
        o.ln1_g = at; at += h;
        o.ln1_b = at; at += h;
        o.ln2_g = at; at += h;
        o.ln2_b = at; at += h;
        o.total = at;
        return o;
    }
};

// Saved activations of one block besides its input (the recomputable "drop" part of
// simulator.cpp:98-102): carved from one allocation.
// Attention implementation, by shape: flash (head_dim 128, s % 128 == 0: O + per-row lse saved,
// P recomputed in the backward) or unfused (GEMM + softmax + GEMM, P saved). It decides what a
// block keeps (P or lse) and the workspace.
enum class AttnMode { Flash, Unfused };
AttnMode attention_mode(const GptDims& d);

struct BlockActs {
    uint16_t *ln1, *qkv, *P, *att, *x2, *ln2, *fc_pre, *gelu;  // P: [B*nh, s, s] (not in flash mode)
    float* lse2 = nullptr;                                      // flash: [B*nh, s] log2-domain lse
    float *mean1, *rstd1, *mean2, *rstd2;
    static size_t bytes(const GptDims& d);
    static BlockActs carve(const GptDims& d, void* base);
};

// Transient per-step scratch shared by all blocks (part of the constant residue m_gc).
struct Workspace {
    float* S = nullptr;        // unfused: [B*nh, s, s] fp32 scores / dP; fused: D = rowsum(dO*O) [B*nh, s]
    uint16_t* dS = nullptr;    // [B*nh, s, s]
    uint16_t* d4h = nullptr;   // [T, 4h]
    uint16_t* dqkv = nullptr;  // [T, 3h]
    uint16_t* dln = nullptr;   // [T, h]
    uint16_t* datt = nullptr;  // [T, h]
    uint16_t* dx2 = nullptr;   // [T, h]
    float* part = nullptr;     // column-reduction partials
    static size_t bytes(const GptDims& d);
    static Workspace carve(const GptDims& d, void* base);
};

// All launches return cudaSuccess or the first error.
cudaError_t block_forward(const GptDims& d, const uint16_t* W, const uint16_t* x_in, uint16_t* x_out,
                          const BlockActs& a, const Workspace& ws, cudaStream_t st);
// W holds the weights on entry and the weight gradients on exit (the paper's gradient
// buffer aliasing, simulator.hpp:145-147): every slot is overwritten only after its last read.
cudaError_t block_backward(const GptDims& d, uint16_t* W, const uint16_t* x_in, const BlockActs& a,
                           const uint16_t* dy, uint16_t* dx, const Workspace& ws, cudaStream_t st);

}  // namespace ah
