// extern "C" entries of the flash attention kernels (tests / profiling; the executor calls them
// from C++ inside block_forward / block_backward).
#include "autohete.h"
#include "../kernels/gemm.h"
#include "../kernels/gpt_kernels.h"
#include <cmath>
#include <cstdint>
#include "capi_util.h"

extern "C" int ah_attention_flash_fwd(const uint16_t* qkv, uint16_t* O, float* lse2, int32_t batch, int32_t seq_len,
                                      int32_t heads, int32_t head_dim, void* stream) {
    if (!qkv || !O || !lse2) return ah::set_error(AH_ERR_INVALID, "ah_attention_flash_fwd: null argument");
    if (!ah::gpt::flash_supported(head_dim, seq_len))
        return ah::set_error(AH_ERR_INVALID, "ah_attention_flash_fwd: needs head_dim 128 and seq_len % 128 == 0");
    return ah::cuda_status(ah::gpt::flash_fwd(qkv, O, lse2, batch, seq_len, heads, head_dim,
                                              1.0f / std::sqrt((float)head_dim), static_cast<cudaStream_t>(stream)),
                           "ah_attention_flash_fwd");
}

// scratch: D = rowsum(dO * O) [B*heads*s] fp32, then dS^T [B*heads, s, s] bf16 (16-byte aligned)
extern "C" size_t ah_attention_flash_bwd_workspace(int32_t batch, int32_t seq_len, int32_t heads) {
    const size_t rows = (size_t)batch * heads * seq_len;
    return (rows * 4 + 255) / 256 * 256 + rows * (size_t)seq_len * 2;
}

extern "C" int ah_attention_flash_bwd(const uint16_t* qkv, const uint16_t* O, const uint16_t* dO, const float* lse2,
                                      uint16_t* dqkv, int32_t batch, int32_t seq_len, int32_t heads, int32_t head_dim,
                                      void* workspace, size_t workspace_bytes, void* stream) {
    if (!qkv || !O || !dO || !lse2 || !dqkv || !workspace)
        return ah::set_error(AH_ERR_INVALID, "ah_attention_flash_bwd: null argument");
    if (!ah::gpt::flash_supported(head_dim, seq_len))
        return ah::set_error(AH_ERR_INVALID, "ah_attention_flash_bwd: needs head_dim 128 and seq_len % 128 == 0");
    if (workspace_bytes < ah_attention_flash_bwd_workspace(batch, seq_len, heads) ||
        (reinterpret_cast<uintptr_t>(workspace) & 15u))
        return ah::set_error(AH_ERR_INVALID, "ah_attention_flash_bwd: workspace too small or not 16-byte aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long s = seq_len, h = (long long)heads * head_dim, rows = (long long)batch * heads * s;
    const float scale = 1.0f / std::sqrt((float)head_dim);
    float* D = static_cast<float*>(workspace);
    uint16_t* dS = reinterpret_cast<uint16_t*>(static_cast<char*>(workspace) + ((size_t)rows * 4 + 255) / 256 * 256);
    cudaError_t e = ah::gpt::flash_bwd(qkv, O, dO, lse2, D, dS, dqkv, batch, seq_len, heads, head_dim, scale, st);
    if (e == cudaSuccess) {  // dQ = dS K * scale (causal: K range up to the query tile)
        ah::gemm::GemmArgs g;
        g.batch1 = heads;
        g.batch2 = batch;
        g.M = s; g.N = head_dim; g.K = s;
        g.A = dS; g.lda = s; g.a_s1 = s * s; g.a_s2 = (long long)heads * s * s;
        g.a_mn_major = 1;  // dS^T [key][query]
        g.B = qkv + h; g.b_mn_major = 1; g.ldb = 3 * h; g.b_s1 = head_dim; g.b_s2 = s * 3 * h;
        g.C = dqkv; g.ldc = 3 * h; g.c_s1 = head_dim; g.c_s2 = s * 3 * h;
        g.alpha = scale;
        g.causal = ah::gemm::kCausalKUptoM;
        e = ah::gemm::run(g, st);
    }
    return ah::cuda_status(e, "ah_attention_flash_bwd");
}
