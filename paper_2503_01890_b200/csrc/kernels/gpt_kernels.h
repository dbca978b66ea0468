// Launchers for the non-GEMM GPT kernels (gpt_kernels.cu). bf16 tensors are uint16_t*.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace ah {
namespace gpt {

cudaError_t embed_fwd(const int* tok, const uint16_t* wte, const uint16_t* wpe, uint16_t* x, int T, int s, int h,
                      cudaStream_t st);
cudaError_t ln_fwd(const uint16_t* x, const uint16_t* g, const uint16_t* b, uint16_t* y, float* mean, float* rstd,
                   int T, int h, cudaStream_t st);
// dgdb: 2h contiguous bf16 = [dgamma | dbeta]; part: >= ln_bwd_ctas(T) * 2h floats.
int ln_bwd_ctas(int T);
cudaError_t ln_bwd(const uint16_t* dy, const uint16_t* x, const float* mean, const float* rstd, const uint16_t* g,
                   const uint16_t* dres, uint16_t* dx, uint16_t* dgdb, float* part, int T, int h, cudaStream_t st);
// Split LayerNorm backward (dx kernel + deterministic dgamma/dbeta column reduction); same
// contract as ln_bwd; part: >= reduce_chunks(T) * 2h floats.
int reduce_chunks(int T);
cudaError_t ln_bwd2(const uint16_t* dy, const uint16_t* x, const float* mean, const float* rstd, const uint16_t* g,
                    const uint16_t* dres, uint16_t* dx, uint16_t* dgdb, float* part, int T, int h, cudaStream_t st);
// Row-parallel LayerNorm (ln_rows.cu): one CTA of h/8 threads per row chunk, rows read once.
// ln_fwd / ln_bwd2 dispatch here when ln_rows_enabled(h) (h % 256 == 0); the warp-per-row kernels
// in gpt_kernels.cu are the fallback for other h.
bool ln_rows_supported(int h);
bool ln_rows_enabled(int h);
cudaError_t ln_fwd_rows(const uint16_t* x, const uint16_t* g, const uint16_t* b, uint16_t* y, float* mean,
                        float* rstd, int T, int h, cudaStream_t st);
// Fused backward: dx (+ dres), dgdb = [dgamma | dbeta], and optionally the bias gradients
// dres_colsum = sum over rows of dres (needs dres) and dx_colsum = sum over rows of bf16(dx).
// part: >= ln_bwd_ctas(T) * 4h floats.
cudaError_t ln_bwd_rows(const uint16_t* dy, const uint16_t* x, const float* mean, const float* rstd,
                        const uint16_t* g, const uint16_t* dres, uint16_t* dx, uint16_t* dgdb, uint16_t* dres_colsum,
                        uint16_t* dx_colsum, float* part, int T, int h, cudaStream_t st);
// Column sums of X[T][N] (row stride ldx) -> out[N] (bf16 or fp32); part: >= colsum_rows(T)*N floats.
int colsum_rows(int T);
cudaError_t colsum(const uint16_t* X, int T, int N, int ldx, float* part, void* out, int out_f32, cudaStream_t st);
cudaError_t softmax_fwd(const float* S, uint16_t* P, long long rows, int s, cudaStream_t st);
cudaError_t softmax_bwd(const uint16_t* P, const float* dP, uint16_t* dS, long long rows, int s, cudaStream_t st);
// D[b][head][q] = rowsum(dO * O) over the head's 128 columns (hd = 128).
cudaError_t attn_rowdot(const uint16_t* dO, const uint16_t* O, float* D, int B, int s, int nh, cudaStream_t st);
// Flash attention (attn_flash.cu): single-pass online softmax forward that keeps only O and the
// per-row log2-domain log-sum-exp lse2 = max * scale * log2(e) + log2(sum) ([B][nh][s] fp32);
// the backward recomputes P = 2^(S * scale * log2(e) - lse2) from Q, K and lse2, and emits dS
// [B, nh, s, s] (for the dQ = dS K GEMM) and dK (x scale), dV into dqkv. D: B*nh*s scratch.
bool flash_supported(int hd, int s);
cudaError_t flash_fwd(const uint16_t* qkv, uint16_t* O, float* lse2, int B, int s, int nh, int hd, float scale,
                      cudaStream_t st);
// The backward writes dS TRANSPOSED, dS^T [B, nh, s(key), s(query)]: the dQ GEMM reads it as an
// MN-major A operand.
cudaError_t flash_bwd(const uint16_t* qkv, const uint16_t* O, const uint16_t* dO, const float* lse2, float* D,
                      uint16_t* dS, uint16_t* dqkv, int B, int s, int nh, int hd, float scale, cudaStream_t st);
// Register-resident single-read versions (attn_softmax.cu); fall back to the above for s > 2048.
cudaError_t softmax_fwd2(const float* S, uint16_t* P, long long rows, int s, cudaStream_t st);
cudaError_t softmax_bwd2(const uint16_t* P, const float* dP, uint16_t* dS, long long rows, int s, cudaStream_t st);
cudaError_t colsum_finish_wide(const float* part, int R, int N, void* out, int out_f32, cudaStream_t st);
cudaError_t gelu_bwd(const uint16_t* dgelu, const uint16_t* pre, uint16_t* dpre, size_t n, cudaStream_t st);
cudaError_t cross_entropy(uint16_t* logits, const int* tgt, float* loss, int T, int V, int ld, float dscale,
                          cudaStream_t st);
cudaError_t embed_bwd_tok(const uint16_t* dx, const int* uniq, const int* offs, const int* pos, int n_uniq,
                          float* dwte, int h, cudaStream_t st);
cudaError_t embed_bwd_pos(const uint16_t* dx, float* dwpe, int B, int s, int h, cudaStream_t st);
cudaError_t f32_to_bf16(const float* src, uint16_t* dst, size_t n, cudaStream_t st);
cudaError_t mean_loss(const float* loss, int T, float* out, cudaStream_t st);

}  // namespace gpt
}  // namespace ah

namespace ah {
namespace gpt {
// Deterministic counter-based init: p[i] = mean + std * N(0,1)(seed, i).
cudaError_t init_normal(float* p, size_t n, unsigned long long seed, float mean, float std, cudaStream_t st);
cudaError_t fill_f32(float* p, size_t n, float v, cudaStream_t st);
}  // namespace gpt
}  // namespace ah

namespace ah {
namespace gpt {
// Deterministic token -> positions index for the embedding backward, built on device:
// sorts (token, position) pairs (single CTA bitonic sort, T <= 16384) and emits
// uniq[n_uniq], offs[n_uniq + 1], pos[T] and *n_uniq. Buffers: ints of T, T+1, T, 1.
cudaError_t token_index(const int* tok, int T, int* uniq, int* offs, int* pos, int* n_uniq, cudaStream_t st);
// ids in [0, V) are kept; any other id is replaced by 0 and sets *flag (device int) to 1.
cudaError_t sanitize_ids(int* ids, int n, int V, int* flag, cudaStream_t st);
// embedding scatter using the device-side count (grid = T, CTAs beyond n_uniq exit)
cudaError_t embed_bwd_tok_dev(const uint16_t* dx, const int* uniq, const int* offs, const int* pos,
                              const int* n_uniq, int T, float* dwte, int h, cudaStream_t st);
}  // namespace gpt
}  // namespace ah
