// Host interface of the tcgen05 GEMM (gemm_tcgen05.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ah {
namespace gemm {

enum Epilogue : int {
    kEpiBias = 1,      // + bias[n]
    kEpiGelu = 2,      // tanh-GELU (GPT-2)
    kEpiResidual = 4,  // + residual[m, n] (bf16)
    kEpiAux = 16,      // store the pre-GELU value to aux (bf16)
    kEpiGeluBwd = 32,  // multiply by GELU'(aux[m, n]) (aux = pre-activation, bf16)
};

enum Causal : int {
    kCausalNone = 0,
    kCausalSkipUpper = 1,  // skip tiles strictly above the diagonal (S = QK^T, dP = dO V^T)
    kCausalKUptoM = 2,     // reduce only k < m_tile_end      (P V, dS K)
    kCausalKFromM = 3,     // reduce only k >= m_tile_start   (P^T dO, dS^T Q)
};

// C[z](m,n) = epi(alpha * sum_k A[z](m,k) B[z](n,k) + beta * C[z](m,n)), z = z1 + batch1*z2.
// A K-major: A + m*lda + k; MN-major: A + k*lda + m (same for B with n). Strides in
// elements; bf16 operands; C bf16 or fp32.
struct GemmArgs {
    long long M = 0, N = 0, K = 0;
    int batch1 = 1, batch2 = 1;
    const void* A = nullptr;
    int a_mn_major = 0;
    long long lda = 0, a_s1 = 0, a_s2 = 0;
    const void* B = nullptr;
    int b_mn_major = 0;
    long long ldb = 0, b_s1 = 0, b_s2 = 0;
    void* C = nullptr;
    int c_f32 = 0;
    long long ldc = 0, c_s1 = 0, c_s2 = 0;
    const void* bias = nullptr;
    int bias_f32 = 0;
    const void* residual = nullptr;
    long long ld_res = 0, res_s1 = 0, res_s2 = 0;
    void* aux = nullptr;
    long long ld_aux = 0, aux_s1 = 0, aux_s2 = 0;
    float alpha = 1.f, beta = 0.f;
    int epilogue = 0;
    int causal = 0;
    int block_n = 0;  // 0 = auto
};

cudaError_t run(const GemmArgs& g, cudaStream_t stream, int max_ctas = 0);

}  // namespace gemm
}  // namespace ah

namespace ah {
namespace gemm {
// Live per-launch timing of the GEMM (bench roofline): when enabled, every launch is
// bracketed by CUDA events on its stream; collect() sums durations and executed FLOPs.
void timing_enable(bool on);
void timing_collect(double* total_ms, double* total_flops, long long* launches);
// FLOPs a launch actually executes (causal tile / K-range skipping included).
double executed_flops(const GemmArgs& g);
}  // namespace gemm
}  // namespace ah
