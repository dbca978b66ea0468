// extern "C" boundary for the tcgen05 GEMM.
#include "autohete.h"
#include "../kernels/gemm.h"
#include "capi_util.h"

extern "C" int ah_gemm_bf16(const ah_gemm_desc* d, void* stream) {
    if (!d || !d->A || !d->B || !d->C) return ah::set_error(AH_ERR_INVALID, "ah_gemm_bf16: null operand");
    ah::gemm::GemmArgs g;
    g.M = d->M; g.N = d->N; g.K = d->K;
    g.batch1 = d->batch1; g.batch2 = d->batch2;
    g.A = d->A; g.a_mn_major = d->a_mn_major; g.lda = d->lda; g.a_s1 = d->a_s1; g.a_s2 = d->a_s2;
    g.B = d->B; g.b_mn_major = d->b_mn_major; g.ldb = d->ldb; g.b_s1 = d->b_s1; g.b_s2 = d->b_s2;
    g.C = d->C; g.c_f32 = d->c_f32; g.ldc = d->ldc; g.c_s1 = d->c_s1; g.c_s2 = d->c_s2;
    g.bias = d->bias; g.bias_f32 = d->bias_f32;
    g.residual = d->residual; g.ld_res = d->ld_res; g.res_s1 = d->res_s1; g.res_s2 = d->res_s2;
    g.aux = d->aux; g.ld_aux = d->ld_aux; g.aux_s1 = d->aux_s1; g.aux_s2 = d->aux_s2;
    g.alpha = d->alpha; g.beta = d->beta; g.epilogue = d->epilogue; g.causal = d->causal;
    g.block_n = d->block_n;
    if ((g.epilogue & AH_EPI_BIAS) && !g.bias) return ah::set_error(AH_ERR_INVALID, "ah_gemm_bf16: bias missing");
    if ((g.epilogue & AH_EPI_RESIDUAL) && !g.residual) return ah::set_error(AH_ERR_INVALID, "ah_gemm_bf16: residual missing");
    if ((g.epilogue & (AH_EPI_AUX | AH_EPI_GELU_BWD)) && !g.aux)
        return ah::set_error(AH_ERR_INVALID, "ah_gemm_bf16: aux missing (AH_EPI_AUX / AH_EPI_GELU_BWD read it)");
    return ah::cuda_status(ah::gemm::run(g, static_cast<cudaStream_t>(stream)), "ah_gemm_bf16");
}

#include "../kernels/kernels.h"

extern "C" int64_t ah_kernel_launches(void) { return ah::kernel_launch_counter().load(); }

extern "C" int ah_gemm_timing(int32_t enable, double* total_ms, double* total_flops, int64_t* launches) {
    if (enable) {
        ah::gemm::timing_collect(nullptr, nullptr, nullptr);  // drop stale records
        ah::gemm::timing_enable(true);
        return AH_OK;
    }
    ah::gemm::timing_enable(false);
    long long n = 0;
    ah::gemm::timing_collect(total_ms, total_flops, &n);
    if (launches) *launches = n;
    return AH_OK;
}
