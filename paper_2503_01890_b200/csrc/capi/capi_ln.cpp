// extern "C" test / instrumentation entries for the LayerNorm kernels of the block step.
#include <algorithm>

#include "autohete.h"
#include "../kernels/gpt_kernels.h"
#include "capi_util.h"

extern "C" int ah_layernorm_fwd(const uint16_t* x, const uint16_t* gamma, const uint16_t* beta, uint16_t* y,
                                float* mean, float* rstd, int32_t rows, int32_t h, void* stream) {
    if (rows == 0) return 0;
    if (!x || !gamma || !beta || !y || !mean || !rstd) return ah::set_error(AH_ERR_INVALID, "ah_layernorm_fwd: null argument");
    if (rows < 0 || h <= 0 || h % 8 != 0) return ah::set_error(AH_ERR_INVALID, "ah_layernorm_fwd: needs h % 8 == 0");
    return ah::cuda_status(ah::gpt::ln_fwd(x, gamma, beta, y, mean, rstd, rows, h, static_cast<cudaStream_t>(stream)),
                           "ah_layernorm_fwd");
}

extern "C" size_t ah_layernorm_bwd_workspace(int32_t rows, int32_t h) {
    if (rows <= 0 || h <= 0) return 0;
    const int R = std::max(ah::gpt::ln_bwd_ctas(rows), std::max(ah::gpt::reduce_chunks(rows), 1));
    return (size_t)R * 4 * h * sizeof(float);
}

extern "C" int ah_layernorm_bwd(const uint16_t* dy, const uint16_t* x, const float* mean, const float* rstd,
                                const uint16_t* gamma, const uint16_t* dres, uint16_t* dx, uint16_t* dgamma_dbeta,
                                uint16_t* dres_colsum, uint16_t* dx_colsum, int32_t rows, int32_t h, void* workspace,
                                size_t workspace_bytes, void* stream) {
    if (rows == 0) return 0;
    if (!workspace || workspace_bytes < ah_layernorm_bwd_workspace(rows, h))
        return ah::set_error(AH_ERR_INVALID, "ah_layernorm_bwd: workspace missing or too small");
    if (!dy || !x || !mean || !rstd || !gamma || !dx || !dgamma_dbeta)
        return ah::set_error(AH_ERR_INVALID, "ah_layernorm_bwd: null argument");
    if (rows < 0 || h <= 0 || h % 8 != 0) return ah::set_error(AH_ERR_INVALID, "ah_layernorm_bwd: needs h % 8 == 0");
    const bool extra = dres_colsum || dx_colsum;
    if (extra && !ah::gpt::ln_rows_enabled(h))
        return ah::set_error(AH_ERR_INVALID, "ah_layernorm_bwd: fused bias column sums need h % 256 == 0, h <= 6144");
    if (dres_colsum && !dres) return ah::set_error(AH_ERR_INVALID, "ah_layernorm_bwd: dres_colsum needs dres");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    float* part = static_cast<float*>(workspace);
    const cudaError_t e =
        extra ? ah::gpt::ln_bwd_rows(dy, x, mean, rstd, gamma, dres, dx, dgamma_dbeta, dres_colsum, dx_colsum, part,
                                     rows, h, st)
              : ah::gpt::ln_bwd2(dy, x, mean, rstd, gamma, dres, dx, dgamma_dbeta, part, rows, h, st);
    return ah::cuda_status(e, "ah_layernorm_bwd");
}
