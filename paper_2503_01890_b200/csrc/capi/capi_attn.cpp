// extern "C" test / instrumentation entry for the fused attention forward.
#include "autohete.h"
#include "../kernels/gpt_kernels.h"
#include "capi_util.h"

extern "C" int ah_attention_fwd(const uint16_t* qkv, uint16_t* P, uint16_t* O, int32_t batch, int32_t seq_len,
                                int32_t heads, int32_t head_dim, void* stream) {
    if (!qkv || !P || !O) return ah::set_error(AH_ERR_INVALID, "ah_attention_fwd: null argument");
    if (!ah::gpt::attn_fwd_supported(head_dim, seq_len))
        return ah::set_error(AH_ERR_INVALID, "ah_attention_fwd: needs head_dim 128 and seq_len % 128 == 0");
    return ah::cuda_status(ah::gpt::attn_fwd(qkv, P, O, batch, seq_len, heads, head_dim,
                                             1.0f / __builtin_sqrtf((float)head_dim), static_cast<cudaStream_t>(stream)),
                           "ah_attention_fwd");
}
