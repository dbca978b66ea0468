"""Python front-end of ah_gemm_bf16 (tcgen05 GEMM) over torch tensors — used by tests and the
profiler; the training step calls the kernel from C++ directly."""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N


def _stream(stream):
    return torch.cuda.current_stream().cuda_stream if stream is None else stream.cuda_stream


def gemm(a, b, c, *, a_mn=False, b_mn=False, alpha=1.0, beta=0.0, bias=None, residual=None, aux=None,
         gelu=False, gelu_bwd=False, causal=0, block_n=0, stream=None):
    """c = epi(alpha * a @ b^T + beta * c) with logical a (M,K), b (N,K) — 2-D or 3-D (batch first).

    a_mn: `a` is given as its (K, M) storage (MN-major); same for b_mn with (K, N).
    """
    batched = a.dim() == 3
    Z = a.shape[0] if batched else 1
    a2 = a if batched else a.unsqueeze(0)
    b2 = b if batched else b.unsqueeze(0)
    c2 = c if batched else c.unsqueeze(0)
    if a_mn:
        K, M = a2.shape[1], a2.shape[2]
    else:
        M, K = a2.shape[1], a2.shape[2]
    Nn = b2.shape[2] if b_mn else b2.shape[1]
    d = N.GemmDesc()
    d.M, d.N, d.K = M, Nn, K
    d.batch1, d.batch2 = Z, 1
    d.A, d.a_mn_major, d.lda, d.a_s1 = a2.data_ptr(), int(a_mn), a2.stride(1), a2.stride(0)
    d.B, d.b_mn_major, d.ldb, d.b_s1 = b2.data_ptr(), int(b_mn), b2.stride(1), b2.stride(0)
    d.C, d.c_f32, d.ldc, d.c_s1 = c2.data_ptr(), int(c2.dtype == torch.float32), c2.stride(1), c2.stride(0)
    epi = 0
    if bias is not None:
        epi |= N.EPI_BIAS
        d.bias, d.bias_f32 = bias.data_ptr(), int(bias.dtype == torch.float32)
    if residual is not None:
        r2 = residual if batched else residual.unsqueeze(0)
        epi |= N.EPI_RESIDUAL
        d.residual, d.ld_res, d.res_s1 = r2.data_ptr(), r2.stride(1), r2.stride(0)
    if aux is not None:
        x2 = aux if batched else aux.unsqueeze(0)
        epi |= N.EPI_AUX
        d.aux, d.ld_aux, d.aux_s1 = x2.data_ptr(), x2.stride(1), x2.stride(0)
    if gelu:
        epi |= N.EPI_GELU
    if gelu_bwd and aux is None:
        raise ValueError("gemm(gelu_bwd=True) needs aux (the pre-activation)")
    if gelu_bwd:  # c = (a @ b^T) * GELU'(aux): aux holds the pre-activation (read, not written)
        epi = (epi & ~N.EPI_AUX) | N.EPI_GELU_BWD
    d.alpha, d.beta, d.epilogue, d.causal, d.block_n = alpha, beta, epi, causal, block_n
    N.check(N.lib().ah_gemm_bf16(C.byref(d), _stream(stream)), "ah_gemm_bf16")
    return c
