"""Python front-end of ah_layernorm_fwd / ah_layernorm_bwd (tests / profiling)."""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N

_P = C.c_void_p


def _ptr(t):
    return None if t is None else t.data_ptr()


def layernorm_fwd(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor):
    """x [rows, h] bf16 CUDA -> (y bf16, mean fp32 [rows], rstd fp32 [rows])."""
    rows, h = x.shape
    for t in (x, gamma, beta):
        if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("layernorm_fwd: x, gamma, beta must be contiguous bf16 CUDA tensors")
    y = torch.empty_like(x)
    mean = torch.empty(rows, dtype=torch.float32, device=x.device)
    rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    fn = N.lib().ah_layernorm_fwd
    fn.argtypes = [_P] * 6 + [C.c_int32, C.c_int32, _P]
    fn.restype = C.c_int
    N.check(fn(x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
               rows, h, torch.cuda.current_stream().cuda_stream), "ah_layernorm_fwd")
    return y, mean, rstd


def layernorm_bwd(dy, x, mean, rstd, gamma, dres=None, bias_sums=False):
    """-> (dx [rows, h], dgamma_dbeta [2h], dres_colsum [h] | None, dx_colsum [h] | None), bf16."""
    rows, h = x.shape
    for t in (dy, x, gamma) + (() if dres is None else (dres,)):
        if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("layernorm_bwd: dy, x, gamma, dres must be contiguous bf16 CUDA tensors")
    if mean.dtype != torch.float32 or rstd.dtype != torch.float32:
        raise ValueError("layernorm_bwd: mean / rstd must be fp32")
    dx = torch.empty_like(x)
    dgdb = torch.empty(2 * h, dtype=torch.bfloat16, device=x.device)
    cr = torch.empty(h, dtype=torch.bfloat16, device=x.device) if bias_sums and dres is not None else None
    cx = torch.empty(h, dtype=torch.bfloat16, device=x.device) if bias_sums else None
    L = N.lib()
    L.ah_layernorm_bwd_workspace.argtypes = [C.c_int32, C.c_int32]
    L.ah_layernorm_bwd_workspace.restype = C.c_size_t
    nbytes = L.ah_layernorm_bwd_workspace(rows, h)
    ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=x.device)
    fn = L.ah_layernorm_bwd
    fn.argtypes = [_P] * 10 + [C.c_int32, C.c_int32, _P, C.c_size_t, _P]
    fn.restype = C.c_int
    N.check(fn(dy.data_ptr(), x.data_ptr(), mean.data_ptr(), rstd.data_ptr(), gamma.data_ptr(), _ptr(dres),
               dx.data_ptr(), dgdb.data_ptr(), _ptr(cr), _ptr(cx), rows, h, ws.data_ptr(), nbytes,
               torch.cuda.current_stream().cuda_stream), "ah_layernorm_bwd")
    return dx, dgdb, cr, cx
