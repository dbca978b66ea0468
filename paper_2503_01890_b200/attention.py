"""Python front-end of ah_attention_fwd (tests / profiling)."""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N


def attention_fwd(qkv: torch.Tensor, heads: int):
    """qkv [B, s, 3h] bf16 CUDA -> (O [B, s, h], P [B, heads, s, s])."""
    B, s, h3 = qkv.shape
    h = h3 // 3
    P = torch.empty(B, heads, s, s, dtype=torch.bfloat16, device=qkv.device)
    O = torch.empty(B, s, h, dtype=torch.bfloat16, device=qkv.device)
    fn = N.lib().ah_attention_fwd
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
    fn.restype = C.c_int
    N.check(fn(qkv.data_ptr(), P.data_ptr(), O.data_ptr(), B, s, heads, h // heads,
               torch.cuda.current_stream().cuda_stream), "ah_attention_fwd")
    return O, P
