"""Python front-end of the flash attention C-ABI entries (tests / profiling)."""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N


def flash_fwd(qkv: torch.Tensor, heads: int):
    """qkv [B, s, 3h] bf16 CUDA -> (O [B, s, h] bf16, lse2 [B, heads, s] fp32)."""
    B, s, h3 = qkv.shape
    h = h3 // 3
    O = torch.empty(B, s, h, dtype=torch.bfloat16, device=qkv.device)
    lse2 = torch.empty(B, heads, s, dtype=torch.float32, device=qkv.device)
    fn = N.lib().ah_attention_flash_fwd
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
    fn.restype = C.c_int
    N.check(fn(qkv.data_ptr(), O.data_ptr(), lse2.data_ptr(), B, s, heads, h // heads,
               torch.cuda.current_stream().cuda_stream), "ah_attention_flash_fwd")
    return O, lse2


def flash_bwd(qkv: torch.Tensor, O: torch.Tensor, dO: torch.Tensor, lse2: torch.Tensor, heads: int):
    """-> dqkv [B, s, 3h] bf16 (dQ | dK | dV)."""
    B, s, h3 = qkv.shape
    h = h3 // 3
    dqkv = torch.empty_like(qkv)
    L = N.lib()
    L.ah_attention_flash_bwd_workspace.argtypes = [C.c_int32] * 3
    L.ah_attention_flash_bwd_workspace.restype = C.c_size_t
    nbytes = L.ah_attention_flash_bwd_workspace(B, s, heads)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=qkv.device)
    fn = L.ah_attention_flash_bwd
    fn.argtypes = [C.c_void_p] * 5 + [C.c_int32] * 4 + [C.c_void_p, C.c_size_t, C.c_void_p]
    fn.restype = C.c_int
    N.check(fn(qkv.data_ptr(), O.data_ptr(), dO.data_ptr(), lse2.data_ptr(), dqkv.data_ptr(), B, s, heads,
               h // heads, ws.data_ptr(), nbytes, torch.cuda.current_stream().cuda_stream), "ah_attention_flash_bwd")
    return dqkv
