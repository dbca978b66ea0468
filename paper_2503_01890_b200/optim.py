"""Host-side mirror of the optimizer ops the reference schedules
(OpKind::GpuOptim / OpKind::CpuOptim, /root/reference/proj/core/src/simulator.cpp:210-226).

Thin wrappers over the C-ABI taking torch tensors (torch is plumbing here: device memory and
streams). No CPU fallback for the GPU op: a missing extension raises NativeError.
"""
from __future__ import annotations

import ctypes as C

import torch

from ._native import check, hparams, lib

__all__ = ["adam_step", "cpu_adam", "grad_stats", "cast_f32_bf16", "hparams"]


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def adam_step(p, m, v, g, p_bf16=None, *, hp=None, inv_scale=1.0, skip_flag=None, stats=None,
              stream=None) -> None:
    """Fused AdamW (sm_100a) on fp32 p/m/v with bf16 grads g (all CUDA tensors)."""
    assert p.is_cuda and p.dtype == torch.float32 and g.dtype == torch.bfloat16
    hp = hp or hparams()
    check(lib().ah_adam_step(C.byref(hp), _ptr(p), _ptr(m), _ptr(v), _ptr(g), _ptr(p_bf16), p.numel(),
                             float(inv_scale), _ptr(skip_flag), _ptr(stats), _stream(stream)),
          "ah_adam_step")


def grad_stats(g, stats, inv_scale=1.0, stream=None) -> None:
    check(lib().ah_grad_stats(_ptr(g), g.numel(), float(inv_scale), _ptr(stats), _stream(stream)),
          "ah_grad_stats")


def cast_f32_bf16(src, dst, stream=None) -> None:
    check(lib().ah_cast_f32_bf16(_ptr(src), _ptr(dst), src.numel(), _stream(stream)), "ah_cast_f32_bf16")


def cpu_adam(p, m, v, g, p_bf16=None, *, hp=None, inv_scale=1.0, nthreads=0) -> None:
    """Host AdamW over fp32 p/m/v + bf16 g (CPU tensors; g and p_bf16 may alias)."""
    assert not p.is_cuda and p.dtype == torch.float32 and g.dtype == torch.bfloat16
    hp = hp or hparams()
    check(lib().ah_cpu_adam(C.byref(hp), _ptr(p), _ptr(m), _ptr(v), _ptr(g), _ptr(p_bf16), p.numel(),
                            float(inv_scale), int(nthreads)), "ah_cpu_adam")
