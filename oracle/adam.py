"""ORACLE / TEST INFRASTRUCTURE — numpy front-end for oracle/_ref/libadam_oracle.so
(C restatement in oracle/adam_oracle.c; see its header for what it follows and why Adam
parity is unpinned by the reference)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_ref", "libadam_oracle.so")
_lib = None


class HParams(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("step", C.c_int32)]


def build() -> str:
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "adam_oracle.c")):
        subprocess.run(["make", "-C", HERE, "adam"], check=True, capture_output=True)
    return SO


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(SO)
        vp, sz = C.c_void_p, C.c_size_t
        _lib.oracle_adam_f32.argtypes = [C.POINTER(HParams), vp, vp, vp, vp, vp, sz, C.c_float]
        _lib.oracle_adam_f32_mt.argtypes = [C.POINTER(HParams), vp, vp, vp, vp, vp, sz, C.c_float, C.c_int]
        _lib.oracle_adam_f64.argtypes = [C.POINTER(HParams), vp, vp, vp, vp, sz, C.c_double]
        _lib.oracle_grad_stats.argtypes = [vp, sz, C.c_float, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        _lib.oracle_cast_f32_bf16.argtypes = [vp, vp, sz]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def adam_f32(p, m, v, g_bits, *, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, step=1,
             inv_scale=1.0, want_bf16=True, nthreads=0):
    """In-place on float32 numpy p/m/v; g_bits is uint16 (bf16 bit patterns). Returns bf16 bits."""
    hp = HParams(lr, beta1, beta2, eps, weight_decay, step)
    out = np.empty(p.shape, np.uint16) if want_bf16 else None
    if nthreads:
        lib().oracle_adam_f32_mt(C.byref(hp), _p(p), _p(m), _p(v), _p(g_bits), _p(out), p.size, inv_scale, nthreads)
    else:
        lib().oracle_adam_f32(C.byref(hp), _p(p), _p(m), _p(v), _p(g_bits), _p(out), p.size, inv_scale)
    return out


def adam_f64(p, m, v, g_bits, *, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, step=1,
             inv_scale=1.0):
    hp = HParams(lr, beta1, beta2, eps, weight_decay, step)
    lib().oracle_adam_f64(C.byref(hp), _p(p), _p(m), _p(v), _p(g_bits), p.size, inv_scale)


def grad_stats(g_bits, inv_scale=1.0):
    s = C.c_double()
    bad = C.c_int64()
    lib().oracle_grad_stats(_p(g_bits), g_bits.size, inv_scale, C.byref(s), C.byref(bad))
    return s.value, bad.value


def cast_bf16(src):
    out = np.empty(src.shape, np.uint16)
    lib().oracle_cast_f32_bf16(_p(src), _p(out), src.size)
    return out


def synth(n, seed=7, scale=1.0, nonfinite=False):
    """SURVEY.md §8(d) synthetic Adam inputs: p~N(0,.02), m~N(0,1e-3), v=N(0,1e-3)^2,
    bf16 g~N(0,1e-2)*scale (+1 inf, 1 nan when nonfinite)."""
    rng = np.random.default_rng(seed)
    p = rng.standard_normal(n, dtype=np.float32) * np.float32(0.02)
    m = rng.standard_normal(n, dtype=np.float32) * np.float32(1e-3)
    v = np.square(rng.standard_normal(n, dtype=np.float32) * np.float32(1e-3))
    g = rng.standard_normal(n, dtype=np.float32) * np.float32(1e-2 * scale)
    if nonfinite and n >= 2:
        idx = rng.choice(n, 2, replace=False)
        g[idx[0]] = np.inf
        g[idx[1]] = np.nan
    g_bits = cast_bf16(g)
    return p, m, v, g_bits


def bf16_bits_to_f32(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32)
