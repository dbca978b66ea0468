"""ctypes binding of include/hetsim_c.h (the drop-in planner as a C library)."""
from __future__ import annotations

import ctypes as C
import os

from ._native import LIB_DIR, NativeError

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(os.path.join(LIB_DIR, "libhetsim_core.so"))
        _lib.ah_hetsim_last_error.restype = C.c_char_p
        _lib.ah_hetsim_block_param_count.argtypes = [C.c_int64]
        _lib.ah_hetsim_block_param_count.restype = C.c_int64
        _lib.ah_hetsim_plan_json.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
        _lib.ah_hetsim_plan_json.restype = C.c_int64
        _lib.ah_hetsim_plan_dp_json.argtypes = [C.c_char_p, C.c_int32, C.c_double, C.c_char_p, C.c_size_t]
        _lib.ah_hetsim_plan_dp_json.restype = C.c_int64
        _lib.ah_hetsim_simulate_trace.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                  C.c_char_p, C.c_size_t]
        _lib.ah_hetsim_simulate_trace.restype = C.c_int64
    return _lib


def _text(fn, *args) -> str:
    n = fn(*args, None, 0)
    if n < 0:
        raise NativeError(lib().ah_hetsim_last_error().decode())
    buf = C.create_string_buffer(int(n))
    fn(*args, buf, n)
    return buf.value.decode()


def block_param_count(h: int) -> int:
    return lib().ah_hetsim_block_param_count(h)


def plan_json(config_text: str) -> str:
    return _text(lib().ah_hetsim_plan_json, config_text.encode())


def plan_dp_json(config_text: str, dp_size: int, collective_gbps: float = 0.0) -> str:
    """Data-parallel planner extension (hetsim/dp_planner.hpp): per-rank sharded optimizer."""
    return _text(lib().ah_hetsim_plan_dp_json, config_text.encode(), int(dp_size), float(collective_gbps))


def simulate_trace(config_text: str, strategy=(-1, -1, -1), n_iters=2, priority=True) -> str:
    return _text(lib().ah_hetsim_simulate_trace, config_text.encode(), *strategy, n_iters, int(priority))
