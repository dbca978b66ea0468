"""ctypes binding of the C-ABI in include/autohete.h.

The product path has no fallback: if lib/libautohete.so is missing or fails to load, every
entry point raises. Build it with `python -m paper_2503_01890_b200.build` (or
__graft_entry__.build()).
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_DIR = os.path.join(PKG, "lib")
HEADER = os.path.join(ROOT, "include", "autohete.h")

_lib = None


class NativeError(RuntimeError):
    pass


class AdamHParams(C.Structure):
    _fields_ = [
        ("lr", C.c_float),
        ("beta1", C.c_float),
        ("beta2", C.c_float),
        ("eps", C.c_float),
        ("weight_decay", C.c_float),
        ("step", C.c_int32),
    ]


ABI_VERSION = 5  # include/autohete.h ah_abi_version()


def lib() -> C.CDLL:
    """Load libautohete.so (and its libhetsim_core.so dependency) exactly once."""
    global _lib
    if _lib is None:
        path = os.path.join(LIB_DIR, "libautohete.so")
        if not os.path.exists(path):
            raise NativeError(f"{path} not built; run `python -m paper_2503_01890_b200.build`")
        C.CDLL(os.path.join(LIB_DIR, "libhetsim_core.so"), mode=C.RTLD_GLOBAL)
        lib_ = C.CDLL(path, mode=C.RTLD_GLOBAL)
        _declare(lib_)
        _declare_extra(lib_)
        got = lib_.ah_abi_version()
        if got != ABI_VERSION:  # a stale build would read / write the structs with another layout
            raise NativeError(f"{path}: ABI version {got}, this package expects {ABI_VERSION}; rebuild")
        _lib = lib_
    return _lib


def _declare(L: C.CDLL) -> None:
    vp, sz, i32, f32 = C.c_void_p, C.c_size_t, C.c_int, C.c_float
    sigs = {
        "ah_last_error": ([], C.c_char_p),
        "ah_abi_version": ([], i32),
        "ah_adam_step": ([C.POINTER(AdamHParams), vp, vp, vp, vp, vp, sz, f32, vp, vp, vp], i32),
        "ah_grad_stats": ([vp, sz, f32, vp, vp], i32),
        "ah_cast_f32_bf16": ([vp, vp, sz, vp], i32),
        "ah_cpu_adam": ([C.POINTER(AdamHParams), vp, vp, vp, vp, vp, sz, f32, i32], i32),
        "ah_host_alloc": ([C.POINTER(vp), sz], i32),
        "ah_host_free": ([vp], i32),
        "ah_host_register": ([vp, sz], i32),
        "ah_host_unregister": ([vp], i32),
        "ah_copy_h2d": ([vp, vp, sz, vp], i32),
        "ah_copy_d2h": ([vp, vp, sz, vp], i32),
        "ah_stream_create": ([C.POINTER(vp), i32], i32),
        "ah_stream_destroy": ([vp], i32),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().ah_last_error().decode(errors="replace")
        raise NativeError(f"{what or 'autohete'} failed ({rc}): {msg}")


def declared_symbols(header: str = HEADER) -> list[str]:
    """Every function prototype declared in include/autohete.h."""
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ah_[a-z0-9_]+)\s*\(", text)))


def hparams(lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, step=1) -> AdamHParams:
    return AdamHParams(lr, beta1, beta2, eps, weight_decay, step)


class GemmDesc(C.Structure):
    _fields_ = [
        ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64),
        ("batch1", C.c_int32), ("batch2", C.c_int32),
        ("A", C.c_void_p), ("a_mn_major", C.c_int32), ("lda", C.c_int64), ("a_s1", C.c_int64), ("a_s2", C.c_int64),
        ("B", C.c_void_p), ("b_mn_major", C.c_int32), ("ldb", C.c_int64), ("b_s1", C.c_int64), ("b_s2", C.c_int64),
        ("C", C.c_void_p), ("c_f32", C.c_int32), ("ldc", C.c_int64), ("c_s1", C.c_int64), ("c_s2", C.c_int64),
        ("bias", C.c_void_p), ("bias_f32", C.c_int32),
        ("residual", C.c_void_p), ("ld_res", C.c_int64), ("res_s1", C.c_int64), ("res_s2", C.c_int64),
        ("aux", C.c_void_p), ("ld_aux", C.c_int64), ("aux_s1", C.c_int64), ("aux_s2", C.c_int64),
        ("alpha", C.c_float), ("beta", C.c_float),
        ("epilogue", C.c_int32), ("causal", C.c_int32), ("block_n", C.c_int32),
    ]


EPI_BIAS, EPI_GELU, EPI_RESIDUAL, EPI_AUX, EPI_GELU_BWD = 1, 2, 4, 16, 32
CAUSAL_NONE, CAUSAL_SKIP_UPPER, CAUSAL_K_UPTO_M, CAUSAL_K_FROM_M = 0, 1, 2, 3

_EXTRA_SIGS = {
    "ah_gemm_bf16": ([C.POINTER(GemmDesc), C.c_void_p], C.c_int),
}


def _declare_extra(L):
    for name, (args, res) in _EXTRA_SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


class TrainerConfig(C.Structure):
    _fields_ = [
        ("num_blocks", C.c_int32), ("hidden", C.c_int32), ("heads", C.c_int32), ("seq_len", C.c_int32),
        ("batch", C.c_int32), ("vocab", C.c_int32),
        ("c_hat", C.c_int32), ("p_hat", C.c_int32), ("o_hat", C.c_int32),
        ("prefetch_lookahead", C.POINTER(C.c_int32)),
        ("priority_sched", C.c_int32), ("fine_tune", C.c_int32),
        ("gpu_mem_budget", C.c_int64), ("cpu_mem_budget", C.c_int64),
        ("gpu_flops", C.c_double), ("h2d_bw", C.c_double), ("d2h_bw", C.c_double),
        ("cpu_adam_rate", C.c_double), ("gpu_adam_rate", C.c_double), ("bwd_fwd_ratio", C.c_double),
        ("adam", AdamHParams), ("seed", C.c_uint64), ("cpu_threads", C.c_int32),
        ("dp_rank", C.c_int32), ("dp_size", C.c_int32), ("force_collectives", C.c_int32),
        ("nccl_id", C.c_uint8 * 128),
        ("dp_aware_plan", C.c_int32), ("collective_bw", C.c_double),
        ("loopback_comm", C.c_void_p),
    ]


class TrainerStats(C.Structure):
    _fields_ = [
        ("c_hat", C.c_int32), ("p_hat", C.c_int32), ("o_hat", C.c_int32),
        ("activation_coef", C.c_double), ("m_p", C.c_int64), ("m_gc", C.c_int64),
        ("modeled_peak_bytes", C.c_int64), ("simulated_peak_bytes", C.c_int64),
        ("pool_peak_bytes", C.c_int64), ("static_bytes", C.c_int64), ("sim_steady_s", C.c_double),
        ("lane_busy_ms", C.c_double * 4), ("lane_ops", C.c_int32 * 4),
        ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("kernels_per_iter", C.c_int32),
        ("window_iters", C.c_double), ("compute_busy_ms", C.c_double), ("h2d_busy_ms", C.c_double),
        ("d2h_busy_ms", C.c_double), ("offload_blocked_ms", C.c_double), ("h2d_gbps", C.c_double),
        ("d2h_gbps", C.c_double),
        ("copy_blocked_ms", C.c_double), ("upstream_blocked_ms", C.c_double), ("cpu_busy_ms", C.c_double),
        ("window_ms", C.c_double), ("sim_steady_fifo_s", C.c_double), ("sim_steady_ps_s", C.c_double),
        ("priority_sched", C.c_int32), ("grad_norm", C.c_double), ("nonfinite_grads", C.c_int64),
        ("skipped_updates", C.c_int32), ("sim_lane_busy_ms", C.c_double * 4),
        ("stream_chunks", C.c_int32), ("pool_reserved_bytes", C.c_int64),
        ("compute_enqueue_ms", C.c_double), ("compute_enqueue_max_ms", C.c_double),
        ("buffer_overflows", C.c_int32),
    ]


_EXTRA_SIGS.update({
    "ah_trainer_create": ([C.POINTER(TrainerConfig), C.POINTER(C.c_void_p)], C.c_int),
    "ah_trainer_destroy": ([C.c_void_p], C.c_int),
    "ah_trainer_submit": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32], C.c_int),
    "ah_trainer_drain": ([C.c_void_p, C.POINTER(C.c_float)], C.c_int),
    "ah_trainer_step": ([C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_float)], C.c_int),
    "ah_trainer_stats_get": ([C.c_void_p, C.POINTER(TrainerStats)], C.c_int),
    "ah_trainer_reset_stats": ([C.c_void_p], C.c_int),
    "ah_trainer_schedule": ([C.c_void_p, C.c_char_p, C.c_size_t], C.c_int),
    "ah_trainer_read_master": ([C.c_void_p, C.c_int32, C.c_void_p, C.c_size_t], C.c_int),
    "ah_trainer_master_size": ([C.c_void_p, C.c_int32], C.c_int64),
    "ah_trainer_trace": ([C.c_void_p, C.c_char_p, C.c_size_t], C.c_int),
})


class HwProfile(C.Structure):
    _fields_ = [("t_fwd_s", C.c_double), ("t_bwd_s", C.c_double), ("gpu_flops", C.c_double),
                ("bwd_fwd_ratio", C.c_double), ("h2d_bw", C.c_double), ("d2h_bw", C.c_double),
                ("gpu_adam_rate", C.c_double), ("cpu_adam_rate", C.c_double),
                ("t_block_fwd_s", C.c_double), ("t_block_bwd_s", C.c_double),
                ("t_nonblock_fwd_s", C.c_double), ("t_nonblock_bwd_s", C.c_double)]


class HostProfile(C.Structure):
    _fields_ = [("stream_gbps", C.c_double), ("adam_gbps", C.c_double), ("adam_params_per_s", C.c_double),
                ("threads", C.c_int32)]


class Calibration(C.Structure):
    _fields_ = [("t_fwd_s", C.c_double), ("t_bwd_s", C.c_double), ("t_recompute_s", C.c_double),
                ("t_h2d_s", C.c_double), ("t_d2h_s", C.c_double), ("t_opt_cpu_s", C.c_double),
                ("t_opt_gpu_s", C.c_double), ("sim_steady_s", C.c_double), ("c_hat", C.c_int32),
                ("p_hat", C.c_int32), ("o_hat", C.c_int32), ("sim_steady_replan_s", C.c_double),
                ("sim_steady_other_s", C.c_double), ("gpu_flops", C.c_double), ("bwd_fwd_ratio", C.c_double),
                ("h2d_bw", C.c_double), ("d2h_bw", C.c_double), ("cpu_adam_rate", C.c_double),
                ("gpu_adam_rate", C.c_double)]


_EXTRA_SIGS.update({
    "ah_trainer_calibrate": ([C.c_void_p, C.POINTER(Calibration)], C.c_int),
    "ah_trainer_apply_calibration": ([C.c_void_p, C.c_int32, C.POINTER(C.c_int32)], C.c_int),
    "ah_trainer_set_schedule": ([C.c_void_p, C.c_int32], C.c_int),
    "ah_trainer_memory_csv": ([C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_int64)], C.c_int),
    "ah_profile_host": ([C.c_size_t, C.c_int32, C.POINTER(HostProfile)], C.c_int),
    "ah_trainer_timer": ([C.c_void_p, C.c_int32, C.POINTER(C.c_float)], C.c_int),
    "ah_profile_block": ([C.POINTER(TrainerConfig), C.POINTER(HwProfile)], C.c_int),
    "ah_kernel_launches": ([], C.c_int64),
    "ah_gemm_timing": ([C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)], C.c_int),
})

_EXTRA_SIGS.update({
    "ah_dp_unique_id": ([C.c_void_p], C.c_int),
    "ah_dp_loopback_create": ([C.c_int32, C.POINTER(C.c_void_p)], C.c_int),
    "ah_dp_loopback_destroy": ([C.c_void_p], C.c_int),
    "ah_dp_loopback_call": ([C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
    "ah_dp_shard": ([C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                     C.POINTER(C.c_int64)], C.c_int),
})


_EXTRA_SIGS.update({
    "ah_nccl_comm_create": ([C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)], C.c_int),
    "ah_nccl_comm_destroy": ([C.c_void_p], C.c_int),
    "ah_nccl_reduce_scatter_bf16": ([C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p], C.c_int),
    "ah_nccl_all_gather_bf16": ([C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p], C.c_int),
    "ah_nccl_all_reduce": ([C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p, C.c_void_p], C.c_int),
})


def dp_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().ah_dp_unique_id(buf), "ah_dp_unique_id")
    return bytes(buf)


def dp_shard(n: int, rank: int, size: int) -> tuple[int, int, int]:
    """(offset, valid length, padded shard length) of rank's shard of an n-element block vector."""
    off, ln, sh = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().ah_dp_shard(n, rank, size, C.byref(off), C.byref(ln), C.byref(sh)), "ah_dp_shard")
    return off.value, ln.value, sh.value

_EXTRA_SIGS.update({
    "ah_trainer_save": ([C.c_void_p, C.c_char_p], C.c_int),
    "ah_trainer_load": ([C.c_void_p, C.c_char_p], C.c_int),
})
