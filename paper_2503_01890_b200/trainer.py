"""Public training API: a GPT model trained on B200 under an AutoHete plan.

    tr = Trainer(ModelConfig(...), PlanConfig(...))
    loss = tr.step(tokens, targets)          # synchronous, host int32 arrays
    tr.submit(tokens, targets); tr.drain()   # asynchronous pipelining across iterations

The plan is decided by the drop-in hetsim planner (include/hetsim/planner.hpp, reference
proj/core/src/planner.cpp:37-153) unless a strategy is forced, and executed by the C++
executor (csrc/runtime/executor.cpp) through the C-ABI — no Python on the per-op path.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import json

import numpy as np

from . import _native as N


@dataclasses.dataclass
class ModelConfig:
    num_blocks: int = 24
    hidden: int = 2048
    heads: int = 16
    seq_len: int = 1024
    batch: int = 8
    vocab: int = 50257


@dataclasses.dataclass
class PlanConfig:
    c_hat: int = -1  # any < 0: let the planner decide
    p_hat: int = -1
    o_hat: int = -1
    prefetch_lookahead: list[int] | None = None
    priority_sched: bool = True
    fine_tune: bool = True
    gpu_mem_budget: int = 40 << 30
    cpu_mem_budget: int = 128 << 30
    gpu_flops: float = 1.0e15
    h2d_bw: float = 50e9
    d2h_bw: float = 50e9
    cpu_adam_rate: float = 1.0e9
    gpu_adam_rate: float = 2.0e11
    bwd_fwd_ratio: float = 2.0
    # data parallel: plan with the per-rank sharded model (hetsim::dp::solve) when dp_size > 1
    dp_aware: bool = True
    collective_bw: float = 0.0  # bytes/s of one rank's all-gather / reduce-scatter (0: not modelled)


@dataclasses.dataclass
class AdamConfig:
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01


class Trainer:
    def __init__(self, model: ModelConfig, plan: PlanConfig | None = None, adam: AdamConfig | None = None,
                 seed: int = 1234, cpu_threads: int = 0, dp_rank: int = 0, dp_size: int = 1,
                 nccl_id: bytes | None = None, force_collectives: bool = False, loopback=None):
        """dp_size > 1: data parallel over NCCL; every rank passes the same nccl_id (from
        _native.dp_unique_id() on rank 0) and the same seed / plan."""
        plan = plan or PlanConfig()
        adam = adam or AdamConfig()
        self.model = model
        cfg = N.TrainerConfig()
        for f in dataclasses.fields(model):
            setattr(cfg, f.name, getattr(model, f.name))
        cfg.c_hat, cfg.p_hat, cfg.o_hat = plan.c_hat, plan.p_hat, plan.o_hat
        self._la = None
        if plan.prefetch_lookahead is not None:
            self._la = (C.c_int32 * model.num_blocks)(*plan.prefetch_lookahead)
            cfg.prefetch_lookahead = C.cast(self._la, C.POINTER(C.c_int32))
        cfg.priority_sched = int(plan.priority_sched)
        cfg.fine_tune = int(plan.fine_tune)
        cfg.gpu_mem_budget, cfg.cpu_mem_budget = plan.gpu_mem_budget, plan.cpu_mem_budget
        cfg.gpu_flops, cfg.h2d_bw, cfg.d2h_bw = plan.gpu_flops, plan.h2d_bw, plan.d2h_bw
        cfg.cpu_adam_rate, cfg.gpu_adam_rate = plan.cpu_adam_rate, plan.gpu_adam_rate
        cfg.bwd_fwd_ratio = plan.bwd_fwd_ratio
        cfg.adam = N.AdamHParams(adam.lr, adam.beta1, adam.beta2, adam.eps, adam.weight_decay, 1)
        cfg.seed = seed
        cfg.cpu_threads = cpu_threads
        cfg.dp_rank, cfg.dp_size, cfg.force_collectives = dp_rank, dp_size, int(force_collectives)
        cfg.dp_aware_plan, cfg.collective_bw = int(plan.dp_aware), float(plan.collective_bw)
        if loopback is not None:  # in-process ranks on one GPU (validation of the DP path)
            cfg.loopback_comm = loopback.handle
        elif dp_size > 1 or force_collectives:
            nid = nccl_id if nccl_id is not None else N.dp_unique_id()
            C.memmove(cfg.nccl_id, nid, 128)
        self._h = C.c_void_p()
        N.check(N.lib().ah_trainer_create(C.byref(cfg), C.byref(self._h)), "ah_trainer_create")

    def close(self):
        if self._h:
            N.check(N.lib().ah_trainer_destroy(self._h), "ah_trainer_destroy")
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _ptr(x):
        if hasattr(x, "data_ptr"):
            return x.data_ptr(), bool(x.is_cuda)
        x = np.ascontiguousarray(x, dtype=np.int32)
        return x.ctypes.data, False

    def step(self, tokens, targets) -> float:
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        y = np.ascontiguousarray(targets, dtype=np.int32)
        loss = C.c_float()
        N.check(N.lib().ah_trainer_step(self._h, t.ctypes.data, y.ctypes.data, C.byref(loss)), "ah_trainer_step")
        return loss.value

    def submit(self, tokens, targets) -> None:
        """tokens/targets: host numpy int32, or CUDA int32 tensors (kept alive by the caller)."""
        if hasattr(tokens, "data_ptr"):
            N.check(N.lib().ah_trainer_submit(self._h, tokens.data_ptr(), targets.data_ptr(), int(tokens.is_cuda)),
                    "ah_trainer_submit")
        else:
            t = np.ascontiguousarray(tokens, dtype=np.int32)
            y = np.ascontiguousarray(targets, dtype=np.int32)
            N.check(N.lib().ah_trainer_submit(self._h, t.ctypes.data, y.ctypes.data, 0), "ah_trainer_submit")

    def drain(self) -> float:
        loss = C.c_float()
        N.check(N.lib().ah_trainer_drain(self._h, C.byref(loss)), "ah_trainer_drain")
        return loss.value

    def stats(self) -> dict:
        s = N.TrainerStats()
        N.check(N.lib().ah_trainer_stats_get(self._h, C.byref(s)), "ah_trainer_stats_get")
        out = {f: getattr(s, f) for f, _ in s._fields_}
        out["lane_busy_ms"] = list(s.lane_busy_ms)
        out["lane_ops"] = list(s.lane_ops)
        out["sim_lane_busy_ms"] = list(s.sim_lane_busy_ms)
        return out

    def reset_stats(self) -> None:
        N.check(N.lib().ah_trainer_reset_stats(self._h), "ah_trainer_reset_stats")

    def calibrate(self) -> dict:
        """In-step block durations of the drained window, the running plan's simulated iteration
        with them, and the plan the reference planner would pick with them."""
        out = N.Calibration()
        N.check(N.lib().ah_trainer_calibrate(self._h, C.byref(out)), "ah_trainer_calibrate")
        return {f: getattr(out, f) for f, _ in out._fields_}

    def apply_calibration(self, keep_strategy: bool = False) -> bool:
        """Adopt the last calibrate()'s rates in place if the planner keeps the running plan with
        them (or keep_strategy); False: a different plan, build a new Trainer from the rates."""
        applied = C.c_int32()
        N.check(N.lib().ah_trainer_apply_calibration(self._h, int(keep_strategy), C.byref(applied)),
                "ah_trainer_apply_calibration")
        return bool(applied.value)

    def set_schedule(self, priority: bool) -> None:
        """Priority-based (True) or FIFO (False) per-lane order for the following iterations."""
        N.check(N.lib().ah_trainer_set_schedule(self._h, int(priority)), "ah_trainer_set_schedule")

    def schedule(self) -> list[str]:
        n = N.lib().ah_trainer_schedule(self._h, None, 0)
        buf = C.create_string_buffer(n)
        N.lib().ah_trainer_schedule(self._h, buf, n)
        return buf.value.decode().split()

    def master(self, block: int) -> np.ndarray:
        n = N.lib().ah_trainer_master_size(self._h, block)
        out = np.empty(n, dtype=np.float32)
        N.check(N.lib().ah_trainer_read_master(self._h, block, out.ctypes.data, n), "ah_trainer_read_master")
        return out

    def save(self, path: str) -> None:
        """Optimizer-state checkpoint (plan-independent)."""
        N.check(N.lib().ah_trainer_save(self._h, path.encode()), "ah_trainer_save")

    def load(self, path: str) -> None:
        """Resume from save() into a fresh trainer (any plan, same model / dp layout)."""
        N.check(N.lib().ah_trainer_load(self._h, path.encode()), "ah_trainer_load")

    def memory_csv(self) -> tuple[str, int]:
        """Measured GPU-memory timeline ("time_us,gpu_bytes", the reference's CSV schema) of the
        last drained iterations, and its peak in bytes."""
        peak = C.c_int64()
        n = N.lib().ah_trainer_memory_csv(self._h, None, 0, C.byref(peak))
        if n < 0:
            N.check(n, "ah_trainer_memory_csv")
        buf = C.create_string_buffer(n + 4096)
        N.check(min(0, N.lib().ah_trainer_memory_csv(self._h, buf, len(buf), C.byref(peak))), "ah_trainer_memory_csv")
        return buf.value.decode(), peak.value

    def timer(self, stop: bool) -> float:
        ms = C.c_float()
        N.check(N.lib().ah_trainer_timer(self._h, int(stop), C.byref(ms)), "ah_trainer_timer")
        return ms.value

    def trace(self) -> list:
        n = N.lib().ah_trainer_trace(self._h, None, 0)
        if n < 0:
            N.check(n, "ah_trainer_trace")
        buf = C.create_string_buffer(max(n, 1) + 4096)
        N.check(min(0, N.lib().ah_trainer_trace(self._h, buf, len(buf))), "ah_trainer_trace")
        return json.loads(buf.value.decode())


class LoopbackComm:
    """ah_dp_loopback_create: an in-process communicator for `nranks` Trainers on one GPU."""

    def __init__(self, nranks: int):
        self.handle = C.c_void_p()
        N.check(N.lib().ah_dp_loopback_create(nranks, C.byref(self.handle)), "ah_dp_loopback_create")

    def close(self):
        if self.handle:
            N.lib().ah_dp_loopback_destroy(self.handle)
            self.handle = C.c_void_p()


def profile_hardware(model: ModelConfig, cpu_threads: int = 0) -> dict:
    """Runtime profiler (paper §3.1): measure one block on this GPU/host -> planner rates."""
    cfg = N.TrainerConfig()
    for f in dataclasses.fields(model):
        setattr(cfg, f.name, getattr(model, f.name))
    cfg.adam = N.AdamHParams(1e-4, 0.9, 0.999, 1e-8, 0.01, 1)
    cfg.cpu_threads = cpu_threads
    out = N.HwProfile()
    N.check(N.lib().ah_profile_block(C.byref(cfg), C.byref(out)), "ah_profile_block")
    return {f: getattr(out, f) for f, _ in out._fields_}


def profile_host(n: int = 100_000_000, threads: int = 0) -> dict:
    """Host side of the profiler: the CpuOptim lane's roofline (in-place 28 B/param stream) and
    the host AdamW on the same pinned buffers."""
    out = N.HostProfile()
    N.check(N.lib().ah_profile_host(n, threads, C.byref(out)), "ah_profile_host")
    return {f: getattr(out, f) for f, _ in out._fields_}


def plan_from_profile(prof: dict, gpu_mem_budget: int, cpu_mem_budget: int, **kw) -> PlanConfig:
    return PlanConfig(gpu_mem_budget=gpu_mem_budget, cpu_mem_budget=cpu_mem_budget, gpu_flops=prof["gpu_flops"],
                      h2d_bw=prof["h2d_bw"], d2h_bw=prof["d2h_bw"], cpu_adam_rate=prof["cpu_adam_rate"],
                      gpu_adam_rate=prof["gpu_adam_rate"], bwd_fwd_ratio=prof["bwd_fwd_ratio"], **kw)
