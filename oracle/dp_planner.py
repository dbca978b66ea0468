"""ORACLE / TEST INFRASTRUCTURE — pure-Python restatement of the planner on the per-rank model
of the data-parallel extension (include/hetsim/dp_planner.hpp). Used only by
tests/test_dp_planner.py as the checker.

At dp_size = 1 it is the reference planner itself, restated from
  /root/reference/proj/core/src/workload.cpp:41-115  (block_param_count, activation_sizes,
                                                      estimate_block_times, build_profile)
  /root/reference/proj/core/src/costmodel.cpp:36-82  (Eq.(1)-(5), evaluate)
  /root/reference/proj/core/src/planner.cpp:37-108   (exhaustive scan, (objective, o, p, c) order)
  /root/reference/proj/core/src/config.cpp:162-191   (GiB -> bytes llround, unit scaling)
keeping every double expression's operand order (Python floats are IEEE doubles, no FMA), so
objectives compare bit-identically with the C++ core. For dp_size > 1 the optimizer terms use
the rank's shard: Eq.(1)_N / Eq.(2)_N and shard durations as documented in the header above.
"""
from __future__ import annotations

import math


def llround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def profile(L, h, s, b, V, gpu_tflops, h2d_gbps, d2h_gbps, cpu_mps, gpu_mps, coef=16.0, ratio=2.0):
    mp = 12 * h * h + 13 * h
    m_a_in = b * s * h
    m_a = llround(coef * float(m_a_in))
    rate = gpu_tflops * 1e12
    flops = 2.0 * float(mp) * float(b) * float(s) + 4.0 * float(b) * float(s) * float(s) * float(h)
    fp = flops / rate
    return dict(L=L, m_p=mp, m_a=m_a, m_a_in=m_a_in, m_gc=2 * V * h + 2 * m_a_in, m_cc=0,
                t_fp=fp, t_bp=ratio * fp, t_h2d=2.0 * float(mp) / (h2d_gbps * 1e9),
                t_d2h=2.0 * float(mp) / (d2h_gbps * 1e9), t_opt_cpu=float(mp) / (cpu_mps * 1e6),
                t_opt_gpu=float(mp) / (gpu_mps * 1e6), h2d=h2d_gbps * 1e9, d2h=d2h_gbps * 1e9,
                cpu=cpu_mps * 1e6, gpu=gpu_mps * 1e6)


def shard(mp, n):
    return mp if n <= 1 else ((mp + n - 1) // n + 7) // 8 * 8


def gather(mp, n):
    return mp if n <= 1 else shard(mp, n) * n


def rank_profile(pr, n, coll_bw=0.0):
    if n <= 1:
        return dict(pr)
    r = dict(pr)
    sh = float(shard(pr["m_p"], n))
    r["t_h2d"] = 2.0 * sh / pr["h2d"]
    r["t_d2h"] = 2.0 * sh / pr["d2h"]
    r["t_opt_cpu"] = sh / pr["cpu"]
    r["t_opt_gpu"] = sh / pr["gpu"]
    if coll_bw > 0:
        t = 2.0 * float(gather(pr["m_p"], n)) * (n - 1) / n / coll_bw
        r["t_fp"] = max(r["t_fp"], t)
        r["t_bp"] = max(r["t_bp"], 2.0 * t)
    return r


def peak_gpu(pr, c, p, o, n):
    L = pr["L"]
    return (2 * pr["m_a_in"] * c + 2 * pr["m_a"] * (L - c + 1) + 2 * gather(pr["m_p"], n) * (L - p + 1)
            + 12 * shard(pr["m_p"], n) * (L - o) + pr["m_gc"])


def cpu_bytes(pr, o, n):
    return 14 * shard(pr["m_p"], n) * o + pr["m_cc"]


def objective(r, c, p, o):
    L = r["L"]
    t_fwd = max(r["t_fp"] * L, r["t_h2d"] * o + r["t_fp"])
    v = p if p < c else c
    t_sync = v * max(r["t_h2d"] - r["t_fp"] - r["t_bp"], 0.0) + (p - v) * max(r["t_h2d"] - r["t_bp"], 0.0)
    comp = r["t_bp"] * L + r["t_fp"] * c + r["t_opt_gpu"] * (L - o) + t_sync
    cpu = r["t_bp"] + r["t_d2h"] + r["t_opt_cpu"] * o
    return t_fwd + max(comp, cpu)


def solve(pr, gpu_budget, cpu_budget, n=1, coll_bw=0.0):
    """-> ((c, p, o), objective, feasible_count) or None when infeasible."""
    r = rank_profile(pr, n, coll_bw)
    L = pr["L"]
    best, feas = None, 0
    for o in range(L + 1):
        if cpu_bytes(pr, o, n) > cpu_budget:
            break
        for p in range(o + 1):
            for c in range(L + 1):
                if peak_gpu(pr, c, p, o, n) > gpu_budget:
                    continue
                feas += 1
                key = (objective(r, c, p, o), o, p, c)
                if best is None or key < best:
                    best = key
    if best is None:
        return None
    return (best[3], best[2], best[1]), best[0], feas
