"""Sustained (power-capped) GEMM throughput: the GPT-1.3B block's forward + backward GEMM mix run
back to back for ~3 s, ours vs torch/cuBLAS on the same operands; SM clock sampled via NVML."""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01890_b200.gemm import gemm  # noqa: E402

T, h = 8192, 2048
SHAPES = [("qkv_fwd", T, 3 * h, h, 0, 0), ("proj_fwd", T, h, h, 0, 0), ("fc_fwd", T, 4 * h, h, 0, 0),
          ("fc2_fwd", T, h, 4 * h, 0, 0), ("fc2_dgrad", T, 4 * h, h, 0, 1), ("fc_dgrad", T, h, 4 * h, 0, 1),
          ("proj_dgrad", T, h, h, 0, 1), ("qkv_dgrad", T, h, 3 * h, 0, 1), ("fc2_wgrad", h, 4 * h, T, 1, 1),
          ("fc_wgrad", 4 * h, h, T, 1, 1), ("proj_wgrad", h, h, T, 1, 1), ("qkv_wgrad", 3 * h, h, T, 1, 1)]
ops = []
for name, M, N, K, a_mn, b_mn in SHAPES:
    A = torch.randn(K, M, device="cuda").bfloat16() if a_mn else torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16() if b_mn else torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.append((M, N, K, A, B, C, a_mn, b_mn))
flops = sum(2 * M * N * K for M, N, K, *_ in ops)


def ours():
    for M, N, K, A, B, C, a_mn, b_mn in ops:
        gemm(A, B, C, a_mn=bool(a_mn), b_mn=bool(b_mn))


def cublas():
    for M, N, K, A, B, C, a_mn, b_mn in ops:
        torch.matmul(A.t() if a_mn else A, B if b_mn else B.t(), out=C)


def clock_median(stop, out):
    import pynvml as nv
    nv.nvmlInit()
    hd = nv.nvmlDeviceGetHandleByIndex(0)
    while not stop.is_set():
        out.append((nv.nvmlDeviceGetClockInfo(hd, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetPowerUsage(hd) / 1000.0))
        time.sleep(0.05)


which = sys.argv[1] if len(sys.argv) > 1 else "both"
runs = (("ours", ours), ("cublas", cublas)) if which == "both" else (("ours", ours),)
for name, fn in runs:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    reps = 0
    clocks, stop = [], threading.Event()
    th = threading.Thread(target=clock_median, args=(stop, clocks))
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.time()
    while time.time() - t0 < 3.0:
        fn()
        reps += 1
        if reps % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"impl": name, "reps": reps, "tflops": flops * reps / (ms / 1e3) / 1e12,
                      "sm_mhz_median": sorted(c for c, _ in clocks)[len(clocks) // 2] if clocks else None,
                      "power_w_median": sorted(w for _, w in clocks)[len(clocks) // 2] if clocks else None,
                      "tflops_per_mhz": flops * reps / (ms / 1e3) / 1e12 / max(1, sorted(c for c, _ in clocks)[len(clocks) // 2])}),
          flush=True)
