"""Time the LayerNorm kernels at the bench shape with CUDA events (and under ncu: one launch each)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01890_b200.layernorm import layernorm_bwd, layernorm_fwd  # noqa: E402


def timed(fn, iters=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--h", type=int, default=2048)
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    T, h = a.rows, a.h
    x = torch.randn(T, h, device="cuda").bfloat16()
    g = torch.ones(h, device="cuda").bfloat16()
    b = torch.zeros(h, device="cuda").bfloat16()
    dy = torch.randn(T, h, device="cuda").bfloat16()
    dres = torch.randn(T, h, device="cuda").bfloat16()
    y, mean, rstd = layernorm_fwd(x, g, b)
    mb = T * h * 2 / 1e6
    t_f = timed(lambda: layernorm_fwd(x, g, b), a.iters)
    t_b = timed(lambda: layernorm_bwd(dy, x, mean, rstd, g, dres, bias_sums=h % 256 == 0), a.iters)
    t_b0 = timed(lambda: layernorm_bwd(dy, x, mean, rstd, g, dres, bias_sums=False), a.iters)
    print(json.dumps({"rows": T, "h": h, "fwd_us": t_f, "fwd_GBps": 2 * mb / t_f * 1e3 / 1e3,
                      "bwd_fused_us": t_b, "bwd_fused_GBps": 4 * mb / t_b * 1e3 / 1e3,
                      "bwd_us": t_b0, "bwd_GBps": 4 * mb / t_b0 * 1e3 / 1e3}))
