"""Fused-Adam HBM sweep (config C5): params/s and GB/s at 28 B/param for
N in {10M, 32M, 100M, 316M, 1B, 2B}; CUDA events on the launch stream, inputs >> L2."""
import argparse
import json
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01890_b200 import optim  # noqa: E402


def measure(n, iters=20, warmup=3, bf16_out=True):
    p = torch.randn(n, device="cuda") * 0.02
    m = torch.randn(n, device="cuda") * 1e-3
    v = (torch.randn(n, device="cuda") * 1e-3) ** 2
    g = (torch.randn(n, device="cuda") * 1e-2).to(torch.bfloat16)
    out = torch.empty(n, dtype=torch.bfloat16, device="cuda") if bf16_out else None
    hp = optim.hparams(step=10)
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        optim.adam_step(p, m, v, g, out, hp=hp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(iters):
        optim.adam_step(p, m, v, g, out, hp=hp)
    e1.record(s)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / iters
    bpp = 28 if bf16_out else 26
    del p, m, v, g, out
    torch.cuda.empty_cache()
    return {"n": n, "s": t, "params_per_s": n / t, "GBps": n * bpp / t / 1e9}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="10000000,31600000,100000000,316000000,1000000000,2000000000")
    a = ap.parse_args()
    for n in [int(x) for x in a.sizes.split(",")]:
        print(json.dumps(measure(n)), flush=True)
