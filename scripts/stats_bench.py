"""grad_stats (overflow / norm pre-pass) HBM throughput at the BASELINE block sizes."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01890_b200 import optim  # noqa: E402

for n in (50_358_272, 453_064_704):
    g = torch.randn(n, device="cuda").bfloat16()
    st = torch.zeros(520, device="cuda")
    for _ in range(3):
        optim.grad_stats(g, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        optim.grad_stats(g, st)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 / 1e3
    print(json.dumps({"params": n, "us": t * 1e6, "GBps": 2 * n / t / 1e9}))
