"""Attention kernels at the GPT-1.3B shape (B=8, s=1024, 16 heads), for ncu / timing.
python scripts/attn_one.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01890_b200.attention import flash_bwd, flash_fwd  # noqa: E402

B, s, nh, hd = 8, 1024, 16, 128
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
qkv = (torch.randn(B, s, 3 * nh * hd, device="cuda") * 0.5).bfloat16()
dO = torch.randn(B, s, nh * hd, device="cuda").bfloat16()


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


O, lse = flash_fwd(qkv, nh)
print(f"flash_fwd {timed(lambda: flash_fwd(qkv, nh)):.1f} us")
print(f"flash_bwd (+dQ GEMM) {timed(lambda: flash_bwd(qkv, O, dO, lse, nh)):.1f} us")
