"""Diagnose the pipelined (submit without drain) timing: repeat {K device-resident submits}
trials and print, per trial, ms/step and the largest idle gaps on the compute lane."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv += []
from paper_2503_01890_b200.trainer import ModelConfig, Trainer, plan_from_profile, profile_hardware  # noqa: E402

m = dict(num_blocks=24, hidden=2048, heads=16, seq_len=1024, batch=8, vocab=50257)
threads = max(1, (os.cpu_count() or 8) - 4)
model = ModelConfig(**m)
prof = profile_hardware(model, cpu_threads=threads)
plan = plan_from_profile(prof, 32 << 30, 150 << 30)
tr = Trainer(model, plan, seed=1234, cpu_threads=threads)
T = m["batch"] * m["seq_len"]
rng = np.random.default_rng(1)
tok = [torch.from_numpy(rng.integers(0, m["vocab"], size=T, dtype=np.int32)).cuda() for _ in range(4)]
for i in range(3):
    tr.submit(tok[i % 4], tok[(i + 1) % 4])
tr.drain()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
mode = sys.argv[2] if len(sys.argv) > 2 else "none"
import contextlib  # noqa: E402
from bench import ClockSampler  # noqa: E402
for trial in range(10):
    ctx = ClockSampler(0) if mode in ("nvml", "all") else contextlib.nullcontext()
    if mode == "smi":
        ctx = ClockSampler(0)
        ctx._open_nvml = lambda: None
    import ctypes as C
    from paper_2503_01890_b200 import _native as N
    if mode in ("gemm", "all"):
        N.check(N.lib().ah_gemm_timing(1, None, None, None))
    with ctx:
        tr.timer(False)
        for i in range(K):
            tr.submit(tok[i % 4], tok[(i + 1) % 4])
        ms = tr.timer(True)
    if mode in ("gemm", "all"):
        g_ms, g_fl, g_n = C.c_double(), C.c_double(), C.c_int64()
        N.check(N.lib().ah_gemm_timing(0, C.byref(g_ms), C.byref(g_fl), C.byref(g_n)))
    tr_ops = tr.trace()
    comp = sorted([o for o in tr_ops if o["tid"] == 1], key=lambda o: o["ts"])
    gaps = []
    for a, b in zip(comp, comp[1:]):
        gaps.append((b["ts"] - (a["ts"] + a["dur"]), a["name"], b["name"], b["ts"]))
    gaps.sort(reverse=True)
    print(json.dumps({"trial": trial, "ms_per_step": ms / K, "top_gaps_us": gaps[:6]}), flush=True)
tr.close()
