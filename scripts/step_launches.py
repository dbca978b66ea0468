"""One training iteration between cudaProfilerStart / Stop, for an ncu launch list of exactly one
step (run under `ncu --profile-from-start off ...`). The plan is forced (no profiling pass), the
rates are the measured ones of profiles/r2 so the per-lane order matches the bench's.

  python scripts/step_launches.py 10b 25,9,15 [warmup]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, GPU_BUDGET_GIB  # noqa: E402
from paper_2503_01890_b200.trainer import ModelConfig, PlanConfig, Trainer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "10b"
c, p, o = (int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "25,9,15").split(","))
warmup = int(sys.argv[3]) if len(sys.argv) > 3 else 3
m = CONFIGS[name]
plan = PlanConfig(c_hat=c, p_hat=p, o_hat=o, fine_tune=False, gpu_mem_budget=GPU_BUDGET_GIB[name] << 30,
                  cpu_mem_budget=150 << 30, gpu_flops=1.11e15, h2d_bw=43.7e9, d2h_bw=35.1e9, cpu_adam_rate=5.58e9,
                  gpu_adam_rate=2.09e11, bwd_fwd_ratio=1.83)
tr = Trainer(ModelConfig(**m), plan, seed=1234, cpu_threads=os.cpu_count() or 8)
T = m["batch"] * m["seq_len"]
rng = np.random.default_rng(1)
tok = torch.from_numpy(rng.integers(0, m["vocab"], size=T, dtype=np.int32)).cuda()
for _ in range(warmup):
    tr.submit(tok, tok)
tr.drain()
torch.cuda.synchronize()
torch.cuda.profiler.start()
tr.submit(tok, tok)
tr.drain()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("one iteration profiled; loss", tr.drain())
tr.close()
