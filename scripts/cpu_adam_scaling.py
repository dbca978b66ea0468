"""Host AdamW (OpKind::CpuOptim) throughput vs thread count on pinned 14 B/param buffers, with
and without a concurrent pinned H2D copy (the 10B regime shares host DRAM with the DMA)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01890_b200 import optim  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000_000
p = torch.empty(n, dtype=torch.float32).pin_memory().normal_(0, 0.02)
m = torch.zeros(n, dtype=torch.float32).pin_memory()
v = torch.zeros(n, dtype=torch.float32).pin_memory()
g = torch.empty(n, dtype=torch.bfloat16).pin_memory().normal_(0, 0.01)
print(open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0], os.cpu_count(), flush=True)
for t in (1, 2, 4, 8, 12, 16):
    optim.cpu_adam(p, m, v, g, g, nthreads=t)
    t0 = time.perf_counter()
    for _ in range(3):
        optim.cpu_adam(p, m, v, g, g, nthreads=t)
    dt = (time.perf_counter() - t0) / 3
    print(json.dumps({"threads": t, "gparams_per_s": n / dt / 1e9, "host_GBps": 28 * n / dt / 1e9}), flush=True)
# with a concurrent H2D stream of a separate pinned buffer
src = torch.empty(4 << 30, dtype=torch.uint8).pin_memory()
dst = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for t in (12, 16):
    with torch.cuda.stream(s):
        for _ in range(6):
            dst.copy_(src, non_blocking=True)
    t0 = time.perf_counter()
    for _ in range(3):
        optim.cpu_adam(p, m, v, g, g, nthreads=t)
    dt = (time.perf_counter() - t0) / 3
    e0 = torch.cuda.Event(enable_timing=True)
    s.synchronize()
    print(json.dumps({"threads": t, "with_h2d": True, "gparams_per_s": n / dt / 1e9}), flush=True)
t0 = time.perf_counter()
dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
print(json.dumps({"h2d_alone_GBps": (4 << 30) / (time.perf_counter() - t0) / 1e9}))
