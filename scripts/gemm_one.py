"""One GEMM shape, for ncu: python scripts/gemm_one.py M N K a_mn b_mn [reps]"""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01890_b200.gemm import gemm  # noqa: E402
M, N, K, a_mn, b_mn = (int(x) for x in sys.argv[1:6])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 5
A = torch.randn(K, M, device="cuda").bfloat16() if a_mn else torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(K, N, device="cuda").bfloat16() if b_mn else torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    gemm(A, B, C, a_mn=bool(a_mn), b_mn=bool(b_mn))
torch.cuda.synchronize()
