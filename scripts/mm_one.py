"""cuBLAS (torch.matmul) on one shape, for ncu comparisons: python scripts/mm_one.py M N K [reps]"""
import sys
import torch
M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    torch.matmul(A, B.t(), out=C)
torch.cuda.synchronize()
