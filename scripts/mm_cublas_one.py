"""One cuBLAS GEMM (torch.matmul) of the same shape, for ncu comparison."""
import sys
import torch
M, N, K = (int(x) for x in sys.argv[1:4])
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    torch.matmul(A, B.t(), out=C)
torch.cuda.synchronize()
