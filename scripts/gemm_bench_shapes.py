"""tcgen05 GEMM throughput on a GPT block's shapes (T=8192, h from argv) with the step's fused
epilogues, vs torch/cuBLAS (plain GEMM). python scripts/gemm_bench_shapes.py [h] [iters]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01890_b200.gemm import gemm  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 6144
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
T = 8192
SHAPES = [  # name, M, N, K, a_mn, b_mn, epilogue
    ("qkv_fwd+bias", T, 3 * h, h, 0, 0, "bias"), ("proj_fwd+bias+res", T, h, h, 0, 0, "bias_res"),
    ("fc_fwd+bias+gelu+aux", T, 4 * h, h, 0, 0, "gelu"), ("fc2_fwd+bias+res", T, h, 4 * h, 0, 0, "bias_res"),
    ("fc2_dgrad+gelu_bwd", T, 4 * h, h, 0, 1, "gelu_bwd"), ("fc_dgrad", T, h, 4 * h, 0, 1, ""),
    ("qkv_dgrad", T, h, 3 * h, 0, 1, ""), ("proj_dgrad", T, h, h, 0, 1, ""),
    ("fc_wgrad", 4 * h, h, T, 1, 1, ""), ("fc2_wgrad", h, 4 * h, T, 1, 1, ""), ("qkv_wgrad", 3 * h, h, T, 1, 1, ""),
    ("proj_wgrad", h, h, T, 1, 1, ""),
]


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / iters


for name, M, N, K, a_mn, b_mn, epi in SHAPES:
    A = torch.randn(K, M, device="cuda").bfloat16() if a_mn else torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16() if b_mn else torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    bias = torch.randn(N, device="cuda").bfloat16()
    aux = torch.randn(M, N, device="cuda").bfloat16()
    res = torch.randn(M, N, device="cuda").bfloat16()
    kw = {"bias": dict(bias=bias), "bias_res": dict(bias=bias, residual=res), "gelu": dict(bias=bias, aux=aux, gelu=True),
          "gelu_bwd": dict(aux=aux, gelu_bwd=True), "": {}}[epi]
    out = {"shape": name, "M": M, "N": N, "K": K}
    t = timeit(lambda: gemm(A, B, C, a_mn=bool(a_mn), b_mn=bool(b_mn), **kw))
    out["ours_epi_tflops"] = round(2 * M * N * K / t / 1e12, 1)
    if epi:
        t = timeit(lambda: gemm(A, B, C, a_mn=bool(a_mn), b_mn=bool(b_mn)))
        out["ours_plain_tflops"] = round(2 * M * N * K / t / 1e12, 1)
    At = A.t() if a_mn else A
    Bt = B if b_mn else B.t()
    t = timeit(lambda: torch.matmul(At, Bt, out=C))
    out["cublas_plain_tflops"] = round(2 * M * N * K / t / 1e12, 1)
    print(json.dumps(out), flush=True)
