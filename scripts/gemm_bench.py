"""tcgen05 GEMM throughput on the GPT-1.3B block shapes (T=8192, h=2048) vs torch/cuBLAS."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01890_b200.gemm import gemm  # noqa: E402

T, h = 8192, 2048
SHAPES = [  # name, M, N, K, a_mn, b_mn
    ("qkv_fwd", T, 3 * h, h, 0, 0), ("proj_fwd", T, h, h, 0, 0), ("fc_fwd", T, 4 * h, h, 0, 0),
    ("fc2_fwd", T, h, 4 * h, 0, 0),
    ("fc2_dgrad", T, 4 * h, h, 0, 1), ("fc_wgrad", 4 * h, h, T, 1, 1), ("qkv_wgrad", 3 * h, h, T, 1, 1),
]


def timeit(fn, iters=20):
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


for name, M, N, K, a_mn, b_mn in SHAPES:
    A = torch.randn(K, M, device="cuda").bfloat16() if a_mn else torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16() if b_mn else torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    res = {}
    for bn in (128, 256):
        t = timeit(lambda: gemm(A, B, C, a_mn=bool(a_mn), b_mn=bool(b_mn), block_n=bn))
        res[f"ours_bn{bn}_tflops"] = round(2 * M * N * K / t / 1e12, 1)
    At = A.t() if a_mn else A
    Bt = B if b_mn else B.t()
    t = timeit(lambda: torch.matmul(At, Bt, out=C))
    res["cublas_tflops"] = round(2 * M * N * K / t / 1e12, 1)
    print(json.dumps({"shape": name, "M": M, "N": N, "K": K, **res}), flush=True)

# attention-shaped batched GEMMs (b=8, heads=16, s=1024, hd=128) as the block step issues them
import ctypes as C  # noqa: E402
from paper_2503_01890_b200 import _native as NN  # noqa: E402
b, nh, s, hd = 8, 16, 1024, 128
h = nh * hd
qkv = torch.randn(b, s, 3 * h, device="cuda").bfloat16()
S = torch.empty(b, nh, s, s, device="cuda", dtype=torch.float32)
P = torch.randn(b, nh, s, s, device="cuda").bfloat16()
att = torch.empty(b, s, h, device="cuda").bfloat16()


def desc_S():
    d = NN.GemmDesc()
    d.M, d.N, d.K, d.batch1, d.batch2 = s, s, hd, nh, b
    d.A, d.lda, d.a_s1, d.a_s2 = qkv.data_ptr(), 3 * h, hd, s * 3 * h
    d.B, d.ldb, d.b_s1, d.b_s2 = qkv.data_ptr() + 2 * h, 3 * h, hd, s * 3 * h
    d.C, d.c_f32, d.ldc, d.c_s1, d.c_s2 = S.data_ptr(), 1, s, s * s, nh * s * s
    d.alpha, d.causal = 0.088, 1
    return d


def desc_PV():
    d = NN.GemmDesc()
    d.M, d.N, d.K, d.batch1, d.batch2 = s, hd, s, nh, b
    d.A, d.lda, d.a_s1, d.a_s2 = P.data_ptr(), s, s * s, nh * s * s
    d.B, d.b_mn_major, d.ldb, d.b_s1, d.b_s2 = qkv.data_ptr() + 4 * h, 1, 3 * h, hd, s * 3 * h
    d.C, d.ldc, d.c_s1, d.c_s2 = att.data_ptr(), h, hd, s * h
    d.alpha, d.causal = 1.0, 2
    return d


for name, dsc, useful in (("attn_S_fp32_causal", desc_S(), b * nh * s * s * hd), ("attn_PV_causal", desc_PV(), b * nh * s * s * hd)):
    st = torch.cuda.current_stream().cuda_stream
    t = timeit(lambda: NN.check(NN.lib().ah_gemm_bf16(C.byref(dsc), st)))
    print(json.dumps({"shape": name, "us": round(t * 1e6, 1), "useful_tflops": round(useful / t / 1e12, 1)}), flush=True)
