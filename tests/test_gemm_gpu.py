"""GPU numerics of the tcgen05 GEMM against a plain torch fp32 reference of the same op
(tolerance: bf16 inputs, fp32 accumulation => rel. Frobenius error <= 1e-2 after bf16 output
rounding; fp32 output <= 2e-3)."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def rel_err(x, ref):
    return (x.float() - ref).norm().item() / max(ref.norm().item(), 1e-30)


def operands(M, N, K, a_mn, b_mn, Z=None, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    shp = (lambda r, c: (Z, r, c)) if Z else (lambda r, c: (r, c))
    A = torch.randn(*shp(M, K), device="cuda", generator=g).bfloat16()
    B = torch.randn(*shp(N, K), device="cuda", generator=g).bfloat16()
    a_arg = A.transpose(-1, -2).contiguous() if a_mn else A
    b_arg = B.transpose(-1, -2).contiguous() if b_mn else B
    return A, B, a_arg, b_arg


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 1024), (200, 300, 136), (1024, 768, 2048)])
def test_gemm_layouts(cuda_device, native, a_mn, b_mn, M, N, K):
    from paper_2503_01890_b200.gemm import gemm
    if (a_mn and M % 8) or (b_mn and N % 8):
        pytest.skip("MN-major operands need 16-byte row strides")
    A, B, a_arg, b_arg = operands(M, N, K, a_mn, b_mn)
    ref = A.float() @ B.float().T
    for out_dtype, tol in ((torch.bfloat16, 1e-2), (torch.float32, 2e-3)):
        C = torch.full((M, N), float("nan"), device="cuda", dtype=out_dtype)
        gemm(a_arg, b_arg, C, a_mn=bool(a_mn), b_mn=bool(b_mn))
        torch.cuda.synchronize()
        assert rel_err(C, ref) < tol, (out_dtype, rel_err(C, ref))


@pytest.mark.parametrize("block_n", [64, 128, 256])
def test_gemm_block_n(cuda_device, native, block_n):
    from paper_2503_01890_b200.gemm import gemm
    A, B, a_arg, b_arg = operands(384, 512, 512, 0, 0)
    C = torch.empty(384, 512, device="cuda", dtype=torch.float32)
    gemm(a_arg, b_arg, C, block_n=block_n)
    torch.cuda.synchronize()
    assert rel_err(C, A.float() @ B.float().T) < 2e-3


def test_gemm_epilogues(cuda_device, native):
    from paper_2503_01890_b200.gemm import gemm
    M, N, K = 512, 1024, 768
    A, B, a_arg, b_arg = operands(M, N, K, 0, 0, seed=3)
    bias = torch.randn(N, device="cuda").bfloat16()
    res = torch.randn(M, N, device="cuda").bfloat16()
    pre = A.float() @ B.float().T * 0.5 + bias.float()
    # bias + gelu with pre-activation aux
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    aux = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    gemm(a_arg, b_arg, C, alpha=0.5, bias=bias, gelu=True, aux=aux)
    torch.cuda.synchronize()
    assert rel_err(aux, pre) < 1e-2
    assert rel_err(C, torch.nn.functional.gelu(pre, approximate="tanh")) < 1e-2
    # bias + residual
    C2 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    gemm(a_arg, b_arg, C2, alpha=0.5, bias=bias, residual=res)
    torch.cuda.synchronize()
    assert rel_err(C2, pre + res.float()) < 1e-2
    # beta accumulation into fp32
    C3 = torch.randn(M, N, device="cuda")
    ref3 = A.float() @ B.float().T + 0.75 * C3
    gemm(a_arg, b_arg, C3, beta=0.75)
    torch.cuda.synchronize()
    assert rel_err(C3, ref3) < 2e-3


def test_gemm_batched_strided_heads(cuda_device, native):
    """Attention-style operands: Q/K heads sliced out of a [b, s, 3h] qkv buffer."""
    from paper_2503_01890_b200 import _native as N
    import ctypes as C
    b, s, nh, hd = 2, 256, 4, 128
    h = nh * hd
    qkv = torch.randn(b, s, 3 * h, device="cuda").bfloat16()
    S = torch.empty(b, nh, s, s, device="cuda", dtype=torch.float32)
    d = N.GemmDesc()
    d.M, d.N, d.K = s, s, hd
    d.batch1, d.batch2 = nh, b
    d.A, d.lda, d.a_s1, d.a_s2 = qkv.data_ptr(), 3 * h, hd, s * 3 * h
    d.B, d.ldb, d.b_s1, d.b_s2 = qkv.data_ptr() + 2 * h, 3 * h, hd, s * 3 * h  # K slice (+h elems)
    d.C, d.c_f32, d.ldc, d.c_s1, d.c_s2 = S.data_ptr(), 1, s, s * s, nh * s * s
    d.alpha = 1.0 / math.sqrt(hd)
    N.check(N.lib().ah_gemm_bf16(C.byref(d), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    q = qkv[..., :h].view(b, s, nh, hd).transpose(1, 2).float()
    k = qkv[..., h:2 * h].view(b, s, nh, hd).transpose(1, 2).float()
    ref = q @ k.transpose(-1, -2) / math.sqrt(hd)
    assert rel_err(S, ref) < 2e-3


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_gemm_causal_modes(cuda_device, native, mode):
    from paper_2503_01890_b200.gemm import gemm
    S = 512
    g = torch.Generator(device="cuda").manual_seed(mode)
    if mode == 1:  # skip upper tiles of S = Q K^T: compare lower triangle only
        Q = torch.randn(2, S, 128, device="cuda", generator=g).bfloat16()
        K = torch.randn(2, S, 128, device="cuda", generator=g).bfloat16()
        out = torch.zeros(2, S, S, device="cuda")
        gemm(Q, K, out, causal=1)
        torch.cuda.synchronize()
        ref = Q.float() @ K.float().transpose(-1, -2)
        mask = torch.ones(S, S, device="cuda").tril().bool()
        assert rel_err(out[:, mask], ref[:, mask]) < 2e-3
    else:
        P = torch.randn(2, S, S, device="cuda", generator=g).tril().bfloat16()  # zero above diagonal
        V = torch.randn(2, S, 128, device="cuda", generator=g).bfloat16()
        out = torch.zeros(2, S, 128, device="cuda")
        if mode == 2:  # P V, k < m_end
            gemm(P, V, out, b_mn=True, causal=2)
            ref = P.float() @ V.float()
        else:  # P^T dO: a = P^T given as P storage (MN-major), k >= m_start
            gemm(P, V, out, a_mn=True, b_mn=True, causal=3)
            ref = P.float().transpose(-1, -2) @ V.float()
        torch.cuda.synchronize()
        assert rel_err(out, ref) < 2e-3


def test_gemm_gelu_bwd_epilogue(cuda_device, native):
    """dX = (dY W) * GELU'(pre) fused in the epilogue (the fc2 dgrad of the MLP backward)."""
    import ctypes as C
    from paper_2503_01890_b200 import _native as N
    M, Nn, K = 512, 1024, 256
    A, B, a_arg, b_arg = operands(M, Nn, K, 0, 1, seed=5)
    pre = torch.randn(M, Nn, device="cuda").bfloat16()
    out = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    d = N.GemmDesc()
    d.M, d.N, d.K, d.batch1, d.batch2 = M, Nn, K, 1, 1
    d.A, d.lda = a_arg.data_ptr(), K
    d.B, d.b_mn_major, d.ldb = b_arg.data_ptr(), 1, Nn
    d.C, d.ldc = out.data_ptr(), Nn
    d.aux, d.ld_aux = pre.data_ptr(), Nn
    d.alpha, d.epilogue = 1.0, 32
    N.check(N.lib().ah_gemm_bf16(C.byref(d), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    x = pre.float().requires_grad_(True)
    y = torch.nn.functional.gelu(x, approximate="tanh")
    g = A.float() @ B.float().T
    y.backward(g)
    assert rel_err(out, x.grad) < 1e-2


@pytest.mark.parametrize("M,N,K,a_mn,b_mn", [(8192, 2048, 4096, 0, 0), (2048, 8192, 4096, 1, 1), (4096, 2560, 4160, 0, 1)])
def test_gemm_stream_k_shapes(cuda_device, native, M, N, K, a_mn, b_mn):
    """Tile counts that fill the last wave poorly take the tail split (K halves handed
    between CTAs through a workspace); results must match the reference incl. epilogues."""
    from paper_2503_01890_b200.gemm import gemm
    A, B, a_arg, b_arg = operands(M, N, K, a_mn, b_mn, seed=M + N)
    bias = torch.randn(N, device="cuda").bfloat16()
    res = torch.randn(M, N, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):  # second launch reuses the workspace / flags with a new epoch
        gemm(a_arg, b_arg, C, a_mn=bool(a_mn), b_mn=bool(b_mn), bias=bias, residual=res)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T + bias.float() + res.float()
    assert rel_err(C, ref) < 1e-2


def test_gemm_stream_k_concurrent_streams(cuda_device, native):
    """Stream-K launches on different streams (in-process DP ranks) may overlap: each stream
    has its own partial-tile workspace and flags, so concurrent results equal serial ones."""
    from paper_2503_01890_b200.gemm import gemm
    M, N, K = 8192, 2048, 8192
    ops = [operands(M, N, K, 0, 0, seed=11 + i) for i in range(2)]
    serial = []
    for A, B, a_arg, b_arg in ops:
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        gemm(a_arg, b_arg, C)
        serial.append(C)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in ops]
    outs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in ops]
    for _ in range(20):
        for (A, B, a_arg, b_arg), st, C in zip(ops, streams, outs):
            with torch.cuda.stream(st):
                gemm(a_arg, b_arg, C, stream=st)
    torch.cuda.synchronize()
    for C, ref in zip(outs, serial):
        assert torch.equal(C, ref)
