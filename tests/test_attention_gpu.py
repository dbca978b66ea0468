"""Fused tcgen05 attention forward vs a torch fp32 reference (causal softmax(QK^T/sqrt(d)) V).
Tolerances: bf16 operands / bf16 P, fp32 accumulation."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,s,nh", [(1, 128, 1), (2, 256, 2), (2, 1024, 4)])
def test_attention_fwd_matches_reference(cuda_device, native, B, s, nh):
    from paper_2503_01890_b200.attention import attention_fwd
    hd = 128
    h = nh * hd
    g = torch.Generator(device="cuda").manual_seed(s + nh)
    qkv = (torch.randn(B, s, 3 * h, device="cuda", generator=g) * 0.5).bfloat16()
    O, P = attention_fwd(qkv, nh)
    torch.cuda.synchronize()
    q, k, v = qkv.float().split(h, dim=-1)
    q = q.view(B, s, nh, hd).transpose(1, 2)
    k = k.view(B, s, nh, hd).transpose(1, 2)
    v = v.view(B, s, nh, hd).transpose(1, 2)
    S = q @ k.transpose(-1, -2) / math.sqrt(hd)
    mask = torch.ones(s, s, device="cuda").tril().bool()
    S = S.masked_fill(~mask, float("-inf"))
    Pr = torch.softmax(S, dim=-1)
    Or = (Pr @ v).transpose(1, 2).reshape(B, s, h)
    err = (O.float() - Or).norm() / Or.norm()
    assert err < 1e-2, float(err)
    # P: normalised, zero above the diagonal (within written tiles)
    Pm = P.float().masked_fill(~mask, 0.0)
    assert (Pm - Pr).abs().max() < 4e-3
    tile = torch.zeros(s, s, dtype=torch.bool, device="cuda")
    for i in range(0, s, 128):
        tile[i:i + 128, :i + 128] = True
    assert P.float()[..., tile & ~mask].abs().max() == 0
    assert torch.allclose(Pm.sum(-1), torch.ones_like(Pm.sum(-1)), atol=2e-2)
