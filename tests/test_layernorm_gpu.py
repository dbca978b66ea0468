"""LayerNorm kernels (row-parallel fused forward / backward + fused bias column sums) vs a
torch fp32 reference of the same op, through the C-ABI (ah_layernorm_fwd / _bwd)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

# tolerances: bf16 outputs (8-bit mantissa) of fp32 math -> relative error of a few 1e-3
TOL = 1.5e-2


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30))


def ref_ln(x, g, b):
    xf = x.float().requires_grad_(True)
    gf = g.float().requires_grad_(True)
    bf = b.float().requires_grad_(True)
    y = torch.nn.functional.layer_norm(xf, (x.shape[1],), gf, bf, eps=1e-5)
    return xf, gf, bf, y


@pytest.mark.parametrize("rows,h", [(8192, 2048), (1000, 768), (37, 256), (4096, 6144), (64, 1000), (1, 2048)])
@pytest.mark.parametrize("with_res", [False, True])
def test_layernorm_fwd_bwd(cuda_device, native, rows, h, with_res):
    from paper_2503_01890_b200.layernorm import layernorm_bwd, layernorm_fwd
    torch.manual_seed(rows + h)
    x = (torch.randn(rows, h, device="cuda") * 2 + 0.5).bfloat16()
    g = (1 + 0.1 * torch.randn(h, device="cuda")).bfloat16()
    b = (0.1 * torch.randn(h, device="cuda")).bfloat16()
    dy = torch.randn(rows, h, device="cuda").bfloat16()
    dres = torch.randn(rows, h, device="cuda").bfloat16() if with_res else None
    y, mean, rstd = layernorm_fwd(x, g, b)
    xf, gf, bf, yr = ref_ln(x, g, b)
    assert rel(y, yr) < TOL
    assert torch.allclose(mean, xf.detach().mean(1), atol=1e-4, rtol=1e-4)
    yr.backward(dy.float())
    fused = h % 256 == 0 and h <= 6144
    dx, dgdb, cr, cx = layernorm_bwd(dy, x, mean, rstd, g, dres, bias_sums=fused)
    dx_ref = xf.grad + (dres.float() if with_res else 0)
    assert rel(dx, dx_ref) < TOL
    assert rel(dgdb[:h], gf.grad) < TOL
    assert rel(dgdb[h:], bf.grad) < TOL
    if fused:
        assert rel(cx, dx.float().sum(0)) < TOL
        if with_res:
            assert rel(cr, dres.float().sum(0)) < TOL
    # deterministic: a second launch gives identical bits
    dx2, dgdb2, cr2, cx2 = layernorm_bwd(dy, x, mean, rstd, g, dres, bias_sums=fused)
    assert torch.equal(dx, dx2) and torch.equal(dgdb, dgdb2)
    if fused:
        assert torch.equal(cx, cx2)


def test_layernorm_empty(cuda_device, native):
    from paper_2503_01890_b200.layernorm import layernorm_fwd
    x = torch.empty(0, 2048, dtype=torch.bfloat16, device="cuda")
    g = torch.ones(2048, dtype=torch.bfloat16, device="cuda")
    y, mean, rstd = layernorm_fwd(x, g, g)
    assert y.shape == (0, 2048)
