"""Parity of the composed training step at the BASELINE block shapes:
h = 2048 / 16 heads (1.3B), 6144 / 48 heads (10B), 8192 / 64 heads (20B), s = 1024, the full
GPT-2 vocabulary V = 50257 through the padded (50432-row) LM head — one executor iteration vs a
plain torch fp32 reference of the same model (tests/gpt_reference.py) on the GPU.

The gradient the CUDA path computed is read back through one AdamW step with lr = 1e4, eps = 1,
no decay: p' = p - 1e4 * g / (|g| + 1) in fp32, so -(p' - p) / 1e4 = g / (|g| + 1) ~= g exposes it
(to fp32 rounding of p, ~1e-7 relative here). Tolerances (bf16 weights / activations, fp32
accumulation): loss 1 % relative, every weight slice's gradient 5 % relative Frobenius error."""
import numpy as np
import pytest
import torch

from tests import gpt_reference as ref

pytestmark = pytest.mark.gpu

LR = 1e4

SHAPES = [  # (hidden, heads, blocks, batch): BASELINE block shapes, batch sized for the fp32 reference
    pytest.param(2048, 16, 2, 2, id="1.3b-block"),
    pytest.param(6144, 48, 1, 1, id="10b-block"),
    pytest.param(8192, 64, 1, 1, id="20b-block"),
]


@pytest.mark.parametrize("h,nh,L,B", SHAPES)
def test_step_at_baseline_block_shape(cuda_device, native, h, nh, L, B):
    from paper_2503_01890_b200.trainer import AdamConfig, ModelConfig, PlanConfig, Trainer
    s, V = 1024, 50257
    model = ModelConfig(num_blocks=L, hidden=h, heads=nh, seq_len=s, batch=B, vocab=V)
    # a plan that exercises recompute and the host optimizer on the last block
    plan = PlanConfig(c_hat=L, p_hat=0, o_hat=1, fine_tune=False, gpu_mem_budget=1 << 40)
    tr = Trainer(model, plan, AdamConfig(lr=LR, eps=1.0, weight_decay=0.0), seed=3, cpu_threads=8)
    dev = torch.device("cuda")
    before = [torch.from_numpy(tr.master(i).copy()).to(dev) for i in range(1, L + 1)]
    wte = torch.from_numpy(tr.master(0).copy()).to(dev).view(-1, h)
    wpe = torch.from_numpy(tr.master(-1).copy()).to(dev).view(-1, h)
    lnf = torch.from_numpy(tr.master(-2).copy()).to(dev)
    assert wte.shape[0] == 50432 and not wte[V:].any()  # padded head rows are zero
    rng = np.random.default_rng(h)
    toks = rng.integers(0, V, size=(B, s), dtype=np.int32)
    tgts = rng.integers(0, V, size=(B, s), dtype=np.int32)
    loss = tr.step(toks, tgts)
    after = [torch.from_numpy(tr.master(i).copy()).to(dev) for i in range(1, L + 1)]
    wte_after = torch.from_numpy(tr.master(0).copy()).to(dev).view(-1, h)
    st = tr.stats()
    tr.close()
    assert st["skipped_updates"] == 0 and np.isfinite(st["grad_norm"])

    rl, g_blocks, g_wte, _, _ = ref.loss_and_grads(before, wte, wpe, lnf, torch.from_numpy(toks).long().to(dev),
                                                   torch.from_numpy(tgts).long().to(dev), nh, V)
    assert abs(loss - rl) / rl < 1e-2, (loss, rl)
    slices = ref.block_slices(h)
    for i in range(L):
        est = -(after[i] - before[i]) / LR
        g = g_blocks[i].reshape(-1)
        exp = g / (g.abs() + 1.0)
        for name, (a, shape) in slices.items():
            n = int(np.prod(shape))
            e, x = est[a:a + n], exp[a:a + n]
            if name == "b_qkv":  # the key bias has zero gradient (softmax shift invariance): q, v parts
                keep = torch.ones(n, dtype=torch.bool, device=dev)
                keep[h:2 * h] = False
                assert float(e[h:2 * h].abs().max()) < 5e-2 * float(x[keep].abs().max())
                e, x = e[keep], x[keep]
            err = float((e - x).norm() / x.norm())
            assert err < 5e-2, (i + 1, name, err)
    est = -(wte_after - wte)[:V] / LR
    exp = (g_wte / (g_wte.abs() + 1.0))[:V]
    assert float((est - exp).norm() / exp.norm()) < 5e-2
