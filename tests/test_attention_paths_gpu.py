"""The unfused attention path (S GEMM + softmax kernel + P V GEMM, P kept), taken for shapes the
flash kernels do not cover (head_dim != 128), trains the same step as a torch fp32 reference.
The flash path is checked the same way in test_trainer_gpu.py / test_baseline_shapes_gpu.py."""
import numpy as np
import pytest
import torch

from tests import gpt_reference as ref

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("heads", [4, 8])  # head_dim 64, 32
def test_unfused_path_matches_torch(cuda_device, native, heads):
    from paper_2503_01890_b200.trainer import AdamConfig, ModelConfig, PlanConfig, Trainer
    model = ModelConfig(num_blocks=2, hidden=256, heads=heads, seq_len=256, batch=2, vocab=1000)
    if heads == 8:  # the trainer needs head_dim % 64 == 0
        with pytest.raises(Exception):
            Trainer(model, PlanConfig(c_hat=0, p_hat=0, o_hat=0, fine_tune=False, gpu_mem_budget=1 << 40))
        return
    lr = 1e3
    tr = Trainer(model, PlanConfig(c_hat=1, p_hat=0, o_hat=1, fine_tune=False, gpu_mem_budget=1 << 40),
                 AdamConfig(lr=lr, eps=1.0, weight_decay=0.0), seed=5, cpu_threads=2)
    h = model.hidden
    before = [torch.from_numpy(tr.master(i).copy()) for i in (1, 2)]
    wte = torch.from_numpy(tr.master(0).copy()).view(-1, h)
    wpe = torch.from_numpy(tr.master(-1).copy()).view(-1, h)
    lnf = torch.from_numpy(tr.master(-2).copy())
    rng = np.random.default_rng(1)
    t = rng.integers(0, model.vocab, size=(model.batch, model.seq_len), dtype=np.int32)
    y = rng.integers(0, model.vocab, size=(model.batch, model.seq_len), dtype=np.int32)
    loss = tr.step(t, y)
    after = [torch.from_numpy(tr.master(i).copy()) for i in (1, 2)]
    tr.close()
    rl, g_blocks, _, _, _ = ref.loss_and_grads(before, wte, wpe, lnf, torch.from_numpy(t).long(),
                                               torch.from_numpy(y).long(), heads, model.vocab)
    assert abs(loss - rl) / rl < 1e-2
    for i in range(2):
        est = -(after[i] - before[i]) / lr
        exp = g_blocks[i].reshape(-1) / (g_blocks[i].reshape(-1).abs() + 1.0)
        assert float((est - exp).norm() / exp.norm()) < 5e-2, i
