"""The fused tcgen05 attention paths (flash: O + lse saved, P recomputed; twopass: P saved) and
the unfused GEMM + softmax + GEMM path give the same training step within bf16 tolerance (the
path is selected with AH_ATTENTION in a subprocess, since the choice is latched per process)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, %r)
from paper_2503_01890_b200.trainer import AdamConfig, ModelConfig, PlanConfig, Trainer
m = ModelConfig(num_blocks=2, hidden=256, heads=2, seq_len=512, batch=2, vocab=1000)
tr = Trainer(m, PlanConfig(c_hat=1, p_hat=0, o_hat=0, fine_tune=False, gpu_mem_budget=1 << 40),
             AdamConfig(lr=1.0, eps=1.0, weight_decay=0.0), seed=5, cpu_threads=2)
rng = np.random.default_rng(1)
t = rng.integers(0, m.vocab, size=m.batch * m.seq_len, dtype=np.int32)
y = rng.integers(0, m.vocab, size=m.batch * m.seq_len, dtype=np.int32)
before = [tr.master(i).copy() for i in (1, 2)]
loss = tr.step(t, y)
delta = [(tr.master(i) - b).tolist() for i, b in zip((1, 2), before)]
print(json.dumps({"loss": loss, "delta": delta}))
"""


def run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT % ROOT], env=env, capture_output=True, text=True, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("mode", ["flash", "twopass"])
def test_fused_and_unfused_attention_agree(cuda_device, native, mode):
    fused = run({"AH_ATTENTION": mode})
    unfused = run({"AH_ATTENTION": "unfused"})
    assert abs(fused["loss"] - unfused["loss"]) < 1e-3 * abs(unfused["loss"])
    for a, b in zip(fused["delta"], unfused["delta"]):
        a, b = np.array(a), np.array(b)
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 3e-2
