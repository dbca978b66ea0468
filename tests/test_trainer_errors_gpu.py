"""Error behaviour of the executor's C-ABI mirrors the reference library's exceptions
(proj/core/include/hetsim/planner.hpp:35 InfeasibleError, std::invalid_argument from spec /
strategy validation, workload.cpp:11-13, costmodel.cpp:19): a negative AH_ERR_* code and a
message, no crash, no partially built trainer."""
import pytest

pytestmark = pytest.mark.gpu

MODEL = dict(num_blocks=3, hidden=256, heads=2, seq_len=256, batch=2, vocab=512)


def make(model=None, **plan):
    from paper_2503_01890_b200.trainer import ModelConfig, PlanConfig, Trainer
    return Trainer(ModelConfig(**(model or MODEL)), PlanConfig(fine_tune=False, **plan), seed=1, cpu_threads=2)


def test_infeasible_budget(cuda_device, native):
    from paper_2503_01890_b200._native import NativeError
    with pytest.raises(NativeError) as e:
        make(gpu_mem_budget=1 << 20, cpu_mem_budget=1 << 20)
    assert "(-3)" in str(e.value) and "GPU shortfall" in str(e.value)


def test_invalid_strategy(cuda_device, native):
    from paper_2503_01890_b200._native import NativeError
    with pytest.raises(NativeError) as e:  # p_hat > o_hat is rejected (costmodel.cpp:19)
        make(c_hat=0, p_hat=2, o_hat=1, gpu_mem_budget=1 << 40)
    assert "(-1)" in str(e.value) and "p_hat" in str(e.value)


def test_invalid_shape(cuda_device, native):
    from paper_2503_01890_b200._native import NativeError
    with pytest.raises(NativeError) as e:
        make(model=dict(MODEL, hidden=200), gpu_mem_budget=1 << 40)
    assert "(-1)" in str(e.value)


def test_trainer_usable_after_errors(cuda_device, native):
    import numpy as np
    tr = make(gpu_mem_budget=1 << 40)
    rng = np.random.default_rng(0)
    toks = rng.integers(0, MODEL["vocab"], size=(2, 256), dtype=np.int32)
    assert np.isfinite(tr.step(toks, toks))
    tr.close()
