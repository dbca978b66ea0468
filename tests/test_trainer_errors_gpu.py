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


def test_host_ids_out_of_range_rejected(cuda_device, native):
    """Ids index wte / dwte / the logits rows: a host batch with an id outside [0, V) (e.g. the
    PyTorch ignore_index -100) is rejected before anything is enqueued (AH_ERR_INVALID)."""
    import numpy as np
    from paper_2503_01890_b200._native import NativeError
    tr = make(gpu_mem_budget=1 << 40)
    rng = np.random.default_rng(0)
    toks = rng.integers(0, MODEL["vocab"], size=(2, 256), dtype=np.int32)
    for bad_tok, bad_tgt in ((MODEL["vocab"], 0), (0, -100)):
        t, y = toks.copy(), toks.copy()
        t[1, 7] = bad_tok if bad_tok else t[1, 7]
        y[0, 3] = bad_tgt if bad_tgt else y[0, 3]
        with pytest.raises(NativeError) as e:
            tr.step(t, y)
        assert "(-1)" in str(e.value) and "outside [0, vocab)" in str(e.value)
    assert np.isfinite(tr.step(toks, toks))  # still usable
    tr.close()


def test_device_ids_out_of_range_flagged(cuda_device, native):
    """Device batches are sanitised on the GPU: bad ids are trained as id 0 (no out-of-bounds
    access) and drain() reports the batch; the next clean batch drains normally."""
    import numpy as np
    import torch
    from paper_2503_01890_b200._native import NativeError
    tr = make(gpu_mem_budget=1 << 40)
    rng = np.random.default_rng(1)
    toks = torch.from_numpy(rng.integers(0, MODEL["vocab"], size=512, dtype=np.int32)).cuda()
    bad = toks.clone()
    bad[5] = 1 << 30
    tr.submit(bad, toks)
    with pytest.raises(NativeError) as e:
        tr.drain()
    assert "on-device batch" in str(e.value)
    tr.submit(toks, toks)
    assert np.isfinite(tr.drain())
    tr.close()


def test_reset_stats(cuda_device, native):
    import numpy as np
    tr = make(c_hat=1, p_hat=1, o_hat=2, gpu_mem_budget=1 << 40)
    toks = np.random.default_rng(2).integers(0, MODEL["vocab"], size=(2, 256), dtype=np.int32)
    tr.step(toks, toks)
    tr.step(toks, toks)
    assert sum(tr.stats()["lane_ops"]) > 0
    from paper_2503_01890_b200 import _native as N
    N.check(N.lib().ah_trainer_reset_stats(tr._h), "reset")
    s = tr.stats()
    assert sum(s["lane_ops"]) == 0 and s["lane_busy_ms"] == [0.0] * 4 and s["window_iters"] == 0
    tr.close()
