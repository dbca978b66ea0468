"""CPU tests: the Adam oracle against torch.optim.AdamW, and the product CPU Adam
(ah_cpu_adam, the CpuOptim realisation) bit-exact against the oracle."""
import numpy as np
import pytest
import torch

from oracle import adam as oadam


@pytest.mark.parametrize("step", [1, 1000])
@pytest.mark.parametrize("scale", [1.0, 1024.0])
def test_oracle_matches_torch_adamw(oracle_built, step, scale):
    n = 4099
    p, m, v, g = oadam.synth(n, seed=7, scale=scale)
    inv = 1.0 / scale
    # torch reference in fp64 from the same state, then compare the fp32 oracle to it
    tp = torch.tensor(p, dtype=torch.float64, requires_grad=True)
    f32 = lambda x: float(np.float32(x))  # the C-ABI carries fp32 hyper-parameters
    opt = torch.optim.AdamW([tp], lr=f32(1e-4), betas=(f32(0.9), f32(0.999)), eps=f32(1e-8),
                            weight_decay=f32(0.01))
    opt.state[tp]["step"] = torch.tensor(float(step - 1), dtype=torch.float64)
    opt.state[tp]["exp_avg"] = torch.tensor(m, dtype=torch.float64)
    opt.state[tp]["exp_avg_sq"] = torch.tensor(v, dtype=torch.float64)
    tp.grad = torch.tensor(oadam.bf16_bits_to_f32(g), dtype=torch.float64) * inv
    opt.step()
    p32, m32, v32 = p.copy(), m.copy(), v.copy()
    out = oadam.adam_f32(p32, m32, v32, g, step=step, inv_scale=inv)
    ref_p = tp.detach().numpy()
    ref_m = opt.state[tp]["exp_avg"].numpy()
    ref_v = opt.state[tp]["exp_avg_sq"].numpy()
    # fp32 restatement vs fp64 torch: within 1e-6 relative (north_star tolerance), measured
    # element-wise against the array scale (cancellation in b1*m + (1-b1)*g makes a pure
    # per-element relative bound meaningless for near-zero outputs)
    for got, ref in ((p32, ref_p), (m32, ref_m), (v32, ref_v)):
        assert np.max(np.abs(got - ref)) <= 1e-6 * np.max(np.abs(ref))
    # bf16 cast within 1 ulp of bf16(torch fp64 result)
    ref_bits = oadam.cast_bf16(ref_p.astype(np.float32)).astype(np.int32)
    assert np.max(np.abs(out.astype(np.int32) - ref_bits)) <= 1


def test_oracle_fp64_agrees(oracle_built):
    p, m, v, g = oadam.synth(1000, seed=3)
    p64, m64, v64 = p.astype(np.float64), m.astype(np.float64), v.astype(np.float64)
    oadam.adam_f64(p64, m64, v64, g, step=10)
    oadam.adam_f32(p, m, v, g, step=10)
    np.testing.assert_allclose(p, p64, rtol=1e-6)


def test_oracle_multithread_is_identical(oracle_built):
    a = oadam.synth(300_001, seed=11)
    b = tuple(x.copy() for x in a)
    o1 = oadam.adam_f32(*a[:3], a[3], step=5)
    o2 = oadam.adam_f32(*b[:3], b[3], step=5, nthreads=4)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert np.array_equal(o1, o2)


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 16385, 100_003])
@pytest.mark.parametrize("step,scale,nonfinite", [(1, 1.0, False), (1000, 1024.0, False), (3, 1.0, True)])
def test_product_cpu_adam_bit_exact(native, oracle_built, n, step, scale, nonfinite):
    from paper_2503_01890_b200 import optim
    p, m, v, g = oadam.synth(n, seed=n + step, scale=scale, nonfinite=nonfinite)
    tp, tm, tv = torch.from_numpy(p.copy()), torch.from_numpy(m.copy()), torch.from_numpy(v.copy())
    tg = torch.from_numpy(g.copy()).view(torch.bfloat16)
    out = torch.empty(n, dtype=torch.bfloat16)
    optim.cpu_adam(tp, tm, tv, tg, out, hp=optim.hparams(step=step), inv_scale=1.0 / scale, nthreads=3)
    ref = oadam.adam_f32(p, m, v, g, step=step, inv_scale=1.0 / scale)
    for got, exp in ((tp, p), (tm, m), (tv, v)):
        assert np.array_equal(got.numpy().view(np.uint32), exp.view(np.uint32))  # same host: NaNs too
    assert np.array_equal(out.view(torch.int16).numpy().view(np.uint16), ref)


def test_product_cpu_adam_aliased_host_buffer(native, oracle_built):
    """14 B/param host layout: grad and updated bf16 params share one buffer."""
    from paper_2503_01890_b200 import optim
    p, m, v, g = oadam.synth(5000, seed=1)
    shared = torch.from_numpy(g.copy()).view(torch.bfloat16)
    tp, tm, tv = (torch.from_numpy(x.copy()) for x in (p, m, v))
    optim.cpu_adam(tp, tm, tv, shared, shared, hp=optim.hparams(step=2))
    ref = oadam.adam_f32(p, m, v, g, step=2)
    assert np.array_equal(shared.view(torch.int16).numpy().view(np.uint16), ref)


def test_abi_exports_every_declared_symbol(native):
    from paper_2503_01890_b200 import _native
    syms = _native.declared_symbols()
    assert len(syms) >= 10
    missing = [s for s in syms if not hasattr(native, s)]
    assert not missing, missing
