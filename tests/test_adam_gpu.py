"""GPU parity: fused sm_100a AdamW (ah_adam_step, the GpuOptim realisation) is bit-identical
to the C oracle (oracle/adam_oracle.c) on the same seeded inputs, incl. edge cases."""
import os

import numpy as np
import pytest
import torch

from oracle import adam as oadam

pytestmark = pytest.mark.gpu


def same_f32(got, exp):
    """Bit-identical, except NaN payloads (GPU canonical NaN 0x7fffffff vs x86 0x7fc00000)."""
    gn, en = np.isnan(got), np.isnan(exp)
    return np.array_equal(gn, en) and np.array_equal(got[~gn].view(np.uint32), exp[~en].view(np.uint32))


def same_bf16(got, exp):
    gf, ef = oadam.bf16_bits_to_f32(got), oadam.bf16_bits_to_f32(exp)
    return same_f32(gf, ef)


def _run_gpu(p, m, v, g, step, inv, want_bf16=True, offset=0, stats=None, skip=None):
    from paper_2503_01890_b200 import optim
    n = p.size
    # allocate with an element offset to exercise the unaligned path
    tp = torch.zeros(n + offset, dtype=torch.float32, device="cuda")[offset:]
    tm = torch.zeros_like(tp)
    tv = torch.zeros_like(tp)
    tg = torch.zeros(n + offset, dtype=torch.int16, device="cuda")[offset:]
    tp.copy_(torch.from_numpy(p))
    tm.copy_(torch.from_numpy(m))
    tv.copy_(torch.from_numpy(v))
    tg.copy_(torch.from_numpy(g.view(np.int16)))
    out = torch.zeros(n + offset, dtype=torch.bfloat16, device="cuda")[offset:] if want_bf16 else None
    optim.adam_step(tp, tm, tv, tg.view(torch.bfloat16), out, hp=optim.hparams(step=step), inv_scale=inv,
                    stats=stats, skip_flag=skip)
    torch.cuda.synchronize()
    res = [t.cpu().numpy() for t in (tp, tm, tv)]
    res.append(out.view(torch.int16).cpu().numpy().view(np.uint16) if want_bf16 else None)
    return res


@pytest.mark.parametrize("n", [0, 1, 7, 8, 15, 4096, 1_000_003, 7_087_872])
@pytest.mark.parametrize("step,scale,nonfinite", [(1, 1.0, False), (1000, 1024.0, False), (2, 1.0, True)])
def test_adam_gpu_bit_exact(cuda_device, native, oracle_built, n, step, scale, nonfinite):
    p, m, v, g = oadam.synth(n, seed=n ^ step, scale=scale, nonfinite=nonfinite)
    gp, gm, gv, gout = _run_gpu(p, m, v, g, step, 1.0 / scale)
    ref = oadam.adam_f32(p, m, v, g, step=step, inv_scale=1.0 / scale)
    for got, exp in ((gp, p), (gm, m), (gv, v)):
        assert same_f32(got, exp)
    assert same_bf16(gout, ref)


@pytest.mark.parametrize("offset", [1, 3])
def test_adam_gpu_unaligned(cuda_device, native, oracle_built, offset):
    p, m, v, g = oadam.synth(10_001, seed=5)
    gp, gm, gv, gout = _run_gpu(p, m, v, g, 4, 1.0, offset=offset)
    ref = oadam.adam_f32(p, m, v, g, step=4)
    assert np.array_equal(gp.view(np.uint32), p.view(np.uint32))
    assert np.array_equal(gout, ref)


def test_adam_gpu_no_bf16_out(cuda_device, native, oracle_built):
    p, m, v, g = oadam.synth(65_537, seed=9)
    gp, _, _, _ = _run_gpu(p, m, v, g, 1, 1.0, want_bf16=False)
    oadam.adam_f32(p, m, v, g, step=1, want_bf16=False)
    assert np.array_equal(gp.view(np.uint32), p.view(np.uint32))


STATS_FLOATS = 520  # AH_STATS_FLOATS (include/autohete.h)


def test_adam_gpu_stats_and_skip(cuda_device, native, oracle_built):
    p, m, v, g = oadam.synth(300_000, seed=21, nonfinite=True)
    stats = torch.zeros(STATS_FLOATS, dtype=torch.float32, device="cuda")
    _run_gpu(p, m, v, g, 1, 1.0, stats=stats)
    s = stats.cpu()
    bad = int(s.view(torch.int32)[1])
    assert bad == 2
    # skip flag set: state must be untouched
    skip = torch.ones(1, dtype=torch.int32, device="cuda")
    gp, gm, gv, _ = _run_gpu(p, m, v, g, 1, 1.0, skip=skip)
    assert np.array_equal(gp.view(np.uint32), p.view(np.uint32))
    assert np.array_equal(gv.view(np.uint32), v.view(np.uint32))


def test_grad_stats_matches_oracle(cuda_device, native, oracle_built):
    from paper_2503_01890_b200 import optim
    _, _, _, g = oadam.synth(1_234_567, seed=2, scale=3.0)
    stats = torch.zeros(STATS_FLOATS, dtype=torch.float32, device="cuda")
    tg = torch.from_numpy(g.view(np.int16)).cuda().view(torch.bfloat16)
    optim.grad_stats(tg, stats, inv_scale=0.5)
    torch.cuda.synchronize()
    ref_sum, ref_bad = oadam.grad_stats(g, 0.5)
    assert int(stats.cpu().view(torch.int32)[1]) == ref_bad == 0
    assert abs(float(stats[0]) - ref_sum) <= 1e-4 * ref_sum


def test_cast_bit_exact(cuda_device, native, oracle_built):
    from paper_2503_01890_b200 import optim
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(100_003) * 10).astype(np.float32)
    x[:4] = [np.inf, -np.inf, np.nan, 3.3895314e38]
    out = torch.empty(x.size, dtype=torch.bfloat16, device="cuda")
    optim.cast_f32_bf16(torch.from_numpy(x).cuda(), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.view(torch.int16).cpu().numpy().view(np.uint16), oadam.cast_bf16(x))


def test_grad_stats_deterministic_and_skip_from_stats(cuda_device, native, oracle_built):
    """The cross-CTA reduction has a fixed order (no float atomics): repeated launches give
    bitwise-identical sums, accumulation over launches is in stream order, and the non-finite
    count drives the Adam skip flag (the executor's per-block overflow check)."""
    from paper_2503_01890_b200 import optim
    _, _, _, g = oadam.synth(50_358_272, seed=4, scale=2.0)  # one 1.3B block (C2)
    tg = torch.from_numpy(g.view(np.int16)).cuda().view(torch.bfloat16)
    sums = set()
    for _ in range(5):
        st = torch.zeros(STATS_FLOATS, dtype=torch.float32, device="cuda")
        optim.grad_stats(tg, st)
        optim.grad_stats(tg[:1_000_001], st)  # second launch accumulates
        torch.cuda.synchronize()
        sums.add(int(st[:1].view(torch.int32).item()))
        assert int(st.view(torch.int32)[2].item()) == 0  # ticket re-armed
    assert len(sums) == 1
    ref_a, _ = oadam.grad_stats(g, 1.0)
    ref_b, _ = oadam.grad_stats(g[:1_000_001], 1.0)
    assert abs(float(st[0]) - (ref_a + ref_b)) <= 1e-4 * (ref_a + ref_b)
    # a non-finite grad -> the count is the skip flag of the update that follows
    p, m, v, g2 = oadam.synth(200_000, seed=8, nonfinite=True)
    tg2 = torch.from_numpy(g2.view(np.int16)).cuda().view(torch.bfloat16)
    st = torch.zeros(STATS_FLOATS, dtype=torch.float32, device="cuda")
    optim.grad_stats(tg2, st)
    gp, _, gv, _ = _run_gpu(p, m, v, g2, 1, 1.0, skip=st[1:2].view(torch.int32))
    assert np.array_equal(gp.view(np.uint32), p.view(np.uint32))
    assert np.array_equal(gv.view(np.uint32), v.view(np.uint32))


@pytest.mark.parametrize("n", [50_358_272, 453_064_704])  # m_p of the 1.3B (C2) and 10B (C3) blocks
def test_adam_gpu_bit_exact_block_sizes(cuda_device, native, oracle_built, n):
    """Bit-exact at the BASELINE block sizes the bench updates (SURVEY §8(a) m_p values)."""
    p, m, v, g = oadam.synth(n, seed=n % 1000, scale=1.0)
    gp, gm, gv, gout = _run_gpu(p, m, v, g, 7, 1.0)
    ref = oadam.adam_f32(p, m, v, g, step=7, nthreads=os.cpu_count() or 1)
    for got, exp in ((gp, p), (gm, m), (gv, v)):
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
    assert np.array_equal(gout, ref)
