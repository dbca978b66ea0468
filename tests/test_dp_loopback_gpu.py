"""The data-parallel path end to end on one GPU: N in-process ranks exchange through the
loopback communicator (same in-place all-gather / reduce-scatter / all-reduce semantics as the
NCCL path; NCCL refuses two ranks on one device). Checks: per-rank shards assembled after a step
equal a single-rank step on the concatenated batch (1/N gradient scaling, shard offsets, CPU and
GPU optimizer shards, host-link shards, recompute), replicated embedding state is identical on
every rank, the loss matches, and the run is deterministic."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MODEL = dict(num_blocks=3, hidden=256, heads=2, seq_len=256, batch=2, vocab=512)
PLANS = [dict(c_hat=0, p_hat=0, o_hat=0), dict(c_hat=1, p_hat=1, o_hat=2, prefetch_lookahead=[1, 1, 1])]


def batches(n, seed=0):
    rng = np.random.default_rng(seed)
    shape = (MODEL["batch"], MODEL["seq_len"])
    return [(rng.integers(0, MODEL["vocab"], size=shape, dtype=np.int32),
             rng.integers(0, MODEL["vocab"], size=shape, dtype=np.int32)) for _ in range(n)]


def adam():
    from paper_2503_01890_b200.trainer import AdamConfig
    # eps >> |g|, lr 1, no decay: the step moves p by ~ -g, exposing the gradient
    return AdamConfig(lr=1.0, eps=1.0, weight_decay=0.0)


def run_dp(n, plan, data):
    from paper_2503_01890_b200.trainer import LoopbackComm, ModelConfig, PlanConfig, Trainer
    comm = LoopbackComm(n)
    trs = [Trainer(ModelConfig(**MODEL), PlanConfig(fine_tune=False, gpu_mem_budget=1 << 40, **plan), adam(),
                   seed=7, cpu_threads=2, dp_rank=r, dp_size=n, loopback=comm) for r in range(n)]
    for r, tr in enumerate(trs):
        tr.submit(*data[r])
    losses = [tr.drain() for tr in trs]
    L, mp = MODEL["num_blocks"], None
    blocks = []
    for i in range(1, L + 1):
        shards = [tr.master(i) for tr in trs]
        blocks.append(np.concatenate(shards))
    emb = [[tr.master(i).copy() for i in (0, -1, -2)] for tr in trs]
    for tr in trs:
        tr.close()
    comm.close()
    return losses, blocks, emb


def run_single(plan, data):
    from paper_2503_01890_b200.trainer import ModelConfig, PlanConfig, Trainer
    m = dict(MODEL, batch=MODEL["batch"] * len(data))
    tr = Trainer(ModelConfig(**m), PlanConfig(fine_tune=False, gpu_mem_budget=1 << 40, **plan), adam(), seed=7,
                 cpu_threads=2)
    before = [tr.master(i).copy() for i in range(1, MODEL["num_blocks"] + 1)]
    toks = np.concatenate([d[0] for d in data])
    tgts = np.concatenate([d[1] for d in data])
    loss = tr.step(toks, tgts)
    after = [tr.master(i).copy() for i in range(1, MODEL["num_blocks"] + 1)]
    emb = [tr.master(i).copy() for i in (0, -1, -2)]
    tr.close()
    return loss, before, after, emb


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("plan", PLANS)
@pytest.mark.parametrize("n", [2, 3])
def test_dp_loopback_matches_single_rank(cuda_device, native, plan, n):
    data = batches(n)
    losses, blocks, emb = run_dp(n, plan, data)
    loss1, before, after, emb1 = run_single(plan, data)
    assert abs(float(np.mean(losses)) - loss1) < 1e-2 * abs(loss1)
    for i in range(MODEL["num_blocks"]):
        mp = after[i].size
        d_dp = blocks[i][:mp] - before[i]
        d_1 = after[i] - before[i]
        assert rel(d_dp, d_1) < 5e-2, (i, rel(d_dp, d_1))
        assert not np.any(blocks[i][mp:])  # shard padding stays zero
    for r in range(1, n):  # replicated state: identical bits on every rank
        for a, b in zip(emb[0], emb[r]):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    for a, b in zip(emb[0], emb1):
        assert rel(a - 0, b - 0) < 1e-2


def test_dp_loopback_is_deterministic(cuda_device, native):
    data = batches(2, seed=5)
    l1, b1, _ = run_dp(2, PLANS[1], data)
    l2, b2, _ = run_dp(2, PLANS[1], data)
    assert l1 == l2
    for a, b in zip(b1, b2):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("n", [2, 3, 8])
def test_loopback_reduce_scatter_is_nccl_ring(cuda_device, native, n):
    """The loopback bf16 reduce-scatter computes exactly NCCL's ring algorithm (chunk r summed from
    rank r+1 around the ring to its owner r, rounding the running partial to bf16 at every hop),
    and the dp-n tolerance derived for it holds: |ring - exact| <= (n-1) * 2^-8 * sum_q |g_q|
    per element (bf16 unit roundoff 2^-8, one rounding per hop)."""
    import threading

    import torch

    from oracle import adam as oadam
    from paper_2503_01890_b200 import _native as N
    from paper_2503_01890_b200.trainer import LoopbackComm
    shard = 100_003
    g = torch.Generator(device="cuda").manual_seed(n)
    # mixed magnitudes so the per-hop rounding matters
    bufs = [(torch.randn(n * shard, device="cuda", generator=g) * torch.exp(
        torch.randn(n * shard, device="cuda", generator=g) * 2)).bfloat16() for _ in range(n)]
    host = [b.view(torch.int16).cpu().numpy().view(np.uint16) for b in bufs]
    torch.cuda.synchronize()
    comm = LoopbackComm(n)
    errs = []

    def rank(r):
        rc = N.lib().ah_dp_loopback_call(comm.handle, r, 1, bufs[r].data_ptr(), shard, None)
        errs.append(rc)

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    comm.close()
    assert errs == [0] * n
    for r in range(n):
        sl = slice(r * shard, (r + 1) * shard)
        acc = oadam.bf16_bits_to_f32(host[(r + 1) % n][sl])
        for k in range(1, n):
            acc = oadam.bf16_bits_to_f32(oadam.cast_bf16(acc + oadam.bf16_bits_to_f32(host[(r + 1 + k) % n][sl])))
        got = bufs[r].view(torch.int16).cpu().numpy().view(np.uint16)[sl]
        assert np.array_equal(got, oadam.cast_bf16(acc)), r
        vals = np.stack([oadam.bf16_bits_to_f32(h[sl]).astype(np.float64) for h in host])
        exact, mag = vals.sum(0), np.abs(vals).sum(0)
        err = np.abs(oadam.bf16_bits_to_f32(got).astype(np.float64) - exact)
        assert np.all(err <= (n - 1) * 2.0 ** -8 * mag + 1e-30), r
