"""Multi-process (gloo, world_size 2, CPU) test of the data-parallel optimizer sharding the
executor uses with NCCL on GPUs (north_star (d)): shard layout from the C-ABI
(ah_dp_shard), gradient reduce-scatter semantics (sum, 1/N folded into the optimizer),
sharded CPU AdamW (the product's ah_cpu_adam) and the bf16 all-gather of the updated
shards — bit-identical to one un-sharded update of the same summed gradient."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _bf16(a):
    return torch.from_numpy(a).to(torch.bfloat16)


def _worker(rank, world, port, n, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_01890_b200 import _native as N
    from paper_2503_01890_b200 import optim
    off, ln, sh = N.dp_shard(n, rank, world)
    rng = np.random.default_rng(100)  # identical replicas of the master state
    p = rng.normal(0, 0.02, n).astype(np.float32)
    m = rng.normal(0, 1e-3, n).astype(np.float32)
    v = (rng.normal(0, 1e-3, n) ** 2).astype(np.float32)
    g_local = np.random.default_rng(rank).normal(0, 1e-2, n).astype(np.float32)
    # bf16 local grads, padded to world * shard like the executor's wbuf
    g_pad = torch.zeros(sh * world, dtype=torch.bfloat16)
    g_pad[:n] = _bf16(g_local)
    # reduce-scatter(sum) == all-reduce then take my shard (gloo reduces in fp32 here)
    acc = g_pad.float()
    dist.all_reduce(acc)
    g_shard = acc[off:off + sh].to(torch.bfloat16).contiguous()
    # sharded state (zero padding) and the product CPU AdamW with 1/world folded in
    ps = torch.zeros(sh); ms = torch.zeros(sh); vs = torch.zeros(sh)
    ps[:ln] = torch.from_numpy(p[off:off + ln]); ms[:ln] = torch.from_numpy(m[off:off + ln])
    vs[:ln] = torch.from_numpy(v[off:off + ln])
    out = torch.empty(sh, dtype=torch.bfloat16)
    optim.cpu_adam(ps, ms, vs, g_shard, out, hp=optim.hparams(step=3), inv_scale=1.0 / world, nthreads=1)
    # all-gather of the updated bf16 shards -> full parameters on every rank
    parts = [torch.empty(sh // 2, dtype=torch.int32) for _ in range(world)]  # gloo: no 16-bit types
    dist.all_gather(parts, out.view(torch.int32))
    full = torch.cat(parts).view(torch.bfloat16)[:n]
    if rank == 0:
        out_q.put((off, ln, sh, full.view(torch.int16).numpy().copy(), ps[:ln].numpy().copy(),
                   acc[:n].to(torch.bfloat16).view(torch.int16).numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [8, 1001, 50_000 + 3])
def test_sharded_adam_matches_unsharded(native, n):
    from paper_2503_01890_b200 import _native as N
    from paper_2503_01890_b200 import optim
    world = 2
    # layout: disjoint, 16-byte aligned, covering [0, n)
    covered = 0
    for r in range(world):
        off, ln, sh = N.dp_shard(n, r, world)
        assert off % 8 == 0 and sh % 8 == 0 and off == r * sh
        covered += ln
    assert covered == n
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (n % 1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    off, ln, sh, full_bits, my_master, gsum_bits = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    # single-process reference: the whole vector, same summed bf16 gradient, same 1/N
    rng = np.random.default_rng(100)
    p = rng.normal(0, 0.02, n).astype(np.float32)
    m = rng.normal(0, 1e-3, n).astype(np.float32)
    v = (rng.normal(0, 1e-3, n) ** 2).astype(np.float32)
    tp, tm, tv = torch.from_numpy(p), torch.from_numpy(m), torch.from_numpy(v)
    g = torch.from_numpy(gsum_bits).view(torch.bfloat16)
    ref = torch.empty(n, dtype=torch.bfloat16)
    optim.cpu_adam(tp, tm, tv, g, ref, hp=optim.hparams(step=3), inv_scale=1.0 / world, nthreads=1)
    assert np.array_equal(full_bits, ref.view(torch.int16).numpy())
    assert np.array_equal(my_master.view(np.uint32), tp.numpy()[off:off + ln].view(np.uint32))
