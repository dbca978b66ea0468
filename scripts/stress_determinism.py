"""Race hunt: the product path is deterministic (fixed-order reductions everywhere), so any
bitwise difference between repeated runs on the same input is a race.
  python scripts/stress_determinism.py kernels [reps]   flash fwd/bwd, LN, GEMM at the 1.3B shape
  python scripts/stress_determinism.py trainer [groups] two fresh trainers, bench plan, loss sequences
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def kernels(reps):
    from paper_2503_01890_b200.attention import flash_bwd, flash_fwd
    from paper_2503_01890_b200.gemm import gemm
    from paper_2503_01890_b200.layernorm import layernorm_bwd, layernorm_fwd
    torch.manual_seed(0)
    B, s, nh, hd = 8, 1024, 16, 128
    h = nh * hd
    qkv = (torch.randn(B, s, 3 * h, device="cuda") * 0.5).bfloat16()
    dO = torch.randn(B, s, h, device="cuda").bfloat16()
    x = torch.randn(B * s, h, device="cuda").bfloat16()
    g = (1 + 0.1 * torch.randn(h, device="cuda")).bfloat16()
    bt = (0.1 * torch.randn(h, device="cuda")).bfloat16()
    w = (torch.randn(4 * h, h, device="cuda") * 0.02).bfloat16()
    c = torch.empty(B * s, 4 * h, device="cuda", dtype=torch.bfloat16)

    def run():
        O, lse = flash_fwd(qkv, nh)
        dq = flash_bwd(qkv, O, dO, lse, nh)
        y, mean, rstd = layernorm_fwd(x, g, bt)
        dx, dgdb = layernorm_bwd(dO.view(B * s, h), x, mean, rstd, g)[:2]
        gemm(x, w, c)
        return [O, lse, dq, y, dx, dgdb, c.clone()]

    names = ["flash O", "flash lse", "flash dqkv", "ln y", "ln dx", "ln dgamma|dbeta", "gemm fc"]
    ref = run()
    torch.cuda.synchronize()
    bad = {n: 0 for n in names}
    nan = {n: 0 for n in names}
    for r in range(reps):
        out = run()
        for n, a, b in zip(names, ref, out):
            if not torch.equal(a.view(torch.uint8) if a.dtype != torch.float32 else a.view(torch.int32),
                               b.view(torch.uint8) if b.dtype != torch.float32 else b.view(torch.int32)):
                bad[n] += 1
            if not torch.isfinite(b.float()).all():
                nan[n] += 1
    torch.cuda.synchronize()
    print("reps", reps, "mismatches", bad, "nonfinite", nan, flush=True)


def flash_scales(reps):
    """Large score ranges drive the forward's lazy-rescale path (the running max moves by more than
    2^8 within a row); compare every repetition bitwise with the first and with torch fp32."""
    from paper_2503_01890_b200.attention import flash_bwd, flash_fwd
    B, s, nh, hd = 8, 1024, 16, 128
    h = nh * hd
    for scale in [float(x) for x in os.environ.get("SCALES", "0.5,2,4,8").split(",")]:
        torch.manual_seed(1)
        qkv = torch.randn(B, s, 3 * h, device="cuda")
        ramp = torch.linspace(0.2, 1.0, s, device="cuda").view(1, s, 1)  # later keys score higher
        qkv = (qkv * scale * ramp).bfloat16()
        dO = torch.randn(B, s, h, device="cuda").bfloat16()
        O0, l0 = flash_fwd(qkv, nh)
        d0 = flash_bwd(qkv, O0, dO, l0, nh)
        q, k, v = qkv.float().view(B, s, 3, nh, hd).permute(2, 0, 3, 1, 4)
        ref = torch.nn.functional.scaled_dot_product_attention(q[:2], k[:2], v[:2], is_causal=True)
        err = ((O0[:2].float().view(2, s, nh, hd).transpose(1, 2) - ref).abs().max() / ref.abs().max()).item()
        bo = bl = bd = nf = 0
        for _ in range(reps):
            O, l = flash_fwd(qkv, nh)
            d = flash_bwd(qkv, O, dO, l, nh)
            if not torch.equal(O.view(torch.int16), O0.view(torch.int16)):
                bo += 1
                if bo <= 3:
                    dif = (O.view(torch.int16) != O0.view(torch.int16)).view(B, s // 128, 128, nh, 2, 64)
                    idx = dif.nonzero()
                    tiles = sorted({(int(a), int(b_), int(c)) for a, b_, _, c, _, _ in idx.tolist()})
                    rows = sorted({int(x) for x in idx[:, 2].tolist()})
                    parts = sorted({int(x) for x in idx[:, 4].tolist()})
                    nanc = int((~torch.isfinite(O.float())).sum())
                    print(f"  diff elems {int(dif.sum())} nonfinite {nanc} (b,qtile,head) {tiles[:8]} n={len(tiles)} "
                          f"rows {rows[:10]}..{len(rows)} parts {parts} ref-finite {bool(torch.isfinite(O0.float()).all())}",
                          flush=True)
            bl += not torch.equal(l.view(torch.int32), l0.view(torch.int32))
            bd += not torch.equal(d.view(torch.int16), d0.view(torch.int16))
            nf += not (torch.isfinite(O.float()).all() and torch.isfinite(d.float()).all())
        torch.cuda.synchronize()
        print(f"scale {scale}: rel err vs torch {err:.2e}; mismatches O {bo} lse {bl} dqkv {bd} nonfinite {nf} / {reps}",
              flush=True)


def trainer(groups):
    import bench
    from paper_2503_01890_b200.trainer import ModelConfig, Trainer, plan_from_profile, profile_hardware
    m = bench.CONFIGS["1.3b"]
    model = ModelConfig(**m)
    threads = max(1, (os.cpu_count() or 8) - 4)
    prof = profile_hardware(model, cpu_threads=threads)
    cpu_gib = max(8, int(0.8 * os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30))
    plan = plan_from_profile(prof, bench.GPU_BUDGET_GIB["1.3b"] << 30, cpu_gib << 30)
    T = m["batch"] * m["seq_len"]
    rng = np.random.default_rng(4321)
    tok = [torch.from_numpy(rng.integers(0, m["vocab"], size=T, dtype=np.int32)).cuda() for _ in range(4)]
    tgt = [torch.from_numpy(rng.integers(0, m["vocab"], size=T, dtype=np.int32)).cuda() for _ in range(4)]
    seqs = []
    for run in range(int(os.environ.get("RUNS", "2"))):
        tr = Trainer(model, plan, seed=1234, cpu_threads=threads)
        losses = []
        k = 0
        for gi in range(groups):
            for _ in range(4):
                tr.submit(tok[k % 4], tgt[k % 4])
                k += 1
            losses.append(tr.drain())
        tr.close()
        del tr
        print("run", run, "strategy", (plan.c_hat, plan.p_hat, plan.o_hat), "losses", losses, flush=True)
        seqs.append(losses)
    diff = [(r, i) for r in range(1, len(seqs)) for i, (a, b) in enumerate(zip(seqs[0], seqs[r])) if not (a == b)]
    nonfinite = [i for s in seqs for i, v in enumerate(s) if not np.isfinite(v)]
    print("differing groups", diff, "nonfinite", nonfinite, flush=True)


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "kernels"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    if mode == "flash":
        flash_scales(n or 100)
    elif mode == "kernels":
        kernels(n or 200)
    else:
        trainer(n or 12)
