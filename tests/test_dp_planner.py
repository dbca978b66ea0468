"""Data-parallel planner extension (include/hetsim/dp_planner.hpp) on CPU:
* dp_size = 1 gives exactly the reference planner's plan document;
* dp_size > 1 matches the oracle/dp_planner.py brute force (strategy, objective bit-for-bit,
  feasible count, per-rank Eq.(1)_N / Eq.(2)_N bytes) over seeded random GPT configurations,
  with and without a modelled collective bandwidth, including infeasible budgets."""
import json
import random

import pytest

from oracle import dp_planner as ref
from paper_2503_01890_b200 import hetsim_py as H
from paper_2503_01890_b200._native import NativeError


def config(L, h, s, b, V, gib, cpu_gib, tflops, h2d, d2h, cpu_mps, gpu_mps):
    return f"""[model]
num_blocks = {L}
hidden_size = {h}
seq_len = {s}
batch_size = {b}
vocab_size = {V}

[hardware]
gpu_mem_gib = {gib}
cpu_mem_gib = {cpu_gib}
gpu_tflops = {tflops}
h2d_gbps = {h2d}
d2h_gbps = {d2h}
cpu_optim_mparams_s = {cpu_mps}
gpu_optim_mparams_s = {gpu_mps}
"""


def cases(n=40, seed=2503):
    rng = random.Random(seed)
    out = [(8, 2048, 1024, 8, 50257, 12, 128, 100, 20, 20, 500, 20000)]  # tests/golden/kconfig.conf
    for _ in range(n):
        h = rng.choice([768, 1024, 2048, 4096, 6144, 8192])
        out.append((rng.randint(4, 28), h, rng.choice([512, 1024, 2048]), rng.choice([1, 2, 4, 8]), 50257,
                    rng.choice([8, 16, 24, 40, 80, 120, 180]), rng.choice([16, 64, 128, 256]),
                    rng.choice([300, 600, 1200]), rng.choice([25, 55]), rng.choice([25, 55]),
                    rng.choice([1000, 5000]), rng.choice([100000, 200000])))
    return out


def test_dp1_is_the_reference_plan():
    for c in cases(20):
        text = config(*c)
        try:
            ref_doc = H.plan_json(text)
        except NativeError as e:
            with pytest.raises(NativeError):
                H.plan_dp_json(text, 1, 0.0)
            continue
        assert H.plan_dp_json(text, 1, 0.0) == ref_doc
        assert H.plan_dp_json(text, 1, 400.0) == ref_doc  # collectives do not exist at dp 1


@pytest.mark.parametrize("n,coll", [(2, 0.0), (4, 0.0), (8, 0.0), (8, 400.0), (8, 40.0), (3, 100.0)])
def test_dp_plan_matches_brute_force(n, coll):
    for c in cases():
        L, h, s, b, V, gib, cpu_gib, tflops, h2d, d2h, cpu_mps, gpu_mps = c
        pr = ref.profile(L, h, s, b, V, tflops, h2d, d2h, cpu_mps, gpu_mps)
        want = ref.solve(pr, ref.llround(gib * 2.0**30), ref.llround(cpu_gib * 2.0**30), n, coll * 1e9)
        text = config(*c)
        if want is None:
            with pytest.raises(NativeError):
                H.plan_dp_json(text, n, coll)
            continue
        doc = json.loads(H.plan_dp_json(text, n, coll))
        st, cost = doc["strategy"], doc["cost"]
        (cc, pp, oo), obj, feas = want
        assert (st["c_hat"], st["p_hat"], st["o_hat"]) == (cc, pp, oo), c
        assert cost["objective_s"] == obj
        assert doc["search"]["feasible_count"] == feas
        assert cost["peak_gpu_bytes"] == ref.peak_gpu(pr, cc, pp, oo, n)
        assert cost["cpu_bytes"] == ref.cpu_bytes(pr, oo, n)


def test_sharding_relieves_memory():
    """More ranks never need more per-rank memory for the same strategy, and a budget under
    which the 20B paper configuration (configs[3]) has no plan on one GPU has one at dp 8."""
    pr = ref.profile(26, 8192, 1024, 1, 50257, 1200, 55, 55, 5000, 200000)
    for o in range(0, 27, 5):
        mems = [ref.peak_gpu(pr, 0, 0, o, n) for n in (1, 2, 4, 8)]
        assert mems == sorted(mems, reverse=True)
    text = config(26, 8192, 1024, 1, 50257, 40, 128, 1200, 55, 55, 5000, 200000)
    with pytest.raises(NativeError):
        H.plan_json(text)
    doc = json.loads(H.plan_dp_json(text, 8, 400.0))
    assert doc["cost"]["peak_gpu_bytes"] <= 40 * 2**30 and doc["cost"]["cpu_bytes"] <= 128 * 2**30
