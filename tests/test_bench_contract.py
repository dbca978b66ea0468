"""bench.py keeps the driver's JSON-line contract: the reference arm on CPU (here), the
product arm on a B200 (gpu marker)."""
import json
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "3")
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "tokens/s" and d["warmup"] >= 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_product_arm_contract(cuda_device, native):
    d = run_bench("--config", "tiny", "--steps", "3", "--warmup", "3")
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["scaling"] == "weak" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1.5 and r["peak"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["cpu_baseline"]["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["adam"]["roofline"]["bound"] == "hbm"
    m = d["memory"]  # the executor's transient buffers come from its arenas: nothing allocated on the fly
    assert m["buffer_overflows"] == 0 and m["measured_peak_gib"] <= m["eq1_gib"] * 1.1


def test_bench_spawns_ranks():
    """`bench.py --gpus 2` outside a torch.distributed launcher spawns 2 ranks itself (the
    driver may call it either way); each rank checks WORLD_SIZE == --gpus (gloo here)."""
    d = run_bench("--gpus", "2", "--launch-check", timeout=300)
    assert d["launch_check"] and d["world"] == 2
    assert sorted(r["rank"] for r in d["ranks"]) == [0, 1]
    assert len({r["pid"] for r in d["ranks"]}) == 2
