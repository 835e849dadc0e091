"""bench.py's one-line JSON contract on the GPU (a short C1 run and the reference arm): the keys the driver reads,
their types and the invariants between them (value = elements / step time, the roofline fraction = achieved /
peak, gpu_launches = the per-step launch count x steps)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.timeout(900)
def test_bench_line_contract():
    d = run_bench("--config", "C1", "--steps", "5", "--warmup", "3", "--no-cpu")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["unit"] == "elements/s" and d["dtype"] == "f32" and d["vs_baseline"] is None
    T, D = d["config"]["T"], d["config"]["D"]
    assert (T, D) == (1024, 128) and "workload" in d["config"]
    assert d["value"] == pytest.approx(T * D / (d["ms_per_step"] * 1e-3), rel=1e-9)
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] >= T * D * 4 and e["d2h_bytes_per_step"] >= T * D
    assert d["gpu_launches"] > 0 and d["gpu_launches"] % d["steps"] == 0
    assert d["clocks"]["sm_max_mhz"] > 0


@pytest.mark.timeout(900)
def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "elements/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
