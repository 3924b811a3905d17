"""bench.py's JSON line keeps the driver's contract (keys and units), for the
reference arm on CPU and for the B200 arm on a GPU."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _baseline_metric():
    return json.loads((ROOT / "BASELINE.json").read_text())["metric"]


def _run(args, timeout=900):
    proc = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT, env={**os.environ, "OMP_NUM_THREADS": "4"})
    assert proc.returncode == 0, proc.stderr[-3000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout
    return json.loads(lines[0])


def test_reference_arm_contract(product_libs):
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"])
    assert BASE_KEYS <= d.keys() and d["impl"] == "reference" and d["metric"] == _baseline_metric()
    assert d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True and d["warmup"] >= 3
    assert d["config"]["workload"] and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["cpu_baseline"]["cores"] >= 1 and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_b200_arm_contract():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--steps", "5", "--warmup", "3", "--skip-attention", "--skip-overlap", "--skip-cpu"])
    assert BASE_KEYS <= d.keys() and d["n_gpus"] == 1 and d["scaling"] == "weak"
    assert d["metric"] == _baseline_metric()
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0.5 < r["frac"] < 1.3 and r["traffic"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["clocks"]
    assert c["sm_max_mhz"] and not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(c["reasons"])
    assert d["gpu_launches"] == 2 * 5
