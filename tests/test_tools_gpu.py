"""The measurement tools keep working (they are what a multi-GPU round runs
first) and the C++ example host: the NVLink probe in its same-GPU self-test mode and the PCIe mover
probe, each verifying every variant bit-exact."""
import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _run(args):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    proc = subprocess.run([sys.executable, *args], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr[-3000:]
    return json.loads(proc.stdout.strip().splitlines()[-1])


def test_nvlink_probe_self_test():
    d = _run([str(ROOT / "tools" / "nvlink_probe.py"), "--peer", "0", "--pages", "1024"])
    movers = {v["mover"]: v for v in d["variants"]}
    assert {"sm/all", "tma", "copy-engines"} <= movers.keys()
    assert all(v.get("verified", False) for v in d["variants"] if "error" not in v)


def test_pcie_mover_probe():
    d = _run([str(ROOT / "tools" / "pcie_mover_probe.py"), "--pages", "1024"])
    assert len(d["variants"]) == 12
    assert all(v.get("verified", False) for v in d["variants"] if "error" not in v)
    assert len(d["bidirectional"]) == 6
    assert all(v.get("verified", False) for v in d["bidirectional"] if "error" not in v)


def test_cpp_example_host():
    """examples/decode_step.cpp drives migrate -> fused decode step through the
    C ABI alone (no Python, no CUDA headers) and checks fused == two-launch."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = ROOT / "examples" / "decode_step"
    if not exe.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "examples")], check=True, timeout=300)
    proc = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0, proc.stdout + proc.stderr
    assert "bit-identical" in proc.stdout and "identical" in proc.stdout
