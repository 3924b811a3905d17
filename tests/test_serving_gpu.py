"""The serving engine with every quantum executed on the B200 (SURVEY.md §8a
row a14, configs 4/5 shape at test scale): the reference's unchanged
Simulation drives this repo's KvStore + NodePayload + Engine, whose decode
steps run the Llama-3.1-8B-shaped step (K4 over the pages the payload holds)
and last their measured time (oracle/_ref/serve_gpu, tests/cpp/serve_gpu.cpp).
Every decode step's attended pages are scrubbed against their oracle content
(--verify-every 1): migrated, reloaded and appended caches are consumed
bit-exact. Each policy completes every turn of the trace."""
import json
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = ROOT / "oracle" / "_ref" / "serve_gpu"


def test_gpu_executed_serving_consumes_bit_exact_caches(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not BIN.exists():
        pytest.skip("serve_gpu not built (tests/cpp/build_serve_gpu.sh needs /root/reference)")
    cmd = [str(BIN), "--config", "5", "--policies", "symphony,swap,recompute", "--users", "12", "--sessions", "16",
           "--nodes", "2", "--device-gb", "8", "--host-gb", "8", "--verify-every", "1", "--disk-dir", str(tmp_path)]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    lines = [json.loads(ln) for ln in proc.stdout.splitlines() if ln.startswith("{")]
    cal = lines[0]["calibration"]
    assert len(cal["decode_curve_ms"]) == 7 and all(ms > 0 for _, ms in cal["decode_curve_ms"])
    cells = {c["policy"]: c for c in lines[1:]}
    assert set(cells) == {"symphony", "swap", "recompute"}, lines
    requests = {p: c.get("requests") for p, c in cells.items()}
    assert len(set(requests.values())) == 1 and next(iter(requests.values())) > 0, cells  # every turn served
    for p, c in cells.items():
        assert "error" not in c, c
        assert c["executed"]["decode_steps"] > 0 and c["executed"]["decode_ms_mean"] > 0
        assert c["verify"]["pages"] > 0 and c["verify"]["mismatched"] == 0, (p, c["verify"])
    assert cells["symphony"]["migrations"]["bytes"] > 0
    assert cells["symphony"]["migrations"]["net_arrive_bytes_moved"] == cells["symphony"]["migrations"]["bytes"]
