"""Configs 4 and 5's traffic through the reference's unchanged Simulation on
8 nodes, with real pages behind every node on the GPU (tiny KV shape so all
eight nodes' pools fit one B200; the store's DEVICE / HOST capacities equal
the pools behind them, 4,096 pages each, so cooperative purges happen):
  config 5: Zipf 1.2 popularity, 600 sessions, 300 fast users, advisories
            (113,428 ledger rows, 1,074 migrations, 1,342 requests);
  config 4: ShareGPT-like corpus, 400 sessions, 200 users, Poisson think
            (134,647 ledger rows, 1,840 migrations, 1,588 requests).

Gates: the ledger and request records hash identically to the reference
KvStore's run of the same trace (oracle/_ref/payload_sim_ref, CPU), and every
copy of every block on every node is bit-exact (read back and compared with
the CPU restatement's content for its (session, layer, block)), in both
payload modes."""
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

PROD = ROOT / "oracle" / "_ref" / "payload_sim"
REF = ROOT / "oracle" / "_ref" / "payload_sim_ref"
TRACES = {"config5-zipf": ["--zipf", "600", "--users", "300"], "config4-sharegpt": ["--sharegpt", "400", "--users", "200"]}
COMMON = ["--nodes", "8", "--pages", "4096", "--digest"]


def _digest(out):
    return [ln for ln in out.splitlines() if ln.startswith(("digest ", "policy ", "migrate_rows"))]


@pytest.mark.parametrize("mode", [[], ["--free-running"]], ids=["lockstep", "free-running"])
@pytest.mark.parametrize("trace", list(TRACES))
def test_serving_trace_with_real_pages(trace, mode):
    if not PROD.exists() or not REF.exists():
        pytest.skip("oracle/_ref/payload_sim* not built (needs the reference sources; build here and ship)")
    args = [*TRACES[trace], *COMMON]
    ref = subprocess.run([str(REF), *args], capture_output=True, text=True, timeout=600, check=True).stdout
    proc = subprocess.run([str(PROD), *args, *mode], capture_output=True, text=True, timeout=1200)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    assert _digest(proc.stdout) == _digest(ref)
    assert int(_digest(ref)[-1].split()[1]) > 500  # migrations happened
    summary = [ln for ln in proc.stdout.splitlines() if ln.startswith("payload verified_copies")][0]
    copies, bad = int(summary.split()[2]), int(summary.split()[4])
    assert copies > 10_000 and bad == 0, summary
