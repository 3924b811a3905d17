"""State parity at serving scale: configs 4 and 5.

The reference's unchanged cluster simulator runs the ShareGPT-like trace
(1,000 sessions, Poisson turns, advisories, 8 nodes; config 4) and the Zipf
1.2 load-imbalance trace (config 5) once on this repo's KvStore
(oracle/_ref/serve_sim) and once on the reference KvStore
(oracle/_ref/serve_sim_ref); the whole transfer ledger (millions of rows)
and every request record must hash identically.
"""
import subprocess

import pytest

from conftest import ROOT

BUILD = ROOT / "tests" / "cpp" / "build_serve_sim.sh"
PROD = ROOT / "oracle" / "_ref" / "serve_sim"
REF = ROOT / "oracle" / "_ref" / "serve_sim_ref"

CELLS = [
    ("4", "symphony", "64", "0"),
    ("4", "symphony", "256", "0.1"),
    ("4", "swap", "128", "0"),
    ("4", "recompute", "128", "0"),
    ("5", "symphony", "128", "0.1"),
    ("5", "retain", "64", "0"),
]


@pytest.fixture(scope="module")
def binaries(reference_present):
    subprocess.run(["bash", str(BUILD)], check=True, capture_output=True, timeout=900)
    return PROD, REF


@pytest.mark.parametrize("config,policy,users,miss", CELLS)
def test_serving_trace_ledger_matches_reference(binaries, config, policy, users, miss):
    prod, ref = binaries
    a = subprocess.run([str(prod), "digest", config, policy, users, miss], capture_output=True, text=True,
                       timeout=600, check=True).stdout.strip()
    b = subprocess.run([str(ref), "digest", config, policy, users, miss], capture_output=True, text=True,
                       timeout=600, check=True).stdout.strip()
    assert a == b
    fields = dict(zip(a.split()[0::2], a.split()[1::2]))
    assert int(fields["transfers"]) > 0 or policy in ("retain", "recompute")
    if policy == "symphony":
        assert int(fields["migrate_bytes"]) > 0
