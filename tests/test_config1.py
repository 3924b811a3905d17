"""Config 1 (tiny Llama-style KV, 8 sessions x 4 turns, 2 nodes) end to end.

The reference's own cluster simulator (Simulation, Engine, NodeManager,
ClusterScheduler — unchanged, compiled from /root/reference into
oracle/_ref/payload_sim by tests/cpp/build_payload_sim.sh) drives this repo's
KvStore with a NodePayload behind every node, so every append, write-behind
persist, purge, load, advisory promotion and node-to-node migration of the
trace moves real pages on the GPU.

Gates:
  * the full transfer ledger and every request record equal the reference
    KvStore's run of the same trace (golden fixtures tests/golden/config1_*.txt,
    made by tests/golden/make_config1_golden.sh from oracle/_ref/payload_sim_ref);
  * every physical copy of every block on both nodes is bit-exact against the
    CPU restatement's content for its (session, layer, block), and every page
    in use is accounted for by a residency bit ("mismatches 0").
"""
import subprocess

import pytest

from conftest import ROOT

REF_BIN = ROOT / "oracle" / "_ref" / "payload_sim_ref"
PROD_BIN = ROOT / "oracle" / "_ref" / "payload_sim"
GOLDEN = ROOT / "tests" / "golden"

VARIANTS = {
    "default": [],
    "dev30": ["--device-pages", "30"],
    "dev40": ["--device-pages", "40"],
    "swap": ["--policy", "swap"],
}
MODES = {"lockstep": [], "free-running": ["--free-running"]}


def _state_lines(text):
    return [ln for ln in text.splitlines() if ln.startswith(("T ", "R ", "policy ", "migrate_rows"))]


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_golden_matches_reference_store(reference_present, variant):
    """The committed fixtures are what the reference store produces (CPU)."""
    subprocess.run(["bash", str(ROOT / "tests/cpp/build_payload_sim.sh")], check=True, capture_output=True)
    out = subprocess.run([str(REF_BIN), *VARIANTS[variant]], capture_output=True, text=True, check=True).stdout
    assert _state_lines(out) == _state_lines((GOLDEN / f"config1_{variant}.txt").read_text())


def test_golden_has_migrations_and_purges():
    text = (GOLDEN / "config1_default.txt").read_text()
    assert int(text.split("migrate_rows ")[1].split()[0]) > 0
    assert " purge" in (GOLDEN / "config1_dev30.txt").read_text()
    assert "device>host" in (GOLDEN / "config1_swap.txt").read_text()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("variant", list(VARIANTS))
def test_config1_trace_with_real_pages(variant, mode):
    if not PROD_BIN.exists():
        pytest.skip("oracle/_ref/payload_sim not built (needs the reference sources; build here and ship)")
    proc = subprocess.run([str(PROD_BIN), *VARIANTS[variant], *MODES[mode]], capture_output=True, text=True,
                          timeout=600)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    assert _state_lines(proc.stdout) == _state_lines((GOLDEN / f"config1_{variant}.txt").read_text())
    summary = [ln for ln in proc.stdout.splitlines() if ln.startswith("payload verified_copies")][0]
    copies, bad = int(summary.split()[2]), int(summary.split()[4])
    assert copies > 0 and bad == 0, summary


@pytest.mark.gpu
@pytest.mark.parametrize("mode", list(MODES))
def test_config1_with_disk_tier_in_files(mode, tmp_path):
    """Same gates with the DISK tier backed by one file per node: every
    write-behind DiskWrite of the purge-heavy variant lands in the node's file
    (read back with pread for the bit-exact check)."""
    if not PROD_BIN.exists():
        pytest.skip("oracle/_ref/payload_sim not built (needs the reference sources; build here and ship)")
    proc = subprocess.run([str(PROD_BIN), *VARIANTS["dev30"], *MODES[mode], "--disk-dir", str(tmp_path)],
                          capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    assert _state_lines(proc.stdout) == _state_lines((GOLDEN / "config1_dev30.txt").read_text())
    summary = [ln for ln in proc.stdout.splitlines() if ln.startswith("payload verified_copies")][0]
    copies, bad = int(summary.split()[2]), int(summary.split()[4])
    assert copies > 0 and bad == 0, summary
    assert sorted(p.name for p in tmp_path.iterdir()) == ["node0.pages", "node1.pages"]
    disk_pages = [int(ln.split(" disk ")[1].split()[0]) for ln in proc.stdout.splitlines()
                  if ln.startswith("payload node") and " disk " in ln]
    assert sum(disk_pages) > 0, "the trace must leave DISK copies in the files"
