"""The N>1 migration path of bench.py, exercised with two ranks on the one
available GPU: real CUDA IPC between two processes, the K3 kernel storing
into the peer process's page pool, max-over-ranks timing, and the receivers'
bit-exact check of what landed. (On an 8-GPU box the same code runs one rank
per GPU with NCCL as the control plane; here the control plane is gloo.)"""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["p2p", "nccl", "p2p-refused"])
def test_two_process_migration_plus_serving_on_one_gpu(mode):
    """p2p: K3 stores into the peer process's pool (IPC). nccl: the
    comparison path (pack, send/recv, unpack) — here over gloo with host
    staging, since NCCL refuses two ranks on one GPU. Both run a decode batch
    beside the migration and verify what landed bit for bit. p2p-refused: one
    rank cannot open its peer's pool, so both agree to migrate over the
    collective path instead and the line says why."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--same-device", "--dist-backend", "gloo", "--layers", "2", "--path", "kvx",
           "--migrate-mode", mode.split("-")[0],
           "--serve-batch", "2"]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                          env={**os.environ, "OMP_NUM_THREADS": "1",
                               **({"BENCH_FAIL_IPC_RANK": "1"} if mode == "p2p-refused" else {})})
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-5000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout
    res = json.loads(lines[0])
    assert res["n_gpus"] == 2 and res["value"] > 0
    assert res["roofline"]["bound"] == "nvlink"
    if mode == "p2p-refused":
        assert res["config"]["migrate_mode"] == "nccl" and "rank 1" in res["config"]["p2p_unavailable"]
        mode = "nccl"
    assert res["config"]["layers"] == 2 and res["config"]["migrate_mode"] == mode
    sv = res["serving"]
    assert sv["decode_steps_per_migration"] >= 1 and sv["decode_step_ms_alone"] > 0
    if mode == "p2p":
        assert res["e2e"]["value"] > 0 and res["e2e"]["h2d_bytes_per_step"] > 0


def test_store_path_ring_through_the_store_api():
    """The default N>1 path: every session migrates one hop around the ring
    per step through the store API (mark_migrating_out -> import_migration ->
    NetArrive applies -> release) with real pages; here both nodes sit on the
    one GPU (--same-device). Probe pages of every session are checked
    against the CPU oracle after the timed steps."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--same-device", "--dist-backend", "gloo", "--layers", "4", "--path", "store"]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                          env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-5000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout
    res = json.loads(lines[0])
    assert res["n_gpus"] == 2 and res["value"] > 0 and res["config"]["path"] == "store"
    assert res["store_path"]["probe_pages_checked"] == 8 and res["store_path"]["devices"] == 1
    assert res["gpu_launches"] >= 3 * 2 * 4  # >= one K3 push per layer per session per step
    assert res["e2e"]["value"] > 0
