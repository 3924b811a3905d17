"""A whole Llama-3.1-70B @32K session (80 x 2,048 blocks, 10.7 GB) migrated
through the store API on one B200: import_migration -> 80 NetArrive K3
pushes into the receiver's landing pool -> release -> layer-wise demand load,
free-running. Every one of the 163,840 pages the receiver ends with equals
the K5 fill of its (session, layer, block) tag, sampled pages equal the CPU
oracle, and the host bookkeeping of the migration itself (import_migration
posting every layer's K3 push) costs less per 2,048-block layer than the
NVLink transfer it schedules (128 MiB at the measured 770 GB/s: 174 us), so
a 70B migration is GPU-bound, not host-bound (VERDICT r01 "next" item 4;
driver in tools/store_path_70b.py)."""
import os
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_70b_session_migrates_bit_exact_through_the_store():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import store_path_70b
    r = store_path_70b.run(verify=True)
    assert r["mismatched_pages"] == 0 and r["verified_pages"] == 80 * 2048
    # host bookkeeping (store + payload, excluding GPU waits) per layer
    per_layer_nvlink_us = 128 * 2**20 / 770e9 * 1e6
    assert r["host_us_per_layer"]["import_migration"] < per_layer_nvlink_us, r["host_us_per_layer"]
    assert r["host_us_per_layer_migration_total"] < 400.0, r["host_us_per_layer"]
