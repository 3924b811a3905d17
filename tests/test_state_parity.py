"""Block-table state parity: the B200 build's KvStore vs the reference KvStore.

The oracle is the reference store itself (proj/src/kvstore.cpp +
costmodel.cpp compiled from /root/reference into oracle/_ref, namespace
renamed). Parity is bit-exact: statuses and exception messages, transfer ids
and completion times, ledger rows, counters, per-session state and eviction
order must be identical after every call.
"""
import subprocess
from pathlib import Path

import pytest

from conftest import ROOT

pytestmark = pytest.mark.timeout(600) if hasattr(pytest.mark, "timeout") else []

DIFF_SRC = ROOT / "tests" / "cpp" / "diff_kvstore.cpp"
DIFF_BIN = ROOT / "build" / "tests" / "diff_kvstore"


@pytest.fixture(scope="module")
def diff_binary():
    DIFF_BIN.parent.mkdir(parents=True, exist_ok=True)
    deps = [DIFF_SRC, ROOT / "tests/cpp/kvs_dyn.hpp", ROOT / "tests/cpp/kvs_fns.inc", ROOT / "include/kvs.h"]
    if not DIFF_BIN.exists() or any(d.stat().st_mtime > DIFF_BIN.stat().st_mtime for d in deps):
        subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"-I{ROOT}/tests/cpp", str(DIFF_SRC),
                        "-ldl", "-o", str(DIFF_BIN)], check=True)
    return DIFF_BIN


@pytest.mark.parametrize("seed,cases,ops", [(20260417, 3000, 80), (7, 1500, 200), (99, 4000, 30)])
def test_randomized_differential(diff_binary, product_libs, oracle_ref_lib, seed, cases, ops):
    proc = subprocess.run([str(diff_binary), str(product_libs.HOST_LIB), oracle_ref_lib, str(cases), str(ops),
                           str(seed)], capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stdout + proc.stderr[-4000:]
    assert "0 mismatches" in proc.stdout


def _stores(oracle_ref_lib, **opts):
    from paper_2412_16434_b200 import kvstore as K
    o = K.Options(**opts)
    return K.KvStore(opts=o), K.KvStore(opts=o, lib=oracle_ref_lib)


def _pump(store, sched):
    out = []
    for tid, at in sorted(sched, key=lambda t: (t[1], t[0])):
        out.append(store.apply_transfer(tid, at))
    return out


KBLOCK = 550_000


def test_migration_import_known_answers(product_libs, oracle_ref_lib):
    """reference test_kvstore.cpp:350-383: per-layer arrivals at 1 ms + 54 us * (l+1)."""
    for store in _stores(oracle_ref_lib):
        store.register_session(7, "mig")
        store.finalize_sessions()
        sched = store.import_migration(7, 16, 1_000_000)
        assert len(sched) == 64
        assert store.host_used() == 32 * KBLOCK
        for l in range(32):
            assert sched[2 * l][1] == 1_000_000 + 54_000 * (l + 1)
        res = _pump(store, sched)
        assert sum(r.migration_arrived for r in res) == 32
        assert sum(r.migration_complete for r in res) == 1
        assert store.pending_persists(7) == 0
        store.check_budgets()


def test_layerwise_load_known_answers(product_libs, oracle_ref_lib):
    """reference test_kvstore.cpp:430-458: demand load lands layer l at t + 32 us * (l+1)."""
    from paper_2412_16434_b200 import kvstore as K
    at = 50_000_000
    plans = []
    for store in _stores(oracle_ref_lib):
        store.register_session(3, "p")
        store.finalize_sessions()
        _pump(store, store.import_migration(3, 16, 0))
        plan, sched = store.plan_layerwise_load(3, at, 400_000, K.DEMAND)
        assert plan.layer_ready == [at + 32_000 * (l + 1) for l in range(32)]
        assert plan.finish == K.pipeline_gate(plan.layer_ready, at, 32 * 400_000)[0]
        _pump(store, sched)
        assert store.fully_device_resident(3)
        plans.append((plan, store.ledger()))
    assert plans[0] == plans[1]


def test_error_behaviour_matches(product_libs, oracle_ref_lib):
    from paper_2412_16434_b200 import kvstore as K
    for store in _stores(oracle_ref_lib, device_capacity=1000):
        store.reserve_device(600)
        with pytest.raises(K.KvsLogicError, match="overflows capacity"):
            store.reserve_device(500)
        with pytest.raises(K.KvsLogicError, match="bad unreserve"):
            store.unreserve_device(700)
        with pytest.raises(K.KvsLogicError, match="unknown session"):
            store.append_blocks(99, 16, 0)
        store.register_session(1, "x")
        with pytest.raises(K.KvsLogicError, match="token count must be positive"):
            store.append_blocks(1, 0, 0)


def test_library_exports_every_declared_symbol(product_libs):
    import ctypes
    import re
    decl = (ROOT / "include" / "kvs.h").read_text()
    names = re.findall(r"^\s*(?:int|void|size_t|const char\*)\s+(kvs_\w+)\(", decl, re.M)
    assert len(names) >= 40
    lib = ctypes.CDLL(str(product_libs.HOST_LIB))
    for n in names:
        assert hasattr(lib, n), n
