"""Shared test fixtures.

Markers: `gpu` — needs a CUDA device (run on the B200 box with -m gpu).
Everything else runs on CPU (-m "not gpu").
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

REF = Path(os.environ.get("REF", "/root/reference/proj"))
ORACLE_REF_LIB = ROOT / "oracle" / "_ref" / "libsymsim_oracle.so"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def product_libs():
    from paper_2412_16434_b200 import _build
    _build.build_product()
    return _build


@pytest.fixture(scope="session")
def oracle_ref_lib(product_libs):
    """Path to the reference KvStore compiled as the oracle; skip without it."""
    from paper_2412_16434_b200 import _build
    _build.build_oracle(ref=True)
    if not ORACLE_REF_LIB.exists():
        pytest.skip("oracle/_ref not built (reference sources absent and no prebuilt copy)")
    return str(ORACLE_REF_LIB)


@pytest.fixture(scope="session")
def reference_present():
    if not (REF / "src" / "kvstore.cpp").exists():
        pytest.skip("reference sources not present (GPU box)")
    return REF


def run(cmd, **kw):
    return subprocess.run(cmd, capture_output=True, text=True, **kw)
