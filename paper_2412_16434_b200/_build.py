"""Build helpers: compile the in-tree product libraries (and, for tests, the
oracle) with make. The .so files land in-tree so they travel to the GPU box.

Product: paper_2412_16434_b200/lib/libkvx.so (sm_100a kernels, include/kvx.h)
         paper_2412_16434_b200/lib/libsymsim_b200.so (host store, include/kvs.h)
"""
from __future__ import annotations

import contextlib
import fcntl
import os
import shutil
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
ROOT = PKG_DIR.parent
LIB_DIR = PKG_DIR / "lib"
CSRC = PKG_DIR / "csrc"
ORACLE_DIR = ROOT / "oracle"

KVX_LIB = LIB_DIR / "libkvx.so"
HOST_LIB = LIB_DIR / "libsymsim_b200.so"


def _jobs() -> str:
    return str(max(1, min(16, os.cpu_count() or 1)))


@contextlib.contextmanager
def _build_lock():
    """One build at a time across processes (pytest-xdist workers share the
    build tree and the overlay headers)."""
    (ROOT / "build").mkdir(exist_ok=True)
    with open(ROOT / "build" / ".lock", "w") as fh:
        fcntl.flock(fh, fcntl.LOCK_EX)
        try:
            yield
        finally:
            fcntl.flock(fh, fcntl.LOCK_UN)


def _make(directory: Path, *targets: str) -> None:
    if shutil.which("make") is None:
        raise RuntimeError("make is required to build the B200 libraries")
    cmd = ["make", "-s", "-j", _jobs(), "-C", str(directory), *targets]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")


def build_product() -> None:
    """Compile every CUDA/C++ product source for sm_100a (idempotent)."""
    with _build_lock():
        _make(CSRC, "all")


def build_oracle(ref: bool = True) -> None:
    """Compile the oracle's C restatement, and the reference oracle when the
    reference sources are present (they are not on the GPU box, which uses the
    prebuilt oracle/_ref files)."""
    with _build_lock():
        _make(ORACLE_DIR, "payload")
    ref_src = Path(os.environ.get("REF", "/root/reference/proj")) / "src" / "kvstore.cpp"
    if ref and ref_src.exists():
        with _build_lock():
            _make(ORACLE_DIR, "ref")
        for name in ("build_payload_sim.sh", "build_serve_sim.sh", "build_serve_gpu.sh"):
            script = ROOT / "tests" / "cpp" / name  # takes build/.lock itself
            proc = subprocess.run(["bash", str(script)], capture_output=True, text=True)
            if proc.returncode != 0:
                raise RuntimeError(f"build failed: {script}\n{proc.stdout}\n{proc.stderr}")


def ensure_built() -> None:
    if not (KVX_LIB.exists() and HOST_LIB.exists()):
        build_product()
