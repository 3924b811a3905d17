"""Symphony (arXiv 2412.16434) KV-migration hot path, built B200-native.

Host state machine: symsim::KvStore (C++; include/symsim/kvstore.hpp, C ABI
include/kvs.h, Python mirror `kvstore`). Device payload: sm_100a kernels for
page pack/unpack/migrate, KV append/fill and paged decode attention (C ABI
include/kvx.h, Python wrapper `kvx`). See DESIGN.md.
"""
from . import _build  # noqa: F401

__all__ = ["kvstore", "kvx"]
