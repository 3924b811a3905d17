"""Python mirror of the reference KvStore API over the kvs_* C ABI.

The reference store is C++ only (/root/reference/proj/include/symsim/
kvstore.hpp:107-229). This class keeps its method names, argument meaning and
error behaviour (std::logic_error -> KvsLogicError, std::runtime_error ->
KvsRuntimeError; a declined load plan returns None like std::nullopt), so
tests read like the reference's own (proj/tests/test_kvstore.cpp).

The same wrapper drives any library exporting include/kvs.h: the product
(paper_2412_16434_b200/lib/libsymsim_b200.so, the default) or — in tests
only — the reference oracle (oracle/_ref/libsymsim_oracle.so).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path
from typing import Dict, List, Optional, Sequence, Tuple

from . import _build

DEVICE, HOST, DISK = 0, 1, 2
TIER_NAMES = ("device", "host", "disk")
PREFETCH, DEMAND, PURGE, PERSIST, MIGRATE = range(5)
REASON_NAMES = ("prefetch", "demand", "purge", "persist", "migrate")
PCIE_H2D, PCIE_D2H, DISK_READ, DISK_WRITE, NETWORK = range(5)


class KvsError(Exception):
    pass


class KvsLogicError(KvsError):
    """std::logic_error raised by the store (contract violation)."""


class KvsRuntimeError(KvsError):
    """std::runtime_error raised by the store (resource or config failure)."""


class _Gpu(C.Structure):
    _fields_ = [("prefill_throughput", C.c_double), ("decode_base_ms", C.c_double),
                ("decode_half_batch", C.c_double), ("hbm_capacity", C.c_int64),
                ("kv_bytes_per_token", C.c_int64), ("num_layers", C.c_int32),
                ("curve_points", C.c_int32), ("curve_batch", C.POINTER(C.c_int32)),
                ("curve_ms", C.POINTER(C.c_double))]


class _Links(C.Structure):
    _fields_ = [("pcie_bandwidth", C.c_double), ("disk_bandwidth", C.c_double),
                ("network_bandwidth", C.c_double), ("per_transfer_latency", C.c_int64)]


class _Opts(C.Structure):
    _fields_ = [("node_id", C.c_int32), ("block_tokens", C.c_int32),
                ("device_capacity", C.c_int64), ("host_capacity", C.c_int64),
                ("disk_capacity", C.c_int64), ("write_behind", C.c_int32)]


class _Sched(C.Structure):
    _fields_ = [("id", C.c_uint64), ("complete_at", C.c_int64)]


class _Key(C.Structure):
    _fields_ = [("session", C.c_uint32), ("layer", C.c_uint16), ("pad_", C.c_uint16),
                ("block_index", C.c_uint32)]


class _Record(C.Structure):
    _fields_ = [("time", C.c_int64), ("node", C.c_int32), ("session", C.c_uint32),
                ("layer_lo", C.c_uint16), ("layer_hi", C.c_uint16), ("from_", C.c_int32),
                ("to", C.c_int32), ("reason", C.c_int32), ("bytes", C.c_int64)]


class _Apply(C.Structure):
    _fields_ = [("session", C.c_uint32), ("layer", C.c_uint16), ("device_layer_ready", C.c_uint8),
                ("persists_drained", C.c_uint8), ("migration_arrived", C.c_uint8),
                ("migration_complete", C.c_uint8), ("voided", C.c_uint8), ("pad_", C.c_uint8)]


class _Plan(C.Structure):
    _fields_ = [("has_plan", C.c_int32), ("any_load", C.c_int32), ("decode_start", C.c_int64),
                ("finish", C.c_int64), ("total_stall", C.c_int64)]


class _Promote(C.Structure):
    _fields_ = [("device_layers", C.c_int32), ("staged_layers", C.c_int32), ("scheduled", C.c_int32)]


class _Gate(C.Structure):
    _fields_ = [("first_step_end", C.c_int64), ("gate_start", C.c_int64), ("stall", C.c_int64)]


class _Counters(C.Structure):
    _fields_ = [("device_capacity", C.c_int64), ("device_used", C.c_int64), ("device_free", C.c_int64),
                ("host_used", C.c_int64), ("disk_used", C.c_int64), ("layer_block_bytes", C.c_int64)]


class _SessionInfo(C.Structure):
    _fields_ = [("cached_tokens", C.c_int64), ("session_bytes", C.c_int64),
                ("fully_device_resident", C.c_int32), ("has_any_copy", C.c_int32),
                ("pending_persists", C.c_int32), ("migrating_out", C.c_int32),
                ("is_active", C.c_int32), ("pad_", C.c_int32)]


class _Meta(C.Structure):
    _fields_ = [("key", _Key), ("session_bytes", C.c_int64), ("session_id", C.c_char_p),
                ("pinned", C.c_int32), ("pad_", C.c_int32)]


class _PayloadOpts(C.Structure):
    _fields_ = [("device", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("block_tokens", C.c_int32), ("dtype", C.c_int32), ("fill_mode", C.c_int32),
                ("device_pages", C.c_uint64), ("host_pages", C.c_uint64), ("landing_pages", C.c_uint64),
                ("disk_pages", C.c_uint64), ("seed", C.c_uint64), ("free_running", C.c_int32),
                ("pad_", C.c_int32), ("disk_path", C.c_char_p), ("migrate_max_ctas", C.c_uint32),
                ("pad2_", C.c_uint32)]


@dataclass
class GpuProfile:
    """reference costmodel.hpp:17-27 (same defaults)."""
    prefill_throughput: float = 8192.0
    decode_base_ms: float = 12.0
    decode_half_batch: float = 16.0
    hbm_capacity: int = 80_000_000_000
    kv_bytes_per_token: int = 1_100_000
    num_layers: int = 32
    decode_curve_ms: List[Tuple[int, float]] = field(default_factory=list)

    def _c(self) -> Tuple[_Gpu, tuple]:
        n = len(self.decode_curve_ms)
        b = (C.c_int32 * max(n, 1))(*[p[0] for p in self.decode_curve_ms])
        m = (C.c_double * max(n, 1))(*[p[1] for p in self.decode_curve_ms])
        g = _Gpu(self.prefill_throughput, self.decode_base_ms, self.decode_half_batch, self.hbm_capacity,
                 self.kv_bytes_per_token, self.num_layers, n, b, m)
        return g, (b, m)


@dataclass
class LinkProfile:
    """reference costmodel.hpp:29-36 (same defaults)."""
    pcie_bandwidth: float = 25e9
    disk_bandwidth: float = 3e9
    network_bandwidth: float = 12.5e9
    per_transfer_latency: int = 10_000

    def _c(self) -> _Links:
        return _Links(self.pcie_bandwidth, self.disk_bandwidth, self.network_bandwidth,
                      self.per_transfer_latency)


@dataclass
class Options:
    """KvStore::Options, reference kvstore.hpp:109-116."""
    node_id: int = 0
    block_tokens: int = 16
    device_capacity: int = 0
    host_capacity: int = 256_000_000_000
    disk_capacity: int = -1
    write_behind: bool = True

    def _c(self) -> _Opts:
        return _Opts(self.node_id, self.block_tokens, self.device_capacity, self.host_capacity,
                     self.disk_capacity, int(self.write_behind))


@dataclass(frozen=True)
class TransferRecord:
    time: int
    node: int
    session: int
    layer_lo: int
    layer_hi: int
    from_tier: int
    to_tier: int
    bytes: int
    reason: int


@dataclass
class LoadPlan:
    layer_ready: List[int]
    decode_start: int
    finish: int
    total_stall: int
    any_load: bool


@dataclass(slots=True)
class ApplyResult:
    session: int
    layer: int
    device_layer_ready: bool
    persists_drained: bool
    migration_arrived: bool
    migration_complete: bool
    voided: bool


@dataclass
class BlockMeta:
    session: int
    layer: int
    block_index: int
    session_id: str
    session_bytes: int
    pinned: bool = False


_LIBS: Dict[str, C.CDLL] = {}


def load_kvs_library(path: Optional[str] = None) -> C.CDLL:
    """Load a kvs_* library (default: the product build, built on demand)."""
    if path is None:
        _build.ensure_built()
        path = str(_build.HOST_LIB)
    path = str(Path(path).resolve())
    if path in _LIBS:
        return _LIBS[path]
    lib = C.CDLL(path, mode=C.RTLD_LOCAL)
    P = C.POINTER
    sigs = {
        "kvs_last_error": ([], C.c_char_p),
        "kvs_is_product": ([], C.c_int),
        "kvs_create": ([P(_Gpu), P(_Links), P(_Opts), P(C.c_void_p)], C.c_int),
        "kvs_destroy": ([C.c_void_p], None),
        "kvs_register_session": ([C.c_void_p, C.c_uint32, C.c_char_p, C.c_int32], C.c_int),
        "kvs_finalize_sessions": ([C.c_void_p], C.c_int),
        "kvs_get_counters": ([C.c_void_p, P(_Counters)], C.c_int),
        "kvs_get_session": ([C.c_void_p, C.c_uint32, P(_SessionInfo)], C.c_int),
        "kvs_bytes_for_new_blocks": ([C.c_void_p, C.c_uint32, C.c_int64, P(C.c_int64)], C.c_int),
        "kvs_bytes_for_load": ([C.c_void_p, C.c_uint32, P(C.c_int64)], C.c_int),
        "kvs_bytes_for_promote": ([C.c_void_p, C.c_uint32, P(C.c_int64)], C.c_int),
        "kvs_reserve_device": ([C.c_void_p, C.c_int64], C.c_int),
        "kvs_unreserve_device": ([C.c_void_p, C.c_int64], C.c_int),
        "kvs_set_active": ([C.c_void_p, C.c_uint32, C.c_int32, C.c_int64], C.c_int),
        "kvs_append_blocks": ([C.c_void_p, C.c_uint32, C.c_int64, C.c_int64], C.c_int),
        "kvs_purge_from_device": ([C.c_void_p, C.c_int64, C.c_int64, C.c_int32, P(C.c_int64)], C.c_int),
        "kvs_plan_layerwise_load": ([C.c_void_p, C.c_uint32, C.c_int64, C.c_int64, C.c_int32, P(_Plan)], C.c_int),
        "kvs_promote": ([C.c_void_p, C.c_uint32, C.c_int64, P(_Promote)], C.c_int),
        "kvs_offload_session": ([C.c_void_p, C.c_uint32, C.c_int64], C.c_int),
        "kvs_release_session": ([C.c_void_p, C.c_uint32, C.c_int64], C.c_int),
        "kvs_mark_migrating_out": ([C.c_void_p, C.c_uint32], C.c_int),
        "kvs_import_migration": ([C.c_void_p, C.c_uint32, C.c_int64, C.c_int64], C.c_int),
        "kvs_apply_transfer": ([C.c_void_p, C.c_uint64, C.c_int64, P(_Apply)], C.c_int),
        "kvs_void_session_loads": ([C.c_void_p, C.c_uint32], C.c_int),
        "kvs_void_session_offload": ([C.c_void_p, C.c_uint32], C.c_int),
        "kvs_evictable_blocks": ([C.c_void_p, C.c_int32], C.c_int),
        "kvs_check_budgets": ([C.c_void_p], C.c_int),
        "kvs_device_usage_debug": ([C.c_void_p, C.c_char_p, C.c_size_t], C.c_int),
        "kvs_ledger_size": ([C.c_void_p], C.c_size_t),
        "kvs_ledger_copy": ([C.c_void_p, C.c_size_t, C.c_size_t, P(_Record)], C.c_int),
        "kvs_out_scheduled": ([C.c_void_p, P(P(_Sched))], C.c_size_t),
        "kvs_out_keys": ([C.c_void_p, P(P(_Key))], C.c_size_t),
        "kvs_out_times": ([C.c_void_p, P(P(C.c_int64))], C.c_size_t),
        "kvs_out_metas": ([C.c_void_p, P(P(_Meta))], C.c_size_t),
        "kvs_evict_order": ([P(_Meta), C.c_size_t, P(C.c_uint32)], C.c_int),
        "kvs_pipeline_gate": ([P(C.c_int64), C.c_size_t, C.c_int64, C.c_int64, P(_Gate)], C.c_int),
        "kvs_transfer_time": ([C.c_int64, C.c_int32, P(_Links), P(C.c_int64)], C.c_int),
        "kvs_decode_step_time": ([C.c_int32, P(_Gpu), P(C.c_int64)], C.c_int),
        "kvs_prefill_time": ([C.c_int64, P(_Gpu), P(C.c_int64)], C.c_int),
        "kvs_kv_bytes_per_layer": ([C.c_int64, P(_Gpu), P(C.c_int64)], C.c_int),
        "kvs_residency": ([C.c_void_p, C.c_uint32, C.c_uint16, C.c_uint32, P(C.c_uint8)], C.c_int),
        "kvs_cluster_create": ([P(C.c_void_p)], C.c_int),
        "kvs_cluster_destroy": ([C.c_void_p], None),
        "kvs_payload_create": ([C.c_void_p, C.c_int32, P(_PayloadOpts), P(C.c_void_p)], C.c_int),
        "kvs_payload_destroy": ([C.c_void_p], None),
        "kvs_attach_payload": ([C.c_void_p, C.c_void_p], C.c_int),
        "kvs_payload_read_block": ([C.c_void_p, C.c_uint32, C.c_uint16, C.c_uint32, C.c_int32, C.c_void_p], C.c_int),
        "kvs_payload_pages_in_use": ([C.c_void_p, C.c_int32, P(C.c_uint64)], C.c_int),
        "kvs_payload_pool_of": ([C.c_void_p, C.c_uint32, C.c_uint16, C.c_uint32, C.c_int32, P(C.c_int32)], C.c_int),
        "kvs_payload_bytes_moved": ([C.c_void_p, P(C.c_uint64)], C.c_int),
        "kvs_payload_stats": ([C.c_void_p, P(C.c_uint64)], C.c_int),
        "kvs_payload_host_ns": ([C.c_void_p, P(C.c_uint64)], C.c_int),
        "kvs_payload_block_table": ([C.c_void_p, C.c_uint32, C.c_uint16, C.c_uint32, P(C.c_uint32)], C.c_int),
        "kvs_payload_pool": ([C.c_void_p, C.c_int32, P(C.c_void_p)], C.c_int),
        "kvs_payload_synchronize": ([C.c_void_p], C.c_int),
        "kvs_payload_stream": ([C.c_void_p, C.c_int32, P(C.c_void_p)], C.c_int),
        "kvs_set_default_payload": ([C.c_void_p, P(_PayloadOpts), C.c_int32], C.c_int),
        "kvs_cluster_node": ([C.c_void_p, C.c_int32, P(C.c_void_p)], C.c_int),
        "kvs_traffic_zipf_turns": ([C.c_uint64, C.c_double, C.c_double, C.c_int32, C.c_uint64, P(C.c_int32)], C.c_int),
        "kvs_traffic_poisson_gaps": ([C.c_uint64, C.c_double, C.c_uint64, P(C.c_int64)], C.c_int),
        "kvs_traffic_percentile": ([P(C.c_double), C.c_uint64, C.c_double, P(C.c_double)], C.c_int),
        "kvs_traffic_rps_within_slo": ([P(C.c_int32), P(C.c_double), P(C.c_double), C.c_uint64, C.c_double,
                                        P(C.c_double)], C.c_int),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _LIBS[path] = lib
    return lib


def _check(lib: C.CDLL, rc: int) -> None:
    if rc == 0:
        return
    msg = (lib.kvs_last_error() or b"").decode()
    if rc == 1:
        raise KvsLogicError(msg)
    if rc == 2:
        raise KvsRuntimeError(msg)
    raise KvsError(msg)


class KvStore:
    """One node's tiered store; method-for-method the reference KvStore."""

    def __init__(self, gpu: Optional[GpuProfile] = None, links: Optional[LinkProfile] = None,
                 opts: Optional[Options] = None, lib: Optional[str] = None):
        self._lib = load_kvs_library(lib)
        self.gpu = gpu or GpuProfile()
        self.links = links or LinkProfile()
        self.opts = opts or Options()
        g, keep = self.gpu._c()
        handle = C.c_void_p()
        _check(self._lib, self._lib.kvs_create(C.byref(g), C.byref(self.links._c()), C.byref(self.opts._c()),
                                               C.byref(handle)))
        self._h = handle
        # Hot per-transfer call: bound once, result struct reused (ctypes
        # attribute lookup + struct allocation per apply cost more host time
        # than the store's own bookkeeping).
        self._apply_fn = self._lib.kvs_apply_transfer
        self._apply_buf = _Apply()
        self._apply_ref = C.byref(self._apply_buf)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.kvs_destroy(h)
            self._h = None

    # ---- internals ----
    def _call(self, name: str, *args) -> None:
        _check(self._lib, getattr(self._lib, name)(self._h, *args))

    def _scheduled(self) -> List[Tuple[int, int]]:
        p = C.POINTER(_Sched)()
        n = self._lib.kvs_out_scheduled(self._h, C.byref(p))
        if n <= 0:
            return []
        # One bulk read of the (id u64, complete_at i64) pairs instead of a
        # struct object per element.
        addr = C.addressof(p.contents)
        ids = (C.c_uint64 * (2 * n)).from_address(addr)[0::2]
        at = (C.c_int64 * (2 * n)).from_address(addr)[1::2]
        return list(zip(ids, at))

    # ---- registry ----
    def register_session(self, session: int, sid: str, high_priority: bool = False) -> None:
        self._call("kvs_register_session", session, sid.encode(), int(high_priority))

    def finalize_sessions(self) -> None:
        self._call("kvs_finalize_sessions")

    # ---- capacity ----
    def counters(self) -> _Counters:
        c = _Counters()
        self._call("kvs_get_counters", C.byref(c))
        return c

    def device_capacity(self) -> int:
        return self.counters().device_capacity

    def device_used(self) -> int:
        return self.counters().device_used

    def device_free(self) -> int:
        return self.counters().device_free

    def host_used(self) -> int:
        return self.counters().host_used

    def disk_used(self) -> int:
        return self.counters().disk_used

    def layer_block_bytes(self) -> int:
        return self.counters().layer_block_bytes

    def _i64(self, name: str, *args) -> int:
        out = C.c_int64()
        self._call(name, *args, C.byref(out))
        return out.value

    def bytes_for_new_blocks(self, session: int, new_tokens: int) -> int:
        return self._i64("kvs_bytes_for_new_blocks", session, new_tokens)

    def bytes_for_load(self, session: int) -> int:
        return self._i64("kvs_bytes_for_load", session)

    def bytes_for_promote(self, session: int) -> int:
        return self._i64("kvs_bytes_for_promote", session)

    def reserve_device(self, nbytes: int) -> None:
        self._call("kvs_reserve_device", nbytes)

    def unreserve_device(self, nbytes: int) -> None:
        self._call("kvs_unreserve_device", nbytes)

    # ---- cache state ----
    def session_info(self, session: int) -> _SessionInfo:
        s = _SessionInfo()
        self._call("kvs_get_session", session, C.byref(s))
        return s

    def cached_tokens(self, session: int) -> int:
        return self.session_info(session).cached_tokens

    def session_bytes(self, session: int) -> int:
        return self.session_info(session).session_bytes

    def fully_device_resident(self, session: int) -> bool:
        return bool(self.session_info(session).fully_device_resident)

    def has_any_copy(self, session: int) -> bool:
        return bool(self.session_info(session).has_any_copy)

    def pending_persists(self, session: int) -> int:
        return self.session_info(session).pending_persists

    def migrating_out(self, session: int) -> bool:
        return bool(self.session_info(session).migrating_out)

    def is_active(self, session: int) -> bool:
        return bool(self.session_info(session).is_active)

    def set_active(self, session: int, active: bool, now: int) -> None:
        self._call("kvs_set_active", session, int(active), now)

    def residency(self, session: int, layer: int, block: int) -> int:
        out = C.c_uint8()
        self._call("kvs_residency", session, layer, block, C.byref(out))
        return out.value

    # ---- operations (return values mirror the C++ out-params) ----
    def append_blocks(self, session: int, new_tokens: int, now: int):
        """-> (created BlockKeys as (session, layer, block), scheduled [(id, complete_at)])."""
        rc = self._lib.kvs_append_blocks(self._h, session, new_tokens, now)
        sched = self._scheduled()
        p = C.POINTER(_Key)()
        n = self._lib.kvs_out_keys(self._h, C.byref(p))
        keys = [(p[i].session, p[i].layer, p[i].block_index) for i in range(n)]
        _check(self._lib, rc)
        return keys, sched

    def purge_from_device(self, bytes_needed: int, now: int, spare_high_priority: bool):
        freed = C.c_int64()
        rc = self._lib.kvs_purge_from_device(self._h, bytes_needed, now, int(spare_high_priority), C.byref(freed))
        sched = self._scheduled()
        _check(self._lib, rc)
        return freed.value, sched

    def plan_layerwise_load(self, session: int, now: int, compute_per_layer: int, reason: int = DEMAND):
        plan = _Plan()
        rc = self._lib.kvs_plan_layerwise_load(self._h, session, now, compute_per_layer, reason, C.byref(plan))
        sched = self._scheduled()
        _check(self._lib, rc)
        if not plan.has_plan:
            return None, sched
        p = C.POINTER(C.c_int64)()
        n = self._lib.kvs_out_times(self._h, C.byref(p))
        return LoadPlan([p[i] for i in range(n)], plan.decode_start, plan.finish, plan.total_stall,
                        bool(plan.any_load)), sched

    def promote(self, session: int, now: int):
        r = _Promote()
        rc = self._lib.kvs_promote(self._h, session, now, C.byref(r))
        sched = self._scheduled()
        _check(self._lib, rc)
        return (r.device_layers, r.staged_layers, bool(r.scheduled)), sched

    def offload_session(self, session: int, now: int):
        rc = self._lib.kvs_offload_session(self._h, session, now)
        sched = self._scheduled()
        _check(self._lib, rc)
        return sched

    def release_session(self, session: int, now: int) -> None:
        self._call("kvs_release_session", session, now)

    def mark_migrating_out(self, session: int) -> None:
        self._call("kvs_mark_migrating_out", session)

    def import_migration(self, session: int, tokens: int, now: int):
        self._call("kvs_import_migration", session, tokens, now)
        return self._scheduled()

    def apply_transfer(self, tid: int, now: int) -> ApplyResult:
        r = self._apply_buf
        rc = self._apply_fn(self._h, tid, now, self._apply_ref)
        if rc:
            _check(self._lib, rc)
        return ApplyResult(r.session, r.layer, bool(r.device_layer_ready), bool(r.persists_drained),
                           bool(r.migration_arrived), bool(r.migration_complete), bool(r.voided))

    def void_session_loads(self, session: int) -> None:
        self._call("kvs_void_session_loads", session)

    def void_session_offload(self, session: int) -> None:
        self._call("kvs_void_session_offload", session)

    def evictable_blocks(self, spare_high_priority: bool) -> List[BlockMeta]:
        self._call("kvs_evictable_blocks", int(spare_high_priority))
        p = C.POINTER(_Meta)()
        n = self._lib.kvs_out_metas(self._h, C.byref(p))
        return [BlockMeta(p[i].key.session, p[i].key.layer, p[i].key.block_index,
                          p[i].session_id.decode(), p[i].session_bytes, bool(p[i].pinned)) for i in range(n)]

    def check_budgets(self) -> None:
        self._call("kvs_check_budgets")

    def device_usage_debug(self) -> str:
        buf = C.create_string_buffer(512)
        self._call("kvs_device_usage_debug", buf, len(buf))
        return buf.value.decode()

    def ledger(self) -> List[TransferRecord]:
        n = self._lib.kvs_ledger_size(self._h)
        rows = (_Record * max(n, 1))()
        if n:
            self._call("kvs_ledger_copy", 0, n, rows)
        return [TransferRecord(r.time, r.node, r.session, r.layer_lo, r.layer_hi, r.from_, r.to, r.bytes,
                               r.reason) for r in rows[:n]]


def evict_order(candidates: Sequence[BlockMeta], lib: Optional[str] = None) -> List[BlockMeta]:
    h = load_kvs_library(lib)
    n = len(candidates)
    arr = (_Meta * max(n, 1))()
    ids = [c.session_id.encode() for c in candidates]
    for i, c in enumerate(candidates):
        arr[i] = _Meta(_Key(c.session, c.layer, 0, c.block_index), c.session_bytes, ids[i], int(c.pinned))
    order = (C.c_uint32 * max(n, 1))()
    _check(h, h.kvs_evict_order(arr, n, order))
    return [candidates[order[i]] for i in range(n)]


def pipeline_gate(layer_ready: Sequence[int], compute_ready: int, step_ns: int, lib: Optional[str] = None):
    h = load_kvs_library(lib)
    n = len(layer_ready)
    arr = (C.c_int64 * max(n, 1))(*layer_ready)
    g = _Gate()
    _check(h, h.kvs_pipeline_gate(arr, n, compute_ready, step_ns, C.byref(g)))
    return g.first_step_end, g.gate_start, g.stall


def transfer_time(nbytes: int, link: int, links: Optional[LinkProfile] = None, lib: Optional[str] = None) -> int:
    h = load_kvs_library(lib)
    out = C.c_int64()
    _check(h, h.kvs_transfer_time(nbytes, link, C.byref((links or LinkProfile())._c()), C.byref(out)))
    return out.value


def kv_bytes_per_layer(tokens: int, gpu: Optional[GpuProfile] = None, lib: Optional[str] = None) -> int:
    h = load_kvs_library(lib)
    g, keep = (gpu or GpuProfile())._c()
    out = C.c_int64()
    _check(h, h.kvs_kv_bytes_per_layer(tokens, C.byref(g), C.byref(out)))
    return out.value


def decode_step_time(batch: int, gpu: Optional[GpuProfile] = None, lib: Optional[str] = None) -> int:
    h = load_kvs_library(lib)
    g, keep = (gpu or GpuProfile())._c()
    out = C.c_int64()
    _check(h, h.kvs_decode_step_time(batch, C.byref(g), C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# Physical payload (include/symsim/payload.hpp through kvs.h)

POOL_DEVICE, POOL_HOST, POOL_LANDING, POOL_DISK = range(4)
LANE_IN, LANE_OUT, LANE_DISK, LANE_PEER, LANE_FILL = range(5)
BLOCK_EVENTS = ("created", "load_h2d", "load_disk_host", "host_copy", "disk_write", "swap_out", "net_arrive")


@dataclass
class PayloadOptions:
    """Page pools of one node (symsim::PayloadOptions)."""
    device: int = 0
    num_kv_heads: int = 8
    head_dim: int = 128
    block_tokens: int = 16
    dtype: int = 1  # KVX_DTYPE_BF16
    fill_mode: int = 1  # KVX_FILL_VALUES
    device_pages: int = 0
    host_pages: int = 0
    landing_pages: int = 0
    disk_pages: int = 0
    seed: int = 0
    free_running: bool = False
    disk_path: str = ""  # file backing the DISK tier ("" = pinned host stand-in)
    migrate_max_ctas: int = 0  # cap on the K3 grid of migration pushes (0 = all SMs)

    def _c(self) -> "_PayloadOpts":
        return _PayloadOpts(self.device, self.num_kv_heads, self.head_dim, self.block_tokens, self.dtype,
                            self.fill_mode, self.device_pages, self.host_pages, self.landing_pages,
                            self.disk_pages, self.seed, int(self.free_running), 0,
                            self.disk_path.encode() if self.disk_path else None, self.migrate_max_ctas, 0)

    def page_bytes(self) -> int:
        return 2 * self.num_kv_heads * self.block_tokens * self.head_dim * (2 if self.dtype == 1 else 4)


class PayloadCluster:
    """Registry of payload nodes (migration sources are looked up here)."""

    def __init__(self):
        self._lib = load_kvs_library()
        h = C.c_void_p()
        _check(self._lib, self._lib.kvs_cluster_create(C.byref(h)))
        self._h = h
        self.nodes: Dict[int, "NodePayload"] = {}

    def node(self, node_id: int) -> "NodePayload":
        if node_id not in self.nodes:
            h = C.c_void_p()
            _check(self._lib, self._lib.kvs_cluster_node(self._h, node_id, C.byref(h)))
            self.nodes[node_id] = NodePayload(None, node_id, None, _handle=h.value, _cluster=self)
        return self.nodes[node_id]

    def set_default(self, template: Optional[PayloadOptions], num_devices: int = 1) -> None:
        """Every KvStore constructed afterwards (in any caller) gets a node."""
        if template is None:
            _check(self._lib, self._lib.kvs_set_default_payload(None, None, 0))
        else:
            _check(self._lib, self._lib.kvs_set_default_payload(self._h, C.byref(template._c()), num_devices))


class NodePayload:
    """Real pages behind one store's DEVICE/HOST/DISK copies."""

    def __init__(self, cluster: Optional[PayloadCluster], node_id: int, opts: Optional[PayloadOptions],
                 _handle: Optional[int] = None, _cluster=None):
        self._lib = load_kvs_library()
        self.node_id = node_id
        self.cluster = cluster or _cluster
        if _handle is not None:
            self._h = C.c_void_p(_handle)
            self.opts = opts
        else:
            h = C.c_void_p()
            _check(self._lib, self._lib.kvs_payload_create(cluster._h if cluster else None, node_id,
                                                           C.byref(opts._c()), C.byref(h)))
            self._h = h
            self.opts = opts
            if cluster is not None:
                cluster.nodes[node_id] = self

    def attach(self, store: KvStore) -> None:
        _check(self._lib, self._lib.kvs_attach_payload(store._h, self._h))

    def read_block(self, session: int, layer: int, block: int, tier: int, page_bytes: int):
        import numpy as np
        out = np.empty(page_bytes, np.uint8)
        rc = self._lib.kvs_payload_read_block(self._h, session, layer, block, tier, out.ctypes.data)
        if rc == 1:
            return None
        _check(self._lib, rc)
        return out

    def pages_in_use(self, pool: int) -> int:
        out = C.c_uint64()
        _check(self._lib, self._lib.kvs_payload_pages_in_use(self._h, pool, C.byref(out)))
        return out.value

    def pool_of(self, session: int, layer: int, block: int, tier: int) -> int:
        out = C.c_int32()
        _check(self._lib, self._lib.kvs_payload_pool_of(self._h, session, layer, block, tier, C.byref(out)))
        return out.value

    def bytes_moved(self) -> Dict[str, int]:
        out = (C.c_uint64 * 7)()
        _check(self._lib, self._lib.kvs_payload_bytes_moved(self._h, out))
        return dict(zip(BLOCK_EVENTS, list(out)))

    def stats(self) -> Dict[str, int]:
        out = (C.c_uint64 * 7)()
        _check(self._lib, self._lib.kvs_payload_stats(self._h, out))
        return {"apply_wait_ns": out[0], "transfers_posted": out[1], "in_flight": list(out[2:6]),
                "cross_lane_waits": out[6]}

    def host_ns(self) -> Dict[str, int]:
        """Host ns of the payload's bookkeeping by phase (kvs_payload_host_ns)."""
        out = (C.c_uint64 * 8)()
        _check(self._lib, self._lib.kvs_payload_host_ns(self._h, out))
        return dict(zip(("posted", "retired", "issue", "reclaim", "upload", "launch", "close", "alloc"), list(out)))

    def device_block_table(self, session: int, layer: int, n: int):
        """uint32 DEVICE page ids of blocks [0, n) — a decode block-table row."""
        import numpy as np
        out = np.empty(n, np.uint32)
        _check(self._lib, self._lib.kvs_payload_block_table(self._h, session, layer, n,
                                                            out.ctypes.data_as(C.POINTER(C.c_uint32))))
        return out

    def pool_handle(self, pool: int) -> int:
        """The kvx_pool* behind one of this node's pools (for kvx calls)."""
        out = C.c_void_p()
        _check(self._lib, self._lib.kvs_payload_pool(self._h, pool, C.byref(out)))
        return out.value

    def synchronize(self) -> None:
        _check(self._lib, self._lib.kvs_payload_synchronize(self._h))

    def stream(self, lane: int) -> int:
        """cudaStream_t of a lane (LANE_IN / LANE_OUT / LANE_DISK / LANE_PEER)."""
        out = C.c_void_p()
        _check(self._lib, self._lib.kvs_payload_stream(self._h, lane, C.byref(out)))
        return out.value


# ---- serving traffic (include/symsim/traffic.hpp) ---------------------------

def zipf_turns(sessions: int, s: float = 1.2, scale: float = 64.0, min_turns: int = 2, seed: int = 0):
    """Turns per session under Zipf(s) popularity (kvs_traffic_zipf_turns)."""
    import numpy as np
    lib = load_kvs_library()
    out = np.empty(sessions, np.int32)
    _check(lib, lib.kvs_traffic_zipf_turns(sessions, s, scale, min_turns, seed,
                                           out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def poisson_gaps(n: int, mean_s: float, seed: int = 0):
    """n exponential think times (ns) with mean mean_s seconds."""
    import numpy as np
    lib = load_kvs_library()
    out = np.empty(n, np.int64)
    _check(lib, lib.kvs_traffic_poisson_gaps(n, mean_s, seed, out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


def percentile(values, q: float) -> float:
    import numpy as np
    lib = load_kvs_library()
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = C.c_double()
    _check(lib, lib.kvs_traffic_percentile(v.ctypes.data_as(C.POINTER(C.c_double)), v.size, q, C.byref(out)))
    return out.value


def rps_within_slo(sweep, slo: float) -> float:
    """sweep: [(users, rps, p50)] -> highest rps with p50 <= slo."""
    import numpy as np
    lib = load_kvs_library()
    u = np.ascontiguousarray([p[0] for p in sweep], dtype=np.int32)
    r = np.ascontiguousarray([p[1] for p in sweep], dtype=np.float64)
    m = np.ascontiguousarray([p[2] for p in sweep], dtype=np.float64)
    out = C.c_double()
    _check(lib, lib.kvs_traffic_rps_within_slo(u.ctypes.data_as(C.POINTER(C.c_int32)),
                                               r.ctypes.data_as(C.POINTER(C.c_double)),
                                               m.ctypes.data_as(C.POINTER(C.c_double)), len(sweep), slo,
                                               C.byref(out)))
    return out.value
