"""ctypes loader for the oracle libraries. TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline / reference arm — never from the product package.

  payload()  -> oracle/build/libkvx_oracle.so  (CPU restatement, kvx_oracle.c)
  ref_kvs()  -> oracle/_ref/libsymsim_oracle.so (reference KvStore, kvs_* ABI)
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent
PAYLOAD_LIB = ORACLE_DIR / "build" / "libkvx_oracle.so"
REF_KVS_LIB = ORACLE_DIR / "_ref" / "libsymsim_oracle.so"


class Layout(C.Structure):
    _fields_ = [("num_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("block_tokens", C.c_int32),
                ("dtype", C.c_int32)]


_PAYLOAD = None


def build_payload() -> None:
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "payload"], check=True)


def payload() -> C.CDLL:
    global _PAYLOAD
    if _PAYLOAD is None:
        build_payload()
        h = C.CDLL(str(PAYLOAD_LIB))
        V, U64, P = C.c_void_p, C.c_uint64, C.POINTER
        h.kvxo_splitmix64.argtypes, h.kvxo_splitmix64.restype = [U64], U64
        h.kvxo_page_bytes.argtypes, h.kvxo_page_bytes.restype = [P(Layout)], U64
        h.kvxo_threads.argtypes, h.kvxo_threads.restype = [], C.c_int
        h.kvxo_fill_pages.argtypes = [V, U64, V, V, U64, U64, P(Layout), C.c_int]
        h.kvxo_pack.argtypes = [V, U64, V, U64, V, C.c_int]
        h.kvxo_unpack.argtypes = [V, U64, V, U64, V, C.c_int]
        h.kvxo_copy_pages.argtypes = [V, V, V, V, U64, U64, C.c_int]
        h.kvxo_append_kv.argtypes = [V, P(Layout), V, V, V, V, U64]
        h.kvxo_decode_attention.argtypes = [V, P(Layout), C.c_int32, V, C.c_int32, V, V, V, C.c_int32, C.c_float,
                                            C.c_int]
        for fn in ("kvxo_fill_pages", "kvxo_pack", "kvxo_unpack", "kvxo_copy_pages", "kvxo_append_kv",
                   "kvxo_decode_attention"):
            getattr(h, fn).restype = None
        _PAYLOAD = h
    return _PAYLOAD


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def tags_array(session, layer, block) -> np.ndarray:
    """(n, 3) uint32 array of (session, layer, block) tags."""
    return np.ascontiguousarray(np.stack(np.broadcast_arrays(
        np.asarray(session, np.uint32), np.asarray(layer, np.uint32), np.asarray(block, np.uint32)), axis=-1)
        .reshape(-1, 3))


def fill_pages(pool: np.ndarray, page_bytes: int, ids: np.ndarray, tags: np.ndarray, seed: int, layout: Layout,
               mode: int) -> None:
    ids = np.ascontiguousarray(ids, np.uint32)
    tags = np.ascontiguousarray(tags, np.uint32)
    payload().kvxo_fill_pages(_p(pool), page_bytes, _p(ids), _p(tags), len(ids), seed, C.byref(layout), mode)


def pack(pool: np.ndarray, page_bytes: int, ids: np.ndarray, dst: np.ndarray, threads: int = 0) -> None:
    ids = np.ascontiguousarray(ids, np.uint32)
    payload().kvxo_pack(_p(pool), page_bytes, _p(ids), len(ids), _p(dst), threads)


def unpack(pool: np.ndarray, page_bytes: int, ids: np.ndarray, src: np.ndarray, threads: int = 0) -> None:
    ids = np.ascontiguousarray(ids, np.uint32)
    payload().kvxo_unpack(_p(pool), page_bytes, _p(ids), len(ids), _p(src), threads)


def copy_pages(src_pool: np.ndarray, src_ids, dst_pool: np.ndarray, dst_ids, page_bytes: int, threads: int = 0):
    s = np.ascontiguousarray(src_ids, np.uint32)
    d = np.ascontiguousarray(dst_ids, np.uint32)
    payload().kvxo_copy_pages(_p(src_pool), _p(s), _p(dst_pool), _p(d), len(s), page_bytes, threads)


def append_kv(pool: np.ndarray, layout: Layout, ids, slots, k: np.ndarray, v: np.ndarray) -> None:
    ids = np.ascontiguousarray(ids, np.uint32)
    slots = np.ascontiguousarray(slots, np.int32)
    payload().kvxo_append_kv(_p(pool), C.byref(layout), _p(ids), _p(slots), _p(np.ascontiguousarray(k)),
                             _p(np.ascontiguousarray(v)), len(ids))


def decode_attention(pool: np.ndarray, layout: Layout, num_q_heads: int, tables: np.ndarray, ctx_lens: np.ndarray,
                     q: np.ndarray, scale: float, threads: int = 0) -> np.ndarray:
    tables = np.ascontiguousarray(tables, np.uint32)
    ctx_lens = np.ascontiguousarray(ctx_lens, np.int32)
    batch = len(ctx_lens)
    out = np.zeros((batch, num_q_heads, layout.head_dim), np.float64)
    payload().kvxo_decode_attention(_p(pool), C.byref(layout), num_q_heads, _p(tables), tables.shape[1],
                                    _p(ctx_lens), _p(np.ascontiguousarray(q)), _p(out), batch, scale, threads)
    return out


def threads() -> int:
    return payload().kvxo_threads()
