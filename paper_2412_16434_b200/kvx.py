"""ctypes binding of the kvx C ABI (include/kvx.h) — the B200 payload path.

Device memory and streams come from PyTorch (plumbing only): tensors are
passed as raw pointers, streams as cudaStream_t handles. The library is the
in-tree lib/libkvx.so; there is no CPU fallback — if the extension or a CUDA
device is missing, every call raises KvxError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

from . import _build

F32, BF16 = 0, 1
FILL_BITS, FILL_VALUES = 0, 1
COPY_AUTO, COPY_SM, COPY_TMA, COPY_CE = 0, 1, 2, 3
MERGE_AUTO, MERGE_GLOBAL, MERGE_CLUSTER = 0, 1, 2
ATTN_EARLY_PREFETCH = 1


class KvxError(RuntimeError):
    pass


class PageLayout(C.Structure):
    _fields_ = [("num_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("block_tokens", C.c_int32),
                ("dtype", C.c_int32)]

    def page_bytes(self) -> int:
        return 2 * self.num_kv_heads * self.block_tokens * self.head_dim * (2 if self.dtype == BF16 else 4)


class BlockTag(C.Structure):
    _fields_ = [("session", C.c_uint32), ("layer", C.c_uint32), ("block", C.c_uint32)]


class AttnParams(C.Structure):
    _fields_ = [("num_q_heads", C.c_int32), ("max_blocks", C.c_int32), ("num_splits", C.c_int32),
                ("scale", C.c_float), ("split_merge", C.c_int32), ("flags", C.c_int32)]


_LIB: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    _build.ensure_built()
    if not _build.KVX_LIB.exists():
        raise KvxError(f"kvx extension missing: {_build.KVX_LIB}")
    h = C.CDLL(str(_build.KVX_LIB))
    P, V, U64 = C.POINTER, C.c_void_p, C.c_uint64
    sigs = {
        "kvx_last_error": ([], C.c_char_p),
        "kvx_version": ([], C.c_int),
        "kvx_launch_count": ([], C.c_uint64),
        "kvx_migrate_nccl_staging_bytes": ([C.c_uint64, C.c_uint64], C.c_uint64),
        "kvx_migrate_nccl": ([C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                              C.c_int, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p], C.c_int),
        "kvx_nccl_get_unique_id": ([C.c_void_p], C.c_int),
        "kvx_nccl_comm_init_rank": ([C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_int, C.c_int], C.c_int),
        "kvx_nccl_comm_destroy": ([C.c_void_p], C.c_int),
        "kvx_library_launch_count": ([], C.c_uint64),
        "kvx_page_bytes": ([P(PageLayout)], U64),
        "kvx_pool_create": ([C.c_int, U64, U64, P(V)], C.c_int),
        "kvx_pool_create_host": ([U64, U64, P(V)], C.c_int),
        "kvx_pool_wrap": ([C.c_int, V, U64, U64, P(V)], C.c_int),
        "kvx_pool_create_file": ([C.c_char_p, U64, U64, P(V)], C.c_int),
        "kvx_pool_file_direct": ([V], C.c_int),
        "kvx_read_page": ([V, U64, V], C.c_int),
        "kvx_pool_destroy": ([V], C.c_int),
        "kvx_pool_base": ([V], V),
        "kvx_pool_num_pages": ([V], U64),
        "kvx_pool_page_bytes": ([V], U64),
        "kvx_pool_device": ([V], C.c_int),
        "kvx_pool_ipc_export": ([V, V], C.c_int),
        "kvx_pool_ipc_open": ([C.c_int, V, U64, U64, P(V)], C.c_int),
        "kvx_enable_peer_access": ([C.c_int, C.c_int], C.c_int),
        "kvx_signal_write": ([V, C.c_uint32, V], C.c_int),
        "kvx_signal_wait": ([V, C.c_uint32, V], C.c_int),
        "kvx_pack": ([V, V, U64, V, C.c_int, V], C.c_int),
        "kvx_unpack": ([V, V, U64, V, C.c_int, V], C.c_int),
        "kvx_copy_pages": ([V, V, V, V, U64, C.c_int, V], C.c_int),
        "kvx_copy_pages_capped": ([V, V, V, V, U64, C.c_int, C.c_uint32, V], C.c_int),
        "kvx_fill_pages": ([V, V, V, U64, U64, P(PageLayout), C.c_int, V], C.c_int),
        "kvx_append_kv": ([V, P(PageLayout), V, V, V, V, U64, V], C.c_int),
        "kvx_decode_attention_workspace": ([P(PageLayout), P(AttnParams), C.c_int32, C.c_int32], U64),
        "kvx_decode_attention": ([V, P(PageLayout), P(AttnParams), V, V, V, V, C.c_int32, C.c_int32, V, U64, V],
                                 C.c_int),
        "kvx_decode_attention_append": ([V, P(PageLayout), P(AttnParams), V, V, V, V, V, V, C.c_int32, C.c_int32, V,
                                         U64, V], C.c_int),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(h, name)
        fn.argtypes = args
        fn.restype = res
    _LIB = h
    return h


def launch_count() -> int:
    """Launches of libkvx's own kernels so far (kvx_launch_count)."""
    return lib().kvx_launch_count()


def check(rc: int) -> None:
    if rc != 0:
        raise KvxError((lib().kvx_last_error() or b"").decode())


def _ptr(x) -> Optional[int]:
    """Raw address of a tensor / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Pool:
    """A page pool (DEVICE in HBM, or HOST pinned+mapped)."""

    def __init__(self, num_pages: int, page_bytes: int, device: int = 0, host: bool = False,
                 _handle: Optional[int] = None):
        L = lib()
        h = C.c_void_p()
        if _handle is not None:
            h = C.c_void_p(_handle)
        elif host:
            check(L.kvx_pool_create_host(num_pages, page_bytes, C.byref(h)))
        else:
            check(L.kvx_pool_create(device, num_pages, page_bytes, C.byref(h)))
        self.handle = h
        self.num_pages = num_pages
        self.page_bytes = page_bytes
        self.device = -1 if host else device

    @classmethod
    def borrow(cls, handle: int, num_pages: int, page_bytes: int, device: int = 0) -> "Pool":
        """A non-owning view of a kvx_pool* owned elsewhere (e.g. a NodePayload)."""
        p = cls(num_pages, page_bytes, device, _handle=handle)
        p._borrowed = True
        return p

    @classmethod
    def wrap(cls, tensor, num_pages: int, page_bytes: int, device: int = 0) -> "Pool":
        h = C.c_void_p()
        check(lib().kvx_pool_wrap(device, tensor.data_ptr(), num_pages, page_bytes, C.byref(h)))
        p = cls(num_pages, page_bytes, device, _handle=h.value)
        p._keep = tensor
        return p

    @classmethod
    def file(cls, path: str, num_pages: int, page_bytes: int) -> "Pool":
        """DISK-tier pool backed by a file (kvx_pool_create_file); pages move to
        and from HOST pools with copy_pages(..., COPY_CE) on host id arrays."""
        h = C.c_void_p()
        check(lib().kvx_pool_create_file(str(path).encode(), num_pages, page_bytes, C.byref(h)))
        p = cls(num_pages, page_bytes, -1, _handle=h.value)
        p.path = str(path)
        return p

    @property
    def direct_io(self) -> bool:
        return lib().kvx_pool_file_direct(self.handle) == 1

    def read_page(self, page: int):
        """Synchronous copy of one page to a new numpy array (any pool kind)."""
        import numpy as np
        out = np.empty(self.page_bytes, np.uint8)
        check(lib().kvx_read_page(self.handle, page, out.ctypes.data))
        return out

    @classmethod
    def ipc_open(cls, handle64: bytes, num_pages: int, page_bytes: int, device: int) -> "Pool":
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(handle64), 64)
        check(lib().kvx_pool_ipc_open(device, buf, num_pages, page_bytes, C.byref(h)))
        return cls(num_pages, page_bytes, device, _handle=h.value)

    def ipc_export(self) -> bytes:
        buf = C.create_string_buffer(64)
        check(lib().kvx_pool_ipc_export(self.handle, buf))
        return buf.raw

    @property
    def base(self) -> int:
        return lib().kvx_pool_base(self.handle)

    def as_tensor(self):
        """uint8 view [num_pages, page_bytes] of the pool memory (no copy)."""
        import torch
        from torch.utils.dlpack import from_dlpack  # noqa: F401
        n = self.num_pages * self.page_bytes
        if self.device < 0:
            buf = (C.c_uint8 * n).from_address(self.base)
            return torch.frombuffer(buf, dtype=torch.uint8).view(self.num_pages, self.page_bytes)
        return _device_view(self.base, n, self.device).view(self.num_pages, self.page_bytes)

    def close(self) -> None:
        if getattr(self, "_borrowed", False):
            self.handle = None
            return
        if self.handle:
            check(lib().kvx_pool_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _device_view(ptr: int, nbytes: int, device: int):
    """Wrap raw device memory as a uint8 torch tensor (non-owning)."""
    import torch

    class _CudaArray:
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (p, False), "version": 3}

    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArray(ptr, nbytes), device=f"cuda:{device}")


def page_bytes(layout: PageLayout) -> int:
    return lib().kvx_page_bytes(C.byref(layout))


def signal_write(flag_addr: int, value: int, stream=None) -> None:
    """Stream-ordered write of a 32-bit flag (peer memory allowed) after all prior work."""
    check(lib().kvx_signal_write(flag_addr, value, _stream(stream)))


def signal_wait(flag_addr: int, value: int, stream=None) -> None:
    """The stream waits until the 32-bit flag is >= value."""
    check(lib().kvx_signal_wait(flag_addr, value, _stream(stream)))


def pack(pool: Pool, page_ids, n: int, dst, mode: int = COPY_AUTO, stream=None) -> None:
    check(lib().kvx_pack(pool.handle, _ptr(page_ids), n, _ptr(dst), mode, _stream(stream)))


def unpack(pool: Pool, page_ids, n: int, src, mode: int = COPY_AUTO, stream=None) -> None:
    check(lib().kvx_unpack(pool.handle, _ptr(page_ids), n, _ptr(src), mode, _stream(stream)))


def copy_pages(src: Pool, src_ids, dst: Pool, dst_ids, n: int, mode: int = COPY_AUTO, stream=None,
               max_ctas: int = 0) -> None:
    """K3 page -> page. max_ctas > 0 bounds the SM movers' grid (background
    migration beside decode, kvx_copy_pages_capped)."""
    if max_ctas and mode != COPY_CE:
        check(lib().kvx_copy_pages_capped(src.handle, _ptr(src_ids), dst.handle, _ptr(dst_ids), n, mode, max_ctas,
                                          _stream(stream)))
        return
    if mode == COPY_CE:
        import numpy as np
        s = np.ascontiguousarray(src_ids, dtype=np.uint32)
        d = np.ascontiguousarray(dst_ids, dtype=np.uint32)
        check(lib().kvx_copy_pages(src.handle, s.ctypes.data, dst.handle, d.ctypes.data, n, mode, _stream(stream)))
        return
    check(lib().kvx_copy_pages(src.handle, _ptr(src_ids), dst.handle, _ptr(dst_ids), n, mode, _stream(stream)))


def fill_pages(pool: Pool, page_ids, tags, n: int, seed: int, layout: Optional[PageLayout], mode: int,
               stream=None) -> None:
    lay = C.byref(layout) if layout is not None else None
    check(lib().kvx_fill_pages(pool.handle, _ptr(page_ids), _ptr(tags), n, seed, lay, mode, _stream(stream)))


def append_kv(pool: Pool, layout: PageLayout, page_ids, slots, k, v, n: int, stream=None) -> None:
    check(lib().kvx_append_kv(pool.handle, C.byref(layout), _ptr(page_ids), _ptr(slots), _ptr(k), _ptr(v), n,
                              _stream(stream)))


@dataclass
class Attention:
    """Paged decode attention (K4) with its own workspace."""
    layout: PageLayout
    num_q_heads: int
    max_blocks: int
    num_splits: int = 0
    scale: float = 0.0
    split_merge: int = MERGE_AUTO
    flags: int = 0  # ATTN_EARLY_PREFETCH: decode-step contract (see include/kvx.h)

    def params(self) -> AttnParams:
        return AttnParams(self.num_q_heads, self.max_blocks, self.num_splits, self.scale, self.split_merge,
                          self.flags)

    def workspace_bytes(self, batch: int, max_ctx: int) -> int:
        p = self.params()
        return lib().kvx_decode_attention_workspace(C.byref(self.layout), C.byref(p), batch, max_ctx)

    def __call__(self, pool: Pool, block_tables, ctx_lens, q, out, batch: int, max_ctx: int, workspace=None,
                 stream=None, new_k=None, new_v=None) -> None:
        """new_k / new_v ([batch][kv heads][head_dim]): fused decode step —
        append this token at position ctx_lens[b] - 1, then attend
        (kvx_decode_attention_append)."""
        p = self.params()
        ws = _ptr(workspace)
        ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
        if new_k is not None or new_v is not None:
            check(lib().kvx_decode_attention_append(pool.handle, C.byref(self.layout), C.byref(p), _ptr(block_tables),
                                                    _ptr(ctx_lens), _ptr(q), _ptr(new_k), _ptr(new_v), _ptr(out),
                                                    batch, max_ctx, ws, ws_bytes, _stream(stream)))
            return
        check(lib().kvx_decode_attention(pool.handle, C.byref(self.layout), C.byref(p), _ptr(block_tables),
                                         _ptr(ctx_lens), _ptr(q), _ptr(out), batch, max_ctx, ws, ws_bytes,
                                         _stream(stream)))


# ---- K3 over NCCL (kvx_migrate_nccl) -----------------------------------------

def migrate_nccl_staging_bytes(page_bytes: int, pages_per_chunk: int) -> int:
    return lib().kvx_migrate_nccl_staging_bytes(page_bytes, pages_per_chunk)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().kvx_nccl_get_unique_id(buf))
    return buf.raw


def nccl_comm_init_rank(nranks: int, uid: bytes, rank: int, device: int) -> int:
    comm = C.c_void_p()
    buf = C.create_string_buffer(bytes(uid), 128)
    check(lib().kvx_nccl_comm_init_rank(C.byref(comm), nranks, buf, rank, device))
    return comm.value


def nccl_comm_destroy(comm: int) -> None:
    check(lib().kvx_nccl_comm_destroy(comm))


def migrate_nccl(send_pool, send_ids, n_send: int, send_peer: int, recv_pool, recv_ids, n_recv: int,
                 recv_peer: int, pages_per_chunk: int, comm: int, staging, stream=None) -> None:
    """K1 pack -> ncclSend/ncclRecv -> K2 unpack per chunk (kvx_migrate_nccl)."""
    check(lib().kvx_migrate_nccl(send_pool.handle if send_pool is not None else None, _ptr(send_ids), n_send,
                                 send_peer, recv_pool.handle if recv_pool is not None else None, _ptr(recv_ids),
                                 n_recv, recv_peer, pages_per_chunk, comm, _ptr(staging), staging.numel(),
                                 _stream(stream)))
