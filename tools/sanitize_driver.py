"""Small invocations of every kvx kernel for compute-sanitizer (tools/sanitize.sh)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_16434_b200 import kvx  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
for layout in (kvx.PageLayout(8, 128, 16, kvx.BF16), kvx.PageLayout(4, 64, 16, kvx.F32)):
    pb = layout.page_bytes()
    n, pages = 40, 100
    pool = kvx.Pool(pages, pb)
    ids = torch.from_numpy(rng.permutation(pages)[:n].astype(np.int32)).to(dev)
    dst = torch.from_numpy(rng.permutation(pages)[:n].astype(np.int32)).to(dev)
    tags = torch.stack([ids * 0, ids * 0, ids], -1).contiguous()
    kvx.fill_pages(pool, ids, tags, n, 1, layout, kvx.FILL_VALUES)
    kvx.fill_pages(pool, dst, tags, n, 2, layout, kvx.FILL_BITS)
    buf = torch.empty(n * pb, dtype=torch.uint8, device=dev)
    for mode in (kvx.COPY_SM, kvx.COPY_TMA):
        kvx.pack(pool, ids, n, buf, mode)
        kvx.unpack(pool, dst, n, buf, mode)
        kvx.copy_pages(pool, ids, pool, dst, n, mode)
        kvx.copy_pages(pool, ids, pool, dst, n, mode, max_ctas=3)  # capped background mover
    host = kvx.Pool(n, pb, host=True)
    kvx.copy_pages(pool, ids, host, torch.arange(n, dtype=torch.int32, device=dev), n, kvx.COPY_SM)
    elt = torch.bfloat16 if layout.dtype == kvx.BF16 else torch.float32
    k = torch.randn(5, layout.num_kv_heads, layout.head_dim, device=dev).to(elt)
    kvx.append_kv(pool, layout, ids[:5], torch.arange(5, dtype=torch.int32, device=dev), k, k, 5)
    for batch, ctx, splits, merge in ((1, 600, 0, kvx.MERGE_AUTO), (3, 333, 4, kvx.MERGE_GLOBAL),
                                      (3, 333, 4, kvx.MERGE_CLUSTER), (1, 8192, 10, kvx.MERGE_CLUSTER),
                                      (2, 1024, 1, kvx.MERGE_AUTO)):
        blocks = (ctx + 15) // 16
        tables = torch.from_numpy(rng.integers(0, pages, (batch, blocks)).astype(np.int32)).to(dev)
        lens = torch.full((batch,), ctx, dtype=torch.int32, device=dev)
        hq = 4 * layout.num_kv_heads
        q = torch.randn(batch, hq, layout.head_dim, device=dev).to(elt)
        out = torch.empty(batch, hq, layout.head_dim, dtype=torch.float32, device=dev)
        att = kvx.Attention(layout, hq, blocks, num_splits=splits, split_merge=merge)
        ws = torch.zeros(max(att.workspace_bytes(batch, ctx), 1), dtype=torch.uint8, device=dev)
        att(pool, tables, lens, q, out, batch, ctx, ws)
        nk = torch.randn(batch, layout.num_kv_heads, layout.head_dim, device=dev).to(elt)
        att(pool, tables, lens, q, out, batch, ctx, ws, new_k=nk, new_v=nk)  # fused append + attend
        early = kvx.Attention(layout, hq, blocks, num_splits=splits, split_merge=merge, flags=kvx.ATTN_EARLY_PREFETCH)
        early(pool, tables, lens, q, out, batch, ctx, ws)
        early(pool, tables, lens, q, out, batch, ctx, ws, new_k=nk, new_v=nk)
    # round 2: the CE lane with host ids (listed-id SM mover for fragmented
    # ids, per-run copies for runs) and kvx_copy_pages_listed (TMA / SM)
    hids = rng.permutation(n).astype(np.uint32)
    kvx.copy_pages(pool, ids.cpu().numpy().astype(np.uint32), host, hids, n, kvx.COPY_CE)
    kvx.copy_pages(host, hids, pool, dst.cpu().numpy().astype(np.uint32), n, kvx.COPY_CE)
    runs = np.arange(n, dtype=np.uint32)
    kvx.copy_pages(pool, runs, host, runs, n, kvx.COPY_CE)
    import ctypes
    lib = kvx.lib()
    V, U64 = ctypes.c_void_p, ctypes.c_uint64
    lib.kvx_copy_pages_listed.argtypes = [V, V, V, V, U64, ctypes.c_int, ctypes.c_uint32, V]
    s_ids = ids.cpu().numpy().astype(np.uint32)
    d_ids = dst.cpu().numpy().astype(np.uint32)
    for mode in (kvx.COPY_AUTO, kvx.COPY_SM, kvx.COPY_TMA):
        assert lib.kvx_copy_pages_listed(pool.handle, s_ids.ctypes.data, pool.handle, d_ids.ctypes.data, n, mode, 0,
                                         None) == 0, lib.kvx_last_error()

# round 2: K7 projections (one small model's shapes) and the model's kernels
import ctypes  # noqa: E402


class ModelConfig(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("hidden", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("intermediate", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("rms_eps", ctypes.c_float), ("rope_theta", ctypes.c_float)]


lib = kvx.lib()
lib.kvx_model_create.argtypes = [ctypes.c_int, ctypes.POINTER(ModelConfig), ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]
lib.kvx_model_linear.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int32] * 4 + [ctypes.c_void_p]
lib.kvx_model_prefill.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
lib.kvx_model_destroy.argtypes = [ctypes.c_void_p]
cfg = ModelConfig(1, 512, 8, 2, 128, 1024, 1024, 1e-5, 500000.0)
m = ctypes.c_void_p()
assert lib.kvx_model_create(0, ctypes.byref(cfg), 3, ctypes.byref(m)) == 0, lib.kvx_last_error()
for rows in (1, 5, 8, 12):
    for k_, n_ in ((512, 1536), (1024, 512), (512, 1024)):
        x = torch.randn(rows, k_, device=dev).to(torch.bfloat16)
        w = torch.randn(n_, k_, device=dev).to(torch.bfloat16)
        y = torch.zeros(rows, n_, device=dev, dtype=torch.bfloat16)
        for acc in (0, 1):
            assert lib.kvx_model_linear(m, x.data_ptr(), w.data_ptr(), y.data_ptr(), rows, k_, n_, acc, None) == 0
assert lib.kvx_model_prefill(m, 40, None) == 0  # norms, SiLU, argmax of the last row
torch.cuda.synchronize()
lib.kvx_model_destroy(m)
torch.cuda.synchronize()
print("sanitize driver done")
