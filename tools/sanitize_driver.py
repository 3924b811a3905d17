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
torch.cuda.synchronize()
print("sanitize driver done")
