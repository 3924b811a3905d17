"""Drive K4 (paged decode attention) for an ncu capture: one config, a few
launches. usage: python tools/profile_attn.py BATCH CTX [SPLITS] [REPS]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_16434_b200 import kvx  # noqa: E402


def main():
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    splits = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    dev = torch.device("cuda:0")
    layout = kvx.PageLayout(8, 128, 16, kvx.BF16)
    blocks = (ctx + 15) // 16
    pages = batch * blocks
    pool = kvx.Pool(pages, layout.page_bytes())
    ids = torch.arange(pages, dtype=torch.int32, device=dev)
    kvx.fill_pages(pool, ids, torch.stack([ids * 0, ids * 0, ids], -1).contiguous(), pages, 1, layout,
                   kvx.FILL_VALUES)
    tables = torch.randperm(pages, device=dev).to(torch.int32).view(batch, blocks).contiguous()
    lens = torch.full((batch,), ctx, dtype=torch.int32, device=dev)
    q = (torch.randn(batch, 32, 128, device=dev) * 0.5).to(torch.bfloat16)
    out = torch.empty(batch, 32, 128, dtype=torch.float32, device=dev)
    att = kvx.Attention(layout, 32, blocks, num_splits=splits)
    ws = torch.zeros(max(att.workspace_bytes(batch, ctx), 1), dtype=torch.uint8, device=dev)
    for _ in range(reps):
        att(pool, tables, lens, q, out, batch, ctx, ws)
    torch.cuda.synchronize()
    print("done", float(out.abs().mean()))


if __name__ == "__main__":
    main()
