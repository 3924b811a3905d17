"""Measured-bandwidth predictor for the store's link model.

The reference fixes every transfer's completion at enqueue from constant link
bandwidths (LinkProfile, /root/reference/proj/include/symsim/costmodel.hpp:
29-36; transfer_time, costmodel.cpp:82-95) and models the decode step as an
affine function of batch (or a measured curve, costmodel.hpp:11-16). This
module measures those constants on the GPU with the kvx kernels and returns
a LinkProfile / GpuProfile whose predictions match this hardware, so the
store's schedule (and the free-running payload, which completes each move at
its modelled time) tracks the real machine:

  pcie_bandwidth      copy engines, one layer of pages pinned HOST -> HBM
                      and HBM -> pinned HOST (the HostCopy / LoadH2D unit)
  network_bandwidth   K3 page copy into a peer GPU's pool when a second GPU
                      is visible; else the same-GPU page->page copy rate,
                      flagged as such
  decode_curve_ms     per-batch decode step: K4 over every layer at the
                      given context, plus streaming the model weights once at
                      the measured page-copy bandwidth (an estimate: the
                      weights GEMV is not part of this path)

usage: python -m paper_2412_16434_b200.calibrate [--out profiles/calibration.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from typing import Dict, List, Optional

from . import kvstore as K
from . import kvx

LLAMA8B = dict(layers=32, kv_heads=8, head_dim=128, params=8.03e9)


def _time_ms(torch, fn, reps: int = 10) -> float:
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def _hbm_read_gbs(out: Dict) -> float:
    """HBM streaming rate for the weights estimate: the driver-measured copy
    peak (MEASURED_PEAKS.json) when present, else twice the page-copy rate."""
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 2 * out["hbm_page_copy_gbs"]


def measure(device: int = 0, ctx: int = 2048, batches=(1, 8, 16, 32, 64)) -> Dict:
    import numpy as np
    import torch

    dev = torch.device("cuda", device)
    torch.cuda.set_device(dev)
    layout = kvx.PageLayout(LLAMA8B["kv_heads"], LLAMA8B["head_dim"], 16, kvx.BF16)
    pb = layout.page_bytes()
    blocks = 512  # one 8K layer: 32 MiB
    out: Dict = {"device": torch.cuda.get_device_name(dev), "page_bytes": pb}

    # PCIe, copy engines, one layer per transfer
    host = kvx.Pool(blocks, pb, host=True)
    pool = kvx.Pool(2 * blocks, pb, device=device)
    ids = np.arange(blocks, dtype=np.uint32)
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        h2d = _time_ms(torch, lambda: kvx.copy_pages(host, ids, pool, ids, blocks, kvx.COPY_CE, s))
        d2h = _time_ms(torch, lambda: kvx.copy_pages(pool, ids, host, ids, blocks, kvx.COPY_CE, s))
    out["pcie_h2d_gbs"] = blocks * pb / (h2d * 1e-3) / 1e9
    out["pcie_d2h_gbs"] = blocks * pb / (d2h * 1e-3) / 1e9

    # page -> page (HBM) and, when available, into a peer GPU
    d_src = torch.arange(blocks, dtype=torch.int32, device=dev)
    d_dst = d_src + blocks
    local = _time_ms(torch, lambda: kvx.copy_pages(pool, d_src, pool, d_dst, blocks, kvx.COPY_AUTO))
    out["hbm_page_copy_gbs"] = blocks * pb / (local * 1e-3) / 1e9  # session bytes relocated per second
    if torch.cuda.device_count() > 1:
        peer_dev = (device + 1) % torch.cuda.device_count()
        kvx.check(kvx.lib().kvx_enable_peer_access(device, peer_dev))
        peer = kvx.Pool(blocks, pb, device=peer_dev)
        t = _time_ms(torch, lambda: kvx.copy_pages(pool, d_src, peer, d_src, blocks, kvx.COPY_SM))
        out["nvlink_gbs"] = blocks * pb / (t * 1e-3) / 1e9
        out["network_source"] = "K3 into peer GPU pool"
    else:
        out["nvlink_gbs"] = None
        out["network_source"] = "no peer GPU visible: network_bandwidth = same-GPU page copy rate"

    # decode step curve at `ctx`
    ctx_blocks = (ctx + 15) // 16
    pages = max(batches) * ctx_blocks
    apool = kvx.Pool(pages, pb, device=device)
    all_ids = torch.arange(pages, dtype=torch.int32, device=dev)
    kvx.fill_pages(apool, all_ids, torch.stack([all_ids * 0, all_ids * 0, all_ids], -1).contiguous(), pages, 1,
                   layout, kvx.FILL_VALUES)
    perm = torch.randperm(pages, device=dev).to(torch.int32)
    weights_ms = 2 * LLAMA8B["params"] / (_hbm_read_gbs(out) * 1e9) * 1e3
    curve: List = []
    for b in batches:
        tables = perm[:b * ctx_blocks].view(b, ctx_blocks).contiguous()
        lens = torch.full((b,), ctx, dtype=torch.int32, device=dev)
        q = (torch.randn(b, 32, 128, device=dev) * 0.5).to(torch.bfloat16)
        o = torch.empty(b, 32, 128, dtype=torch.float32, device=dev)
        att = kvx.Attention(layout, 32, ctx_blocks)
        ws = torch.zeros(max(att.workspace_bytes(b, ctx), 1), dtype=torch.uint8, device=dev)
        t = _time_ms(torch, lambda: [att(apool, tables, lens, q, o, b, ctx, ws) for _ in range(LLAMA8B["layers"])])
        curve.append([b, round(weights_ms + t, 4)])
    out["decode_curve_ms"] = curve
    out["decode_context"] = ctx
    out["weights_ms_estimate"] = weights_ms
    return out


def link_profile(cal: Dict) -> K.LinkProfile:
    lp = K.LinkProfile()
    lp.pcie_bandwidth = min(cal["pcie_h2d_gbs"], cal["pcie_d2h_gbs"]) * 1e9
    lp.network_bandwidth = (cal["nvlink_gbs"] or cal["hbm_page_copy_gbs"]) * 1e9
    return lp


def gpu_profile(cal: Dict, layers: int = 32, kv_bytes_per_token: int = 131_072,
                hbm_capacity: int = 160_000_000_000) -> K.GpuProfile:
    return K.GpuProfile(hbm_capacity=hbm_capacity, kv_bytes_per_token=kv_bytes_per_token, num_layers=layers,
                        decode_curve_ms=[(int(b), float(ms)) for b, ms in cal["decode_curve_ms"]])


def main(argv: Optional[list] = None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/calibration.json")
    ap.add_argument("--ctx", type=int, default=2048)
    args = ap.parse_args(argv)
    cal = measure(ctx=args.ctx)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(cal, f, indent=1)
    print(json.dumps(cal))
    return 0


if __name__ == "__main__":
    sys.exit(main())
