"""PCIe page movers on fragmented pools: a 1 GiB session of scattered 64 KiB
HBM pages to / from scattered pages of a pinned, device-mapped HOST pool —
copy engines (one descriptor per run of consecutive ids), the SM vector
mover storing straight into mapped host memory, and the TMA mover — so the
HOST-tier moves (SwapOut / HostCopy / LoadH2D) can pick the mover that does
not collapse when free lists are fragmented. Bytes verified.

usage: python tools/pcie_mover_probe.py [--pages 16384]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_16434_b200 import kvx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pages", type=int, default=16384)
    args = ap.parse_args()
    layout = kvx.PageLayout(8, 128, 16, kvx.BF16)
    pb, n = layout.page_bytes(), args.pages
    dev = torch.device("cuda", 0)
    dpool = kvx.Pool(2 * n, pb, device=0)
    hpool = kvx.Pool(2 * n, pb, host=True)
    rng = np.random.default_rng(1)
    res = {"bytes": n * pb, "variants": []}
    for frag in ("contiguous", "fragmented"):
        if frag == "contiguous":
            d_ids = np.arange(n, dtype=np.uint32)
            h_ids = np.arange(n, dtype=np.uint32)
        else:
            d_ids = rng.permutation(2 * n)[:n].astype(np.uint32)
            h_ids = rng.permutation(2 * n)[:n].astype(np.uint32)
        dd = torch.from_numpy(d_ids.view(np.int32)).to(dev)
        dh = torch.from_numpy(h_ids.view(np.int32)).to(dev)
        kvx.fill_pages(dpool, dd, torch.stack([dd * 0, dd * 0, dd], -1).contiguous(), n, 5, layout, kvx.FILL_BITS)
        st = torch.cuda.Stream(dev)
        for name, mode in (("copy-engines", kvx.COPY_CE), ("sm-zero-copy", kvx.COPY_SM), ("tma", kvx.COPY_TMA)):
            for direction in ("d2h", "h2d"):
                def go():
                    if direction == "d2h":
                        if mode == kvx.COPY_CE:
                            kvx.copy_pages(dpool, d_ids, hpool, h_ids, n, mode, st)
                        else:
                            kvx.copy_pages(dpool, dd, hpool, dh, n, mode, st)
                    else:
                        if mode == kvx.COPY_CE:
                            kvx.copy_pages(hpool, h_ids, dpool, d_ids, n, mode, st)
                        else:
                            kvx.copy_pages(hpool, dh, dpool, dd, n, mode, st)
                try:
                    go()
                    st.synchronize()
                    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                    e[0].record(st)
                    for _ in range(3):
                        go()
                    e[1].record(st)
                    st.synchronize()
                    ms = e[0].elapsed_time(e[1]) / 3
                    probe = rng.integers(0, n, 64)
                    ok = bool(np.array_equal(
                        hpool.as_tensor().numpy()[h_ids[probe]],
                        dpool.as_tensor()[torch.from_numpy(d_ids[probe].astype(np.int64)).to(dev)].cpu().numpy()))
                    res["variants"].append({"pool": frag, "mover": name, "dir": direction, "ms": round(ms, 3),
                                            "gbs": round(n * pb / (ms * 1e-3) / 1e9, 1), "verified": ok})
                except Exception as ex:  # noqa: BLE001 — a mover that cannot reach mapped host memory
                    res["variants"].append({"pool": frag, "mover": name, "dir": direction, "error": str(ex)[:200]})
    print(json.dumps(res))
    return 0


if __name__ == "__main__":
    sys.exit(main())
