"""PCIe page movers on fragmented pools: a 1 GiB session of scattered 64 KiB
HBM pages to / from scattered pages of a pinned, device-mapped HOST pool —
copy engines (one descriptor per run of consecutive ids), the SM vector
mover storing straight into mapped host memory, and the TMA mover — so the
HOST-tier moves (SwapOut / HostCopy / LoadH2D) can pick the mover that does
not collapse when free lists are fragmented — one direction at a time, then
both at once (the ceiling for a swap). Bytes verified.

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
        # Both directions at once (what a swap — offload one session while
        # loading another — sees): half the pages go down, half come up, on
        # two streams; GB/s counts both directions.
        half = n // 2
        st2 = torch.cuda.Stream(dev)
        for name, down_mode, up_mode in (("ce+ce", kvx.COPY_CE, kvx.COPY_CE), ("ce-d2h+sm-h2d", kvx.COPY_CE, kvx.COPY_SM),
                                         ("sm-d2h+ce-h2d", kvx.COPY_SM, kvx.COPY_CE)):
            def ids(mode, a, sl):  # host ids for the copy engines, device ids for the SM mover
                return (np.ascontiguousarray(a[sl]) if mode == kvx.COPY_CE else
                        torch.from_numpy(np.ascontiguousarray(a[sl]).view(np.int32)).to(dev))
            down = (ids(down_mode, d_ids, slice(0, half)), ids(down_mode, h_ids, slice(0, half)))
            up = (ids(up_mode, h_ids, slice(half, n)), ids(up_mode, d_ids, slice(half, n)))

            def both():
                kvx.copy_pages(dpool, down[0], hpool, down[1], half, down_mode, st)
                kvx.copy_pages(hpool, up[0], dpool, up[1], n - half, up_mode, st2)
            try:
                kvx.fill_pages(dpool, dd, torch.stack([dd * 0, dd * 0, dd], -1).contiguous(), n, 5, layout,
                               kvx.FILL_BITS)
                torch.cuda.synchronize(dev)
                both()
                torch.cuda.synchronize(dev)
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record(st)
                st2.wait_event(e[0])
                for _ in range(3):
                    both()
                e[1].record(st2)
                st.wait_event(e[1])
                e[2].record(st)
                torch.cuda.synchronize(dev)
                ms = e[0].elapsed_time(e[2]) / 3
                hp = hpool.as_tensor().numpy()
                dp = dpool.as_tensor()
                probe = rng.integers(0, n, 64)
                ok = bool(np.array_equal(hp[h_ids[probe]],
                                         dp[torch.from_numpy(d_ids[probe].astype(np.int64)).to(dev)].cpu().numpy()))
                res.setdefault("bidirectional", []).append(
                    {"pool": frag, "movers": name, "ms": round(ms, 3), "gbs": round(n * pb / (ms * 1e-3) / 1e9, 1),
                     "verified": ok})
            except Exception as ex:  # noqa: BLE001
                res.setdefault("bidirectional", []).append({"pool": frag, "movers": name, "error": str(ex)[:200]})
    print(json.dumps(res))
    return 0


if __name__ == "__main__":
    sys.exit(main())
