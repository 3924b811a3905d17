"""NVLink peer-copy probe for the K3 mover (run on a box with >= 2 GPUs;
exits cleanly with one). One process, pools on GPU 0 and GPU j: K3 page ->
page into the peer pool with the SM vector mover at several grid caps, the
TMA bulk mover (if stores into peer memory through the TMA units work here),
and copy engines; per-direction GB/s against the measured 770 GB/s
peer-copy peak, every variant verified bit-exact.

usage: python tools/nvlink_probe.py [--pages 16384] [--peer 1]
       (--peer 0 is a same-GPU self-test of the probe: local HBM numbers)
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
    ap.add_argument("--pages", type=int, default=16384)  # 1 GiB of 64 KiB pages
    ap.add_argument("--peer", type=int, default=1)
    args = ap.parse_args()
    if torch.cuda.device_count() <= args.peer:
        print(json.dumps({"skipped": f"needs GPU {args.peer}; {torch.cuda.device_count()} visible"}))
        return 0
    layout = kvx.PageLayout(8, 128, 16, kvx.BF16)
    pb, n = layout.page_bytes(), args.pages
    kvx.check(kvx.lib().kvx_enable_peer_access(0, args.peer))
    src = kvx.Pool(2 * n, pb, device=0)
    dst = kvx.Pool(2 * n, pb, device=args.peer)
    rng = np.random.default_rng(0)
    s_ids = rng.permutation(2 * n)[:n].astype(np.uint32)
    d_ids = rng.permutation(2 * n)[:n].astype(np.uint32)
    dev0 = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    ds = torch.from_numpy(s_ids.view(np.int32)).to(dev0)
    dd = torch.from_numpy(d_ids.view(np.int32)).to(dev0)
    tags = torch.stack([ds * 0, ds * 0, ds], -1).contiguous()
    kvx.fill_pages(src, ds, tags, n, 3, layout, kvx.FILL_BITS)
    st = torch.cuda.Stream(dev0)
    res = {"bytes": n * pb, "peak_gbs": 770.0, "variants": []}

    def run(name, fn, reps=5):
        dst.as_tensor().zero_()
        torch.cuda.synchronize(args.peer)
        fn()
        st.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record(st)
        for _ in range(reps):
            fn()
        e[1].record(st)
        st.synchronize()
        ms = e[0].elapsed_time(e[1]) / reps
        probe = rng.integers(0, n, 256)
        ok = torch.equal(src.as_tensor()[torch.from_numpy(s_ids[probe].astype(np.int64)).to(dev0)].cpu(),
                         dst.as_tensor()[torch.from_numpy(d_ids[probe].astype(np.int64)).to(args.peer)].cpu())
        gbs = n * pb / (ms * 1e-3) / 1e9
        res["variants"].append({"mover": name, "ms": ms, "gbs": gbs, "frac": gbs / 770.0, "verified": ok})

    for cap in (0, 296, 148, 74, 37):
        run(f"sm/{cap or 'all'}", lambda c=cap: kvx.copy_pages(src, ds, dst, dd, n, kvx.COPY_SM, st, max_ctas=c))
    try:
        run("tma", lambda: kvx.copy_pages(src, ds, dst, dd, n, kvx.COPY_TMA, st))
    except Exception as e:  # noqa: BLE001 — stores into peer memory through the TMA units may be unsupported
        res["variants"].append({"mover": "tma", "error": str(e)})
    run("copy-engines", lambda: kvx.copy_pages(src, s_ids, dst, d_ids, n, kvx.COPY_CE, st))
    print(json.dumps(res))
    return 0


if __name__ == "__main__":
    sys.exit(main())
