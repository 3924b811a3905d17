"""Requests/s at equal p50 latency (the serving half of BASELINE.json's
metric) from `serve_sim sweep` outputs: for each policy, the users sweep gives
(p50 normalized latency, steady requests/s) points; at a common p50 SLO the
policy's throughput is interpolated on its latency-sorted points (no
extrapolation past the measured range).

usage: python tools/serving_equal_p50.py profiles/serve_loaded_c4_u*.txt [--slo 4,5,6,8]
"""
import argparse
import json
import sys
from collections import defaultdict


def load(paths):
    cells = defaultdict(list)
    config = None
    for p in paths:
        for line in open(p):
            if line.startswith("{"):
                d = json.loads(line)
                config = d["config"]
                for c in d["cells"]:
                    cells[c["policy"]].append((c["p50_norm_ms"], c["rps"], c["users"], c["p50_ttft_s"]))
    return config, cells


def rps_at(points, slo):
    pts = sorted(points)
    best = None
    for (l0, r0, *_), (l1, r1, *_) in zip(pts, pts[1:]):
        if l0 <= slo <= l1 and l1 > l0:
            best = r0 + (r1 - r0) * (slo - l0) / (l1 - l0)
    if best is None and pts and abs(pts[0][0] - slo) < 1e-9:
        best = pts[0][1]
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--slo", default="4,5,6,8,12")
    args = ap.parse_args()
    config, cells = load(args.files)
    slos = [float(x) for x in args.slo.split(",")]
    policies = [p for p in ("symphony", "retain", "swap", "recompute") if p in cells]
    print(f"config {config}: requests/s at equal p50 normalized latency (ms/token)\n")
    print("| p50 SLO | " + " | ".join(policies) + " | symphony / recompute |")
    print("|---:|" + "---:|" * (len(policies) + 1))
    for slo in slos:
        vals = [rps_at(cells[p], slo) for p in policies]
        ratio = (vals[0] / vals[-1]) if vals[0] and vals[-1] else None
        fmt = lambda v: f"{v:.1f}" if v is not None else "—"
        print(f"| {slo:g} | " + " | ".join(fmt(v) for v in vals) + f" | {fmt(ratio)}{'×' if ratio else ''} |")
    return 0


if __name__ == "__main__":
    sys.exit(main())
