"""Requests/s at equal p50 latency from GPU-executed serving runs.

Input: JSON lines of oracle/_ref/serve_gpu (one per (policy, users) cell:
steady_rps from the reference's report, p50 TTFT / TPOT / normalized
latency from the measured quanta). For each policy the users sweep gives
(p50, req/s) points; at a common p50 SLO a policy's throughput is
interpolated on its latency-sorted points (no extrapolation) — the serving
half of BASELINE.json's metric, "requests/s at equal p50 latency".

usage: python tools/serving_gpu_report.py gpurun_out/serve_gpu_c5.jsonl [--latency norm|tpot|ttft] [--slo a,b,c]
"""
import argparse
import json
import sys
from collections import defaultdict

POLICIES = ("symphony", "retain", "swap", "recompute")
KEYS = {"norm": "norm_latency_ms_per_token", "tpot": "tpot_ms", "ttft": "ttft_ms"}


def load(paths):
    cells = []
    for p in paths:
        for line in open(p):
            line = line.strip()
            if line.startswith("{") and '"policy"' in line and '"error"' not in line:
                cells.append(json.loads(line))
    return cells


def rps_at(points, slo):
    """Interpolated req/s at p50 == slo on the (p50, rps) points sorted by p50."""
    pts = sorted(points)
    for (l0, r0), (l1, r1) in zip(pts, pts[1:]):
        if l0 <= slo <= l1 and l1 > l0:
            return r0 + (r1 - r0) * (slo - l0) / (l1 - l0)
    for l, r in pts:
        if abs(l - slo) < 1e-9:
            return r
    return None


def table(cells, latency):
    key = KEYS[latency]
    rows = ["| policy | users | requests | req/s | p50 TTFT ms | p50 TPOT ms | p50 norm ms/token | decode steps | "
            "mean step ms | migrated GB | pages scrubbed (mismatched) |", "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|"]
    for c in sorted(cells, key=lambda c: (POLICIES.index(c["policy"]), c["users"])):
        rows.append(f"| {c['policy']} | {c['users']} | {c['requests']} | {c['steady_rps']:.2f} | "
                    f"{c['ttft_ms']['p50']:.1f} | {c['tpot_ms']['p50']:.2f} | "
                    f"{c['norm_latency_ms_per_token']['p50']:.2f} | {c['executed']['decode_steps']} | "
                    f"{c['executed']['decode_ms_mean']:.2f} | {c['migrations']['bytes'] / 1e9:.1f} | "
                    f"{c['verify']['pages']} ({c['verify']['mismatched']}) |")
    return "\n".join(rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--latency", default="norm", choices=list(KEYS))
    ap.add_argument("--slo", default="")
    args = ap.parse_args()
    cells = load(args.files)
    if not cells:
        print("no cells")
        return 1
    key = KEYS[args.latency]
    pts = defaultdict(list)
    for c in cells:
        pts[c["policy"]].append((c[key]["p50"], c["steady_rps"]))
    if args.slo:
        slos = [float(x) for x in args.slo.split(",")]
    else:
        lat = sorted({round(p[0], 2) for v in pts.values() for p in v})
        slos = lat[:: max(1, len(lat) // 6)]
    print(table(cells, args.latency))
    print()
    pols = [p for p in POLICIES if p in pts]
    print(f"requests/s at equal p50 {key} (interpolated on each policy's sweep; — = outside its measured range)\n")
    print("| p50 SLO | " + " | ".join(pols) + " |")
    print("|---:|" + "---:|" * len(pols))
    for slo in slos:
        vals = [rps_at(pts[p], slo) for p in pols]
        print(f"| {slo:g} | " + " | ".join(f"{v:.2f}" if v is not None else "—" for v in vals) + " |")
    return 0


if __name__ == "__main__":
    sys.exit(main())
