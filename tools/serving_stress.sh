#!/usr/bin/env bash
# Stress: configs 4 / 5 traffic with real pages (payload_sim) vs the reference store (payload_sim_ref), several sizes, policies and payload modes (lockstep, free-running, free-running with the DISK tier in files). Run on a B200: tools/serving_stress.sh
cd "$(dirname "$0")/.."
D=$(mktemp -d /tmp/kvdisk.XXXX)
run() {
  ref=$(oracle/_ref/payload_sim_ref "$@" --digest 2>&1 | grep -E "^digest|^migrate")
  for m in "" "--free-running" "--free-running --disk-dir $D"; do
    out=$(oracle/_ref/payload_sim "$@" --digest $m 2>&1)
    got=$(echo "$out" | grep -E "^digest|^migrate")
    ver=$(echo "$out" | grep "verified_copies")
    if [ "$ref" == "$got" ]; then st=MATCH; else st=DIFF; fi
    echo "$* [$m] $st | $ver | $(echo "$got" | head -1)"
    rm -f $D/*
  done
}
run --zipf 1000 --users 500 --nodes 8 --pages 8192
run --zipf 600 --users 300 --nodes 8 --pages 3072
run --sharegpt 600 --users 300 --nodes 8 --pages 8192
run --zipf 400 --users 200 --nodes 4 --pages 4096 --policy swap
run --sharegpt 300 --users 150 --nodes 4 --pages 8192
run --zipf 300 --users 100 --nodes 2 --pages 16384
rm -rf $D
