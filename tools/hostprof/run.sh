#!/bin/bash
# Host-only profile of the store-path migration (no GPU): builds KvStore +
# NodePayload + costmodel with tools/hostprof/kvx_stub.cpp in place of libkvx,
# runs tools/hostprof/store_path_host.cpp, prints per-layer host us and, with
# PROF=1, a gprof flat profile. DIAGNOSTIC ONLY.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
OUT="$ROOT/build/hostprof"
mkdir -p "$OUT"
FLAGS=(-std=c++20 -O2 -g -I"$ROOT/include" -I/usr/local/cuda/include)
[ "${PROF:-0}" = 1 ] && FLAGS+=(-pg)
g++ "${FLAGS[@]}" "$ROOT/tools/hostprof/store_path_host.cpp" "$ROOT/tools/hostprof/kvx_stub.cpp" \
  "$ROOT/paper_2412_16434_b200/csrc/host/kvstore.cpp" "$ROOT/paper_2412_16434_b200/csrc/host/payload.cpp" \
  "$ROOT/paper_2412_16434_b200/csrc/host/costmodel.cpp" -o "$OUT/store_path_host"
cd "$OUT" && ./store_path_host "${REPS:-5}"
[ "${PROF:-0}" = 1 ] && gprof -b -p "$OUT/store_path_host" gmon.out | head -40 || true
