#!/usr/bin/env bash
# Builds tests/cpp/serve_gpu.cpp into oracle/_ref/serve_gpu — MEASUREMENT
# INFRASTRUCTURE linking the reference's unchanged Simulation / NodeManager /
# ClusterScheduler / workload / report / config sources compiled from
# /root/reference (never copied) with this repo's KvStore, Engine, payload and
# GPU step executor (libsymsim_b200 + libkvx). Built here, shipped prebuilt.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
mkdir -p "$ROOT/build"; exec 9>"$ROOT/build/.lock"; flock 9  # one build at a time (parallel test workers)
REF="${REF:-/root/reference/proj}"
OUT="$ROOT/oracle/_ref"
OBJ="$ROOT/build/serve_gpu"
JSON_DIR="${JSON_DIR:-$(python3 -c 'import os,sysconfig;print(os.path.join(sysconfig.get_paths()["purelib"],"include/cudnn_frontend/thirdparty/nlohmann"))')}"
CXX="${CXX:-g++}"
[ -f "$REF/src/kvstore.cpp" ] || { echo "reference not present at $REF" >&2; exit 3; }
make -s -C "$ROOT/paper_2412_16434_b200/csrc" all
mkdir -p "$OUT" "$OBJ/overlay/symsim"
for h in kvstore costmodel time engine; do  # unchanged headers stay put; changed ones are replaced atomically (parallel test workers)
  d="$OBJ/overlay/symsim/$h.hpp"
  cmp -s "$ROOT/include/symsim/$h.hpp" "$d" || { cp "$ROOT/include/symsim/$h.hpp" "$d.$$" && mv -f "$d.$$" "$d"; }
done
CUDA_INC="${CUDA_HOME:-/usr/local/cuda}/include"
P=(-std=c++20 -O2 -I"$OBJ/overlay" -I"$REF/include" -I"$ROOT/include" -I"$CUDA_INC" -I"$JSON_DIR")
pids=()
for f in nodemanager scheduler simcore workload report config; do
  "$CXX" "${P[@]}" -c "$REF/src/$f.cpp" -o "$OBJ/r_$f.o" & pids+=($!)
done
"$CXX" "${P[@]}" -c "$ROOT/tests/cpp/serve_gpu.cpp" -o "$OBJ/main.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
"$CXX" -o "$OUT/serve_gpu" "$OBJ/main.o" "$OBJ"/r_*.o -L"$ROOT/paper_2412_16434_b200/lib" -lsymsim_b200 -lkvx \
  -Wl,-rpath,'$ORIGIN/../../paper_2412_16434_b200/lib'
echo "built $OUT/serve_gpu"
