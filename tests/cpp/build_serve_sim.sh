#!/usr/bin/env bash
# Builds tests/cpp/serve_sim.cpp twice into oracle/_ref/ (TEST / MEASUREMENT
# INFRASTRUCTURE linking reference sources compiled from /root/reference):
#   oracle/_ref/serve_sim      this repo's KvStore + cost model + Engine
#   oracle/_ref/serve_sim_ref  the reference KvStore + cost model
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
mkdir -p "$ROOT/build"; exec 9>"$ROOT/build/.lock"; flock 9  # one build at a time (parallel test workers)
REF="${REF:-/root/reference/proj}"
OUT="$ROOT/oracle/_ref"
OBJ="$ROOT/build/serve_sim"
JSON_DIR="${JSON_DIR:-$(python3 -c 'import os,sysconfig;print(os.path.join(sysconfig.get_paths()["purelib"],"include/cudnn_frontend/thirdparty/nlohmann"))')}"
CXX="${CXX:-g++}"
[ -f "$REF/src/kvstore.cpp" ] || { echo "reference not present at $REF" >&2; exit 3; }
mkdir -p "$OUT" "$OBJ/overlay/symsim"
for h in kvstore costmodel time engine; do  # unchanged headers stay put; changed ones are replaced atomically (parallel test workers)
  d="$OBJ/overlay/symsim/$h.hpp"
  cmp -s "$ROOT/include/symsim/$h.hpp" "$d" || { cp "$ROOT/include/symsim/$h.hpp" "$d.$$" && mv -f "$d.$$" "$d"; }
done
P=(-std=c++20 -O2 -I"$OBJ/overlay" -I"$REF/include" -I"$JSON_DIR")
R=(-std=c++20 -O2 -I"$REF/include" -I"$JSON_DIR")
pids=()
rm -f "$OBJ"/p_*.o "$OBJ"/b_*.o
for f in nodemanager scheduler simcore workload report config; do
  "$CXX" "${P[@]}" -c "$REF/src/$f.cpp" -o "$OBJ/p_$f.o" & pids+=($!)
done
for f in engine nodemanager scheduler simcore workload report config; do
  "$CXX" "${R[@]}" -c "$REF/src/$f.cpp" -o "$OBJ/r_$f.o" & pids+=($!)
done
"$CXX" "${P[@]}" -c "$ROOT/paper_2412_16434_b200/csrc/host/engine.cpp" -o "$OBJ/b_engine.o" & pids+=($!)
for f in kvstore costmodel; do
  "$CXX" "${P[@]}" -c "$ROOT/paper_2412_16434_b200/csrc/host/$f.cpp" -o "$OBJ/b_$f.o" & pids+=($!)
  "$CXX" "${R[@]}" -c "$REF/src/$f.cpp" -o "$OBJ/r_$f.o" & pids+=($!)
done
# product traffic generators (include/symsim/traffic.hpp) for both builds
"$CXX" "${P[@]}" -I"$ROOT/include" -c "$ROOT/paper_2412_16434_b200/csrc/host/traffic.cpp" -o "$OBJ/b_traffic.o" & pids+=($!)
"$CXX" "${R[@]}" -I"$ROOT/include" -c "$ROOT/paper_2412_16434_b200/csrc/host/traffic.cpp" -o "$OBJ/r_traffic.o" & pids+=($!)
"$CXX" "${P[@]}" -I"$ROOT/include" -c "$ROOT/tests/cpp/serve_sim.cpp" -o "$OBJ/main_p.o" & pids+=($!)
"$CXX" "${R[@]}" -I"$ROOT/include" -c "$ROOT/tests/cpp/serve_sim.cpp" -o "$OBJ/main_r.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
"$CXX" -o "$OUT/serve_sim" "$OBJ/main_p.o" "$OBJ"/p_*.o "$OBJ"/b_*.o
"$CXX" -o "$OUT/serve_sim_ref" "$OBJ/main_r.o" "$OBJ"/r_*.o
echo "built $OUT/serve_sim $OUT/serve_sim_ref"
