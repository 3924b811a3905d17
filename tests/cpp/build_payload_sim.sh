#!/usr/bin/env bash
# Builds the config-1 parity harness (tests/cpp/payload_sim.cpp) twice into
# oracle/_ref/ — TEST INFRASTRUCTURE that links reference sources compiled from
# /root/reference (never copied), so it is built here and shipped prebuilt to
# the GPU box (oracle/_ref is git-ignored, not gpurun-ignored):
#   oracle/_ref/payload_sim      this repo's KvStore + NodePayload + libkvx
#                                under the reference's unchanged Simulation
#   oracle/_ref/payload_sim_ref  the reference KvStore (state oracle, CPU only)
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
mkdir -p "$ROOT/build"; exec 9>"$ROOT/build/.lock"; flock 9  # one build at a time (parallel test workers)
REF="${REF:-/root/reference/proj}"
OUT="$ROOT/oracle/_ref"
OBJ="$ROOT/build/payload_sim"
JSON_DIR="${JSON_DIR:-$(python3 -c 'import os,sysconfig;print(os.path.join(sysconfig.get_paths()["purelib"],"include/cudnn_frontend/thirdparty/nlohmann"))')}"
CXX="${CXX:-g++}"
CC_SYS="$(command -v /usr/bin/gcc || command -v gcc)"
[ -f "$REF/src/kvstore.cpp" ] || { echo "reference not present at $REF" >&2; exit 3; }
mkdir -p "$OUT" "$OBJ/overlay/symsim"
for h in kvstore costmodel time; do  # unchanged headers stay put; changed ones are replaced atomically (parallel test workers)
  d="$OBJ/overlay/symsim/$h.hpp"
  cmp -s "$ROOT/include/symsim/$h.hpp" "$d" || { cp "$ROOT/include/symsim/$h.hpp" "$d.$$" && mv -f "$d.$$" "$d"; }
done
make -s -C "$ROOT/paper_2412_16434_b200/csrc" all

CUDA_INC="${CUDA_HOME:-/usr/local/cuda}/include"
PROD_FLAGS=(-std=c++20 -O2 -DWITH_PAYLOAD -I"$OBJ/overlay" -I"$REF/include" -I"$ROOT/include" -I"$CUDA_INC" -I"$JSON_DIR")
REF_FLAGS=(-std=c++20 -O2 -I"$REF/include" -I"$JSON_DIR")

pids=()
for f in engine nodemanager scheduler simcore workload report config; do
  "$CXX" "${PROD_FLAGS[@]}" -c "$REF/src/$f.cpp" -o "$OBJ/p_$f.o" & pids+=($!)
  "$CXX" "${REF_FLAGS[@]}" -c "$REF/src/$f.cpp" -o "$OBJ/r_$f.o" & pids+=($!)
done
for f in kvstore costmodel payload; do
  "$CXX" "${PROD_FLAGS[@]}" -c "$ROOT/paper_2412_16434_b200/csrc/host/$f.cpp" -o "$OBJ/b_$f.o" & pids+=($!)
done
for f in kvstore costmodel; do
  "$CXX" "${REF_FLAGS[@]}" -c "$REF/src/$f.cpp" -o "$OBJ/r_$f.o" & pids+=($!)
done
"$CXX" "${PROD_FLAGS[@]}" -c "$ROOT/tests/cpp/payload_sim.cpp" -o "$OBJ/main_p.o" & pids+=($!)
"$CXX" "${REF_FLAGS[@]}" -c "$ROOT/tests/cpp/payload_sim.cpp" -o "$OBJ/main_r.o" & pids+=($!)
"$CC_SYS" -std=c11 -O2 -ffp-contract=off -c "$ROOT/oracle/kvx_oracle.c" -o "$OBJ/kvx_oracle.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done

"$CXX" -o "$OUT/payload_sim" "$OBJ/main_p.o" "$OBJ"/p_*.o "$OBJ"/b_*.o "$OBJ/kvx_oracle.o" \
  -L"$ROOT/paper_2412_16434_b200/lib" -lkvx -Wl,-rpath,'$ORIGIN/../../paper_2412_16434_b200/lib' -lm
"$CXX" -o "$OUT/payload_sim_ref" "$OBJ/main_r.o" "$OBJ"/r_*.o
echo "built $OUT/payload_sim $OUT/payload_sim_ref"
