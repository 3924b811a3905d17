#!/usr/bin/env bash
# Drop-in proof, test infrastructure: compiles the REFERENCE's own test suites
# and the reference's UNCHANGED callers of the store (Engine, NodeManager,
# ClusterScheduler, Simulation, workload, report, config — all read from
# /root/reference, never copied) against THIS repo's KvStore + cost model, and
# links them into one test binary per suite under build/ref_harness/.
#
# Include resolution: an overlay directory holds only this repo's
# symsim/{kvstore,costmodel,time}.hpp and comes first on the include path, so
# every reference translation unit that includes "symsim/kvstore.hpp" gets the
# B200 build's store; all other symsim headers come from the reference.
#
# With B200_ENGINE=1 the engine is this repo's too (include/symsim/engine.hpp +
# csrc/host/engine.cpp): the reference's test_engine,
# test_simcore, properties and acceptance suites then exercise the B200
# engine (modelled quanta: no executor), built into build/ref_harness_b200eng.
#
# usage: [B200_ENGINE=1] tests/cpp/build_ref_harness.sh [suite ...]   (default: all suites)
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
mkdir -p "$ROOT/build"; exec 9>"$ROOT/build/.lock"; flock 9  # one build at a time (parallel test workers)
REF="${REF:-/root/reference/proj}"
OUT="$ROOT/build/ref_harness"
HDRS=(kvstore costmodel time)
HOST_SRCS=(kvstore costmodel)
REF_SRCS=(engine nodemanager scheduler simcore workload report config)
if [ "${B200_ENGINE:-0}" = 1 ]; then
  OUT="$ROOT/build/ref_harness_b200eng"
  HDRS+=(engine)
  HOST_SRCS+=(engine)
  REF_SRCS=(nodemanager scheduler simcore workload report config)
fi
JSON_DIR="${JSON_DIR:-$(python3 -c 'import os,sysconfig;p=os.path.join(sysconfig.get_paths()["purelib"],"include/cudnn_frontend/thirdparty/nlohmann");print(p)')}"
CXX="${CXX:-g++}"
[ -f "$REF/src/kvstore.cpp" ] || { echo "reference not present at $REF" >&2; exit 3; }
[ -f "$JSON_DIR/json.hpp" ] || { echo "json.hpp not found in $JSON_DIR" >&2; exit 3; }

mkdir -p "$OUT/overlay/symsim" "$OUT/obj"
for h in "${HDRS[@]}"; do
  cmp -s "$ROOT/include/symsim/$h.hpp" "$OUT/overlay/symsim/$h.hpp" || cp "$ROOT/include/symsim/$h.hpp" "$OUT/overlay/symsim/$h.hpp"
done
FLAGS=(-std=c++20 -O2 -I"$OUT/overlay" -I"$REF/include" -I"$JSON_DIR" -I"$ROOT/tests/cpp/doctest" -include unistd.h)

compile() {  # src obj
  if [ ! -f "$2" ] || [ "$1" -nt "$2" ] || [ "$ROOT/include/symsim/kvstore.hpp" -nt "$2" ] ||
     [ "$ROOT/include/symsim/engine.hpp" -nt "$2" ]; then
    "$CXX" "${FLAGS[@]}" -c "$1" -o "$2"
  fi
}

OBJS=()
# this repo's store and cost model
for f in "${HOST_SRCS[@]}"; do
  compile "$ROOT/paper_2412_16434_b200/csrc/host/$f.cpp" "$OUT/obj/b200_$f.o" &
  OBJS+=("$OUT/obj/b200_$f.o")
done
# the reference's callers, unchanged
for f in "${REF_SRCS[@]}"; do
  compile "$REF/src/$f.cpp" "$OUT/obj/ref_$f.o" &
  OBJS+=("$OUT/obj/ref_$f.o")
done
wait

SUITES=("$@")
[ ${#SUITES[@]} -gt 0 ] || SUITES=(test_kvstore test_costmodel test_engine test_scheduler test_simcore test_report test_workload test_properties acceptance)
for t in "${SUITES[@]}"; do
  (
    compile "$REF/tests/$t.cpp" "$OUT/obj/$t.o"
    "$CXX" -o "$OUT/$t" "$OUT/obj/$t.o" "${OBJS[@]}"
  ) &
done
wait
echo "built: ${SUITES[*]} -> $OUT"
