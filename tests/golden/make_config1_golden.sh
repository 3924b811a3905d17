#!/usr/bin/env bash
# Regenerates tests/golden/config1_*.txt: the reference KvStore (state oracle)
# under the reference Simulation on the config-1 trace, built by
# tests/cpp/build_payload_sim.sh as oracle/_ref/payload_sim_ref.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
BIN="$ROOT/oracle/_ref/payload_sim_ref"
[ -x "$BIN" ] || "$ROOT/tests/cpp/build_payload_sim.sh"
"$BIN" > "$ROOT/tests/golden/config1_default.txt"
"$BIN" --device-pages 30 > "$ROOT/tests/golden/config1_dev30.txt"
"$BIN" --device-pages 40 > "$ROOT/tests/golden/config1_dev40.txt"
"$BIN" --policy swap > "$ROOT/tests/golden/config1_swap.txt"
wc -l "$ROOT"/tests/golden/config1_*.txt
