#!/usr/bin/env bash
# Seeded stress of the store + payload against the reference store: configs 4 / 5
# traffic with real pages for many trace seeds, lockstep and free-running. Where
# the reference itself throws (e.g. its ensure_room device-pressure error), the
# product must throw the same error. Run on a B200: tools/seed_stress.sh [N]
cd "$(dirname "$0")/.."
N=${1:-8}
pass=0; fail=0
for kind in zipf sharegpt; do
  for seed in $(seq 1 $N); do
    args="--$kind 300 --users 150 --nodes 8 --pages 4096 --seed $((seed * 7919)) --digest"
    ref=$(oracle/_ref/payload_sim_ref $args 2>&1); rrc=$?
    for m in "" "--free-running"; do
      out=$(oracle/_ref/payload_sim $args $m 2>&1); prc=$?
      if [ $rrc -ne 0 ]; then
        re=$(echo "$ref" | grep "what()" | sed 's/.*what():  //' | cut -c1-80)
        pe=$(echo "$out" | grep "what()" | sed 's/.*what():  //' | cut -c1-80)
        if [ $prc -ne 0 ] && [ "$re" == "$pe" ]; then st=SAME_ERROR; pass=$((pass+1)); else st="ERROR_DIFF[$re|$pe]"; fail=$((fail+1)); fi
      else
        a=$(echo "$ref" | grep -E "^digest|^migrate"); b=$(echo "$out" | grep -E "^digest|^migrate")
        v=$(echo "$out" | grep -o "mismatches [0-9]*")
        if [ "$a" == "$b" ] && [ "$v" == "mismatches 0" ]; then st="MATCH($v)"; pass=$((pass+1)); else st="DIFF($v)"; fail=$((fail+1)); fi
      fi
      echo "$kind seed=$((seed * 7919)) [$m] $st"
    done
  done
done
echo "pass=$pass fail=$fail"
