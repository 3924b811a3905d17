#!/usr/bin/env bash
# compute-sanitizer over the kvx kernels (memcheck / racecheck /
# synccheck on K1-K5). Small shapes; writes summaries to gpurun_out/.
cd "$(dirname "$0")/.."
OUT=gpurun_out
mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python tools/sanitize_driver.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool exit $? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|No hazards|hazard' $OUT/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
