#!/bin/bash
# Decode-step time of the serving engine's Llama-3.1-8B-shaped step (batch
# 1..64 at ctx 1024), projections on K7 (default) vs cuBLAS (KVX_MODEL_SKINNY=0),
# plus a per-kernel launch list of two batch-1 steps under ncu (diagnostic).
#   tools/model_step_probe.sh gpurun_out/model_step
OUT=${1:-gpurun_out/model_step}
mkdir -p "$(dirname "$OUT")"
for s in 1 0; do
  echo "== KVX_MODEL_SKINNY=$s"
  KVX_MODEL_SKINNY=$s oracle/_ref/serve_gpu --calibrate-only
done > "$OUT.txt" 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT.ncu.csv" \
  oracle/_ref/serve_gpu --profile-batch 1 --profile-steps 2 > /dev/null 2>&1
