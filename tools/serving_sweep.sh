#!/bin/bash
# Requests/s at equal p50 latency on the B200 (BASELINE.json's serving half):
# the reference's unchanged Simulation driving this repo's store + payload +
# GPU-executed engine (oracle/_ref/serve_gpu), one JSON line per (policy,
# users) cell appended to $OUT as it finishes; summarise with
#   python tools/serving_gpu_report.py $OUT
# usage: tools/serving_sweep.sh CONFIG OUT "USERS..." [extra serve_gpu args]
#   e.g. tools/serving_sweep.sh 5 gpurun_out/serve_c5.jsonl "32 96 192" --sessions 240
CONFIG=$1; OUT=$2; USERS=$3; shift 3
mkdir -p /tmp/serve_disk "$(dirname "$OUT")"
for u in $USERS; do
  for pol in symphony retain swap recompute; do
    timeout "${CELL_TIMEOUT:-1200}" oracle/_ref/serve_gpu --config "$CONFIG" --users "$u" --policies "$pol" \
      --disk-dir /tmp/serve_disk "$@" | grep '"policy"' >> "$OUT"
    echo "config $CONFIG users $u $pol rc=${PIPESTATUS[0]}" >&2
    rm -f /tmp/serve_disk/*
  done
done
