#!/bin/bash
# Config 4 on four nodes at light loads (32, 48 users) for symphony / swap /
# recompute, so each policy's p50 range overlaps the others' and requests/s
# at equal p50 can be interpolated (tools/serving_gpu_report.py).
mkdir -p /tmp/serve_disk
for u in 32 48; do
  for pol in symphony swap recompute; do
    timeout 900 oracle/_ref/serve_gpu --config 4 --users $u --policies $pol --sessions 320 --nodes 4 --device-gb 16 \
      --host-gb 8 --disk-dir /tmp/serve_disk | grep '"policy"' >> gpurun_out/serve_c4_n4_low.jsonl
    echo "c4 n4 $u $pol rc=${PIPESTATUS[0]}" >&2
    rm -f /tmp/serve_disk/*
  done
done
