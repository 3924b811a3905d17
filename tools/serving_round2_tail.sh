mkdir -p /tmp/serve_disk
for pol in swap recompute retain; do
  timeout 900 oracle/_ref/serve_gpu --config 4 --users 192 --policies $pol --sessions 320 --nodes 2 --device-gb 32 --host-gb 16 --disk-dir /tmp/serve_disk | grep '"policy"' >> gpurun_out/serve_c4_192.jsonl; echo "c4 192 $pol rc=$?" >&2; rm -f /tmp/serve_disk/*
done
CELL_TIMEOUT=700 tools/serving_sweep.sh 5 gpurun_out/serve_c5_tight.jsonl "32 96 192" --sessions 240 --nodes 2 --device-gb 8 --host-gb 16
