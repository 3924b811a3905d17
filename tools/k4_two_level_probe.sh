#!/bin/bash
# K4 at small batch: one cluster per (request, kv head) (auto) vs G clusters
# of C CTAs with the cross-cluster merge in the workspace (KVX_ATTN_CLUSTERS),
# 8B / 70B shapes at 8K and 32K (diagnostic; flags 1 = early prefetch).
#   tools/k4_two_level_probe.sh > gpurun_out/k4_two_level.log
for hq in 32 64; do
  for ctx in 8192 32768; do
    for b in 1 2; do
      echo "== hq $hq ctx $ctx batch $b auto"; build/attn_trace $b $ctx 0 0 $hq 1 | head -1
      for sg in "12 2" "16 2" "18 2" "20 2" "15 3" "18 3" "16 4" "20 4" "24 4" "24 6"; do
        set -- $sg
        echo "== hq $hq ctx $ctx batch $b splits $1 groups $2"
        build/attn_trace $b $ctx $1 0 $hq $((1 + 256 * $2)) | head -1
      done
    done
  done
done
