#!/bin/bash
# K4 at batch 1: workspace-merged launches on the 4-warp variant (two CTAs
# per SM, so consecutive launches co-reside and the next one's prologue runs
# under this one's stream) vs the clustered auto plan (diagnostic).
#   tools/k4_batch1_probe2.sh > gpurun_out/k4_b1_v2.log
for hq in 32 64; do
  for ctx in 8192 32768; do
    echo "== hq $hq ctx $ctx auto"
    build/attn_trace 1 $ctx 0 0 $hq 1 | head -1
    for sig in 1 2; do
      for s in 16 18 24 32 36 37; do
        echo "== hq $hq ctx $ctx splits $s global wide signal $sig"
        KVX_ATTN_NARROW=0 KVX_ATTN_SIGNAL=$sig build/attn_trace 1 $ctx $s 1 $hq 1 | head -1
      done
    done
  done
done
echo "== detail hq 32 ctx 8192 splits 18 wide signal 2"
KVX_ATTN_NARROW=0 KVX_ATTN_SIGNAL=2 build/attn_trace 1 8192 18 1 32 1
