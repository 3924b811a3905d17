#!/bin/bash
# K4 at batch 1 (Llama-3.1-8B and 70B KV shapes): where one launch's time goes
# for the auto plan and for fixed split counts / merges / PDL signal points
# (diagnostic; needs build/attn_trace and build/cluster_probe, see their headers).
#   tools/k4_batch1_probe.sh > gpurun_out/k4_b1.log
build/cluster_probe
for hq in 32 64; do
  for ctx in 8192 32768; do
    for tma in 1 0; do
      echo "== hq $hq ctx $ctx auto tma=$tma"
      KVX_ATTN_TMA=$tma build/attn_trace 1 $ctx 0 0 $hq 1
    done
    for sig in 0 1 2; do
      for s in 0 6 8 9 10; do
        echo "== hq $hq ctx $ctx splits $s cluster/auto signal $sig"
        KVX_ATTN_SIGNAL=$sig build/attn_trace 1 $ctx $s 0 $hq 1 | head -1
      done
      for s in 9 12 16 18 24 36; do
        echo "== hq $hq ctx $ctx splits $s global signal $sig"
        KVX_ATTN_SIGNAL=$sig build/attn_trace 1 $ctx $s 1 $hq 1 | head -1
      done
    done
  done
done
