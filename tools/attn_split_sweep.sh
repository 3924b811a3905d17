#!/bin/bash
# Split-K sweep of K4 at long context for both GQA shapes (diagnostic):
# one JSON line per (q heads, batch, ctx, splits, merge) from build/attn_trace.
#   tools/attn_split_sweep.sh > gpurun_out/split_sweep.jsonl
for hq in 32 64; do
  for b in 1 2 4 8 16; do
    for ctx in 8192 32768; do
      for s in 0 1 2 3 4 6 8 9 12 16 18 24; do
        for m in 0 1; do
          build/attn_trace $b $ctx $s $m $hq 2>/dev/null | head -1
        done
      done
    done
  done
done
