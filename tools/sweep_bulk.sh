#!/usr/bin/env bash
# Tuning sweep of the TMA page mover geometry (chunk bytes x stages x CTAs/SM).
cd "$(dirname "$0")/.."
for cfg in ${CFGS:-"32768 6 1" "32768 4 1" "32768 5 1" "65536 3 1" "16384 4 3" "32768 4 1" "32768 6 1"}; do
  set -- $cfg
  out=$(KVX_BULK_CHUNK=$1 KVX_BULK_STAGES=$2 KVX_BULK_CTAS_PER_SM=$3 python bench.py --steps 200 --warmup 3 \
        --skip-attention --skip-e2e --skip-cpu --skip-overlap --copy-mode tma 2>/dev/null | tail -1)
  echo "$cfg $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); x=d['detail']; print(round(x['pack_hbm_gbs']), round(x['unpack_hbm_gbs']), round(x['fused_copy_hbm_gbs']))")"
done
