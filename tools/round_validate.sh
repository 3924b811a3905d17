#!/bin/bash
# End-of-round validation on one B200 (run under gpurun): smoke, the GPU
# suite, the bench (both arms), the launch list of the bench under ncu, and
# one ncu --set full capture each of the dominant movers and K4 at batch 1.
# Outputs in gpurun_out/final_*. Numbers printed under ncu are never bench values.
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/final_smoke.log 2>&1; echo "smoke rc=$?"
timeout ${SUITE_TIMEOUT:-2400} python -m pytest tests -m gpu -q -p no:cacheprovider > $O/final_gpu_suite.log 2>&1; echo "suite rc=$?"
timeout 900 python bench.py > $O/final_bench.json 2> $O/final_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/final_bench_ref.json 2> $O/final_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/final_launches.csv \
  python bench.py --steps 2 --warmup 3 --skip-cpu --skip-overlap > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:page_move_bulk -s 4 -c 1 \
  -o $O/final_ncu_pack -f python bench.py --steps 1 --warmup 3 --skip-cpu --skip-attention --skip-e2e --skip-overlap > /dev/null 2>&1; echo "ncu pack rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bf16 -s 3 -c 1 \
  -o $O/final_ncu_attn_b1 -f python tools/profile_attn.py 1 8192 > /dev/null 2>&1; echo "ncu attn rc=$?"
