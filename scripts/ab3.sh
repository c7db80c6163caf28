#!/bin/bash
# A/B between library builds: LIBS="paper_2602_06071_b200/libbps_old.so|paper_2602_06071_b200/libbps.so"
IFS='|' read -ra SETS <<< "${LIBS}"
for c in ${CONFIGS:-ls}; do
 for r in $(seq ${R:-2}); do
  for s in "${SETS[@]}"; do
   BPS_LIB=$PWD/$s timeout 300 python bench.py ${BENCH_EXTRA} --config $c --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c [$s] rep $r', round(d['value'],1), 'GB/s', round(d['ms_per_step'],3), 'ms')"
  done
 done
done
