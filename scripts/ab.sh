#!/bin/bash
# A/B: alternate env settings in one session, R repetitions each (production build)
# usage: AB="BPS_TC_GROUP=32|BPS_TC_GROUP=128" CONFIGS="ls grad" R=3 bash scripts/ab.sh
IFS='|' read -ra SETS <<< "${AB:-X=0}"
for c in ${CONFIGS:-ls}; do
 for r in $(seq ${R:-3}); do
  for s in "${SETS[@]}"; do
   env $s timeout 300 python bench.py ${BENCH_EXTRA} --config $c --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c [$s] rep $r', round(d['value'],1), 'GB/s', round(d['ms_per_step'],3), 'ms')"
  done
 done
done
