#!/bin/bash
# A/B over bench.py flag sets: ARGS="--no-workspace|" CONFIGS="ls grad" R=2
IFS='|' read -ra SETS <<< "${ARGS:-}"
for c in ${CONFIGS:-ls}; do
 for r in $(seq ${R:-2}); do
  for s in "${SETS[@]}"; do
   timeout 300 python bench.py $s --config $c --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c [$s] rep $r', round(d['value'],1), 'GB/s', round(d['ms_per_step'],3), 'ms')"
  done
 done
done
