#!/bin/bash
# A/B between the working tree and an exported older tree in ab_old/ (same bench command).
for c in ${CONFIGS:-ls}; do
 for r in $(seq ${R:-2}); do
  for t in . ab_old; do
   (cd $t && timeout 300 python bench.py ${BENCH_EXTRA} --config $c --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null) | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c [$t] rep $r', round(d['value'],1), 'GB/s', round(d['ms_per_step'],3), 'ms')"
  done
 done
done
