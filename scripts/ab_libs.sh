#!/bin/bash
# A/B across library builds: LIBS="libbps_old libbps" CONFIGS="..." R=2 bash scripts/ab_libs.sh
B="--steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --no-clocks ${BENCH_EXTRA}"
P='import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], round(d["value"],1), "GB/s", round(d["ms_per_step"],3), "ms")'
for r in $(seq ${R:-2}); do
for c in ${CONFIGS:-ls grad}; do
  for lib in ${LIBS:-libbps}; do
    BPS_LIB=$PWD/paper_2602_06071_b200/$lib.so timeout 300 python bench.py --config $c $B 2>/dev/null | python -c "$P" "$lib $c"
  done
done
done
