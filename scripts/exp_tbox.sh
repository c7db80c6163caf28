#!/bin/bash
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
P='import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], round(d["value"],1), "GB/s", round(d["ms_per_step"],3), "ms")'
for c in ${CONFIGS:-sweepT_k4_s4_bf16 grad ls}; do
 for bn in ${BNS:-256}; do
  BPS_TC_BN=$bn timeout 300 python bench.py --layout t --config $c $B 2>/dev/null | python -c "$P" "T $c bn=$bn kg=1"
  for kg in ${KGS:-2 4}; do for tb in ${TBS:-8 16 32 64}; do
   BPS_TC_BN=$bn BPS_TC_KGROUP=$kg BPS_TC_TBOX=$tb timeout 300 python bench.py --layout t --config $c $B 2>/dev/null | python -c "$P" "T $c bn=$bn kg=$kg tb=$tb"
  done; done
 done
done
