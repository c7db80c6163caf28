#!/bin/bash
# trace hash-bound sweep points; transposed pad test; band depth 6
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
P='import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], round(d["value"],1), "GB/s", round(d["ms_per_step"],3), "ms")'
for pad in 0 64 1024; do
  timeout 300 python bench.py --layout t --config grad --t-pad $pad $B 2>/dev/null | python -c "$P" "T grad pad=$pad"
  timeout 300 python bench.py --layout t --config sweepT_k4_s4_bf16 --t-pad $pad $B 2>/dev/null | python -c "$P" "T sweepT_k4_s4 pad=$pad"
done
for c in sweepT_k16_s4_bf16 sweepT_k8_s8_bf16 sweepT_k16_s2_bf16 sweepT_k8_s4_f32 grad ls; do
  for lib in libbps libbps_nb6; do
    BPS_LIB=$PWD/paper_2602_06071_b200/$lib.so timeout 300 python bench.py --config $c $B 2>/dev/null | python -c "$P" "$lib $c"
  done
done
BPS_TC_DEBUG=8 timeout 300 python scripts/tc_trace.py sweepT_k16_s4_bf16 sweepT_k8_s8_bf16 grad 2>&1 | grep -v Warn
