#!/bin/bash
# round-1 follow-up experiments: transposed K-grouping, hash-bound sweep points
mkdir -p gpurun_out
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks"
run() { # label, env..., -- bench args
  local lab="$1"; shift
  env "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', round(d['value'],1), 'GB/s', round(d['ms_per_step'],3), 'ms')" 
}
for r in 1 2; do
for c in grad ls sweepT_k4_s4_bf16; do
 for bn in 256 128; do
  for kg in 1 2 4 8; do
   BPS_TC_BN=$bn BPS_TC_KGROUP=$kg timeout 300 python bench.py --layout t --config $c $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('T $c bn=$bn kg=$kg', round(d['value'],1), 'GB/s', round(d['ms_per_step'],3), 'ms')"
  done
 done
done
done
python paper_2602_06071_b200/build.py --instrument > /dev/null
for c in sweepT_k16_s4_bf16 sweepT_k8_s8_bf16 sweepT_k16_s8_bf16; do
 for f in 0 32 1; do
  BPS_LIB=$PWD/paper_2602_06071_b200/libbps_instr.so BPS_TC_DEBUG=$f timeout 300 python bench.py --config $c $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('instr $c dbg=$f', round(d['value'],1), 'GB/s', round(d['ms_per_step'],3), 'ms')"
 done
 for cs in 2 4; do
  BPS_TC_CLUSTER=$cs timeout 300 python bench.py --config $c $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prod $c cs=$cs', round(d['value'],1), 'GB/s', round(d['ms_per_step'],3), 'ms')"
 done
done
