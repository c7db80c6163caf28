#!/bin/bash
# A/B of the canonical decomposition on LS / grad (round 2 regression hunt)
O=gpurun_out; T=${TAG:-ab}
b() { local nm=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-clocks $BARGS > $O/${T}_$nm.json 2>$O/${T}_$nm.err; echo "$nm: $(python -c "import json;d=json.load(open('$O/${T}_$nm.json'));print(round(d['value'],1), 'ms', round(d['ms_per_step'],4))" 2>&1|tail -1)"; }
for c in ${CFGS:-ls grad}; do
  BARGS="--config $c" b ${c}_new X=1
  BARGS="--config $c --no-workspace" b ${c}_halo X=1
  BARGS="--config $c" b ${c}_nocoop BPS_TC_NOCOOP=1
  BARGS="--config $c" b ${c}_g128 BPS_TC_GROUP=128
  BARGS="--config $c" b ${c}_old BPS_LIB=$PWD/ab_old/libbps_old.so
done
timeout 300 python scripts/tc_trace.py ${CFGS:-ls grad} > $O/${T}_trace.txt 2>&1; echo trace rc=$?; cat $O/${T}_trace.txt | head -40; BPS_LIB=$PWD/ab_old/libbps_old_instr.so timeout 300 python scripts/tc_trace.py ${CFGS:-ls grad} > $O/${T}_trace_old.txt 2>&1; head -16 $O/${T}_trace_old.txt
