#!/bin/bash
# A/B knobs of the canonical tc path (BPS_TC_AB bits, see TcArgs::ab)
O=gpurun_out; T=${TAG:-abk}
b() { local nm=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-clocks $BARGS > $O/${T}_$nm.json 2>$O/${T}_$nm.err; echo "$nm: $(python -c "import json;d=json.load(open('$O/${T}_$nm.json'));print(round(d['value'],1), 'ms', round(d['ms_per_step'],4))" 2>&1|tail -1)"; }
for c in ${CFGS:-ls}; do
  for k in ${KNOBS:-0 4 8 12}; do BARGS="--config $c" b ${c}_ab$k BPS_TC_AB=$k; done
  BARGS="--config $c" b ${c}_old BPS_LIB=$PWD/ab_old/libbps_old.so
done
