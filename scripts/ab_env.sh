#!/bin/bash
# bench one config under several env settings: ENVS="name:VAR=x,VAR2=y name2:..."
O=gpurun_out; T=${TAG:-abe}; C=${CFG:-ls}
for spec in $ENVS; do
  nm=${spec%%:*}; ev=${spec#*:}; ev=${ev//,/ }
  env $ev timeout 300 python bench.py --config $C --no-cpu-baseline --no-e2e --no-clocks $BARGS > $O/${T}_${C}_$nm.json 2>$O/${T}_${C}_$nm.err
  echo "$C $nm: $(python -c "import json;d=json.load(open('$O/${T}_${C}_$nm.json'));print(round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'min', round(d['ms_min'],4))" 2>&1|tail -1)"
done
