#!/bin/bash
# selected sweep points: PTS="k8_s1 k16_s4 ..." DT="bf16 f32" PRE=sweep ENVV="X=1"
O=gpurun_out; T=${TAG:-swp}
for dt in ${DT:-bf16 f32}; do for pt in $PTS; do
  c=${PRE:-sweep}_${pt}_${dt}
  env ${ENVV:-X=1} timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-clocks > $O/${T}_$c.json 2>$O/${T}_$c.err
  echo "$c: $(python -c "import json;d=json.load(open('$O/${T}_$c.json'));r=d['roofline'];print(round(d['value']), round(d['ms_per_step'],4), 'frac', round(d['value']/r['peak'],3), 'kern', round(r['kernel_ms_mean'] or 0,4))" 2>&1 | tail -1)"
done; done
