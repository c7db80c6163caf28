#!/bin/bash
# narrow-n scaling: the smalln and LS sketches at several column counts
mkdir -p gpurun_out
for spec in "smalln 32" "smalln 64" "smalln 128" "smalln 256" "ls 64" "ls 128" "ls 256"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --n $2 --no-cpu-baseline --no-e2e --no-clocks > gpurun_out/nar_$1_$2.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/nar_$1_$2.json'));r=d['roofline'];print('$1 n=$2', round(d['value']), 'GB/s', round(d['value']/r['peak'],3), 'ms', round(d['ms_per_step'],4), 'kern', round(r['kernel_ms_mean'],4))"
done
