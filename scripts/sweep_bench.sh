#!/bin/bash
# κ×s sweep through bench.py (same timing path as the driver's bench), one JSON line per config.
# SWEEP=sweepT (tuned B_r) or sweep (B_r=32), VARIANT=auto|tc|sparse.  Output: gpurun_out/${SWEEP}_${VARIANT}_bench.jsonl
mkdir -p gpurun_out
pre=${SWEEP:-sweepT}
v=${VARIANT:-auto}
out=gpurun_out/${pre}_${v}_bench.jsonl
: > $out
for dt in ${DTYPES:-bf16 f32}; do
 for k in 1 2 4 8 16; do
  for s in 1 2 4 8; do
   c=${pre}_k${k}_s${s}_${dt}
   timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --variant $v --no-e2e --no-cpu-baseline 2>/dev/null \
     | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['config']
print(json.dumps({'dtype':'$dt','kappa':$k,'s':$s,'B_r':c['B_r'],'variant':'$v','config':'$c','gbs':d['value'],'frac':d['roofline']['frac'],'ms':d['ms_per_step'],'sm_mhz':d['clocks'].get('sm_mhz'),'reasons':d['clocks'].get('reasons')}))" >> $out \
     || echo "{\"dtype\":\"$dt\",\"kappa\":$k,\"s\":$s,\"variant\":\"$v\",\"config\":\"$c\",\"unsupported\":\"failed\"}" >> $out
  done
 done
done
wc -l $out
