#!/bin/bash
# timing experiments with parts of the tc kernel disabled (instrumented build; results are wrong by design)
python paper_2602_06071_b200/build.py --instrument > /dev/null
export BPS_LIB=$PWD/paper_2602_06071_b200/libbps_instr.so
for c in ${CONFIGS:-ls grad}; do
for f in ${FLAGS:-0 1 2 3 4 5 7}; do
  BPS_TC_DEBUG=$f timeout 300 python bench.py ${BENCH_EXTRA} --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c dbg=$f', round(d['value'],1), 'GB/s', round(d['ms_per_step'],3), 'ms')"
done; done
