#!/bin/bash
# Quick GPU iteration: smoke, selected tests, a few bench lines.  usage: TAG=x TESTS="..." BENCH="ls grad" bash scripts/gpu_quick.sh
TAG=${TAG:-q}
O=gpurun_out
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/${TAG}_smoke.log
if [ -n "$TESTS" ]; then
  timeout ${TTIME:-1500} python -m pytest $TESTS -m gpu -q ${KEXPR:+-k "$KEXPR"} > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/${TAG}_pytest.log
fi
for c in $BENCH; do
  timeout 600 python bench.py --config $c --no-cpu-baseline ${BARGS} > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err
  echo "bench $c rc=$? $(python -c "import json;d=json.load(open('$O/${TAG}_bench_$c.json'));print(round(d['value'],1), d['unit'], 'frac', round(d['roofline']['frac'],3), 'ms', round(d['ms_per_step'],4), d['clocks'])" 2>&1 | tail -1)"
done
