#!/bin/bash
# Round measurement: smoke, full GPU suite, bench lines, ncu launch lists and full captures.
# usage (on the GPU box): TAG=r01_v12 bash scripts/round_measure.sh ; outputs in gpurun_out/
TAG=${TAG:-rXX}
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/${TAG}_pytest_gpu.log
fi
bench() { # name, args...
  local nm=$1; shift
  timeout 900 python bench.py "$@" > $O/${TAG}_bench_${nm}.json 2> $O/${TAG}_bench_${nm}.err
  echo "bench $nm rc=$? $(python -c "import json;d=json.load(open('$O/${TAG}_bench_${nm}.json'));print(round(d['value'],1), d['unit'], round(d['roofline']['frac'],3))" 2>/dev/null)"
}
bench ls
bench grad --config grad
bench smalln --config smalln
bench ls_transposed --config ls --layout t
bench grad_transposed --config grad --layout t
bench scaleout --config scaleout --steps 3 --warmup 3 --no-cpu-baseline
bench ls_affine --config ls --mode affine
bench grad_affine --config grad --mode affine
bench adjoint_ls --config ls --op adjoint
bench blockrow_ls --config ls --sketch blockrow
python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_reference.json 2>&1
if [ -n "$NCU" ]; then
  for c in ls grad; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/${TAG}_launches_${c}.csv \
       python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1
    echo "ncu launches $c rc=$?"
  done
  for spec in "ls|--config ls" "grad|--config grad" "gradt|--config grad --layout t" "lst|--config ls --layout t"; do
    nm=${spec%%|*}; a=${spec#*|}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:bps_tc_kernel -s 3 -c 1 -o $O/${TAG}_prof_${nm} -f \
       python bench.py $a --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > $O/${TAG}_ncu_${nm}.log 2>&1
    echo "ncu full $nm rc=$?"
    python scripts/ncu_summary.py $O/${TAG}_prof_${nm}.ncu-rep $O/${TAG}_ncu_${nm}.txt > /dev/null 2>&1
    ncu -i $O/${TAG}_prof_${nm}.ncu-rep --page raw --csv > $O/${TAG}_ncu_${nm}_raw.csv 2>/dev/null
    [ -n "$KEEP_REP" ] || rm -f $O/${TAG}_prof_${nm}.ncu-rep   # gpurun copies back at most 64 MiB
  done
fi
