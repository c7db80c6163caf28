#!/bin/bash
# Round measurement: smoke, full GPU suite, bench lines, ncu launch lists and full captures,
# compute-sanitizer.  usage (on the GPU box): TAG=r02_v1 bash scripts/round_measure.sh ; outputs in gpurun_out/
TAG=${TAG:-rXX}
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
if [ -z "$NO_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/${TAG}_pytest_gpu.log
fi
bench() { # name, args...
  local nm=$1; shift
  timeout 900 python bench.py "$@" > $O/${TAG}_bench_${nm}.json 2> $O/${TAG}_bench_${nm}.err
  echo "bench $nm rc=$? $(python -c "import json;d=json.load(open('$O/${TAG}_bench_${nm}.json'));r=d['roofline'];print(round(d['value'],1), d['unit'], 'step_frac', round(d['value']/r['peak'],3), 'kernel_frac', round(r['frac'],3))" 2>/dev/null)"
}
if [ -z "$NO_BENCH" ]; then
bench ls
bench ls_coherent --kind coherent --no-cpu-baseline
bench ls_lowrank --kind lowrank --no-cpu-baseline
bench grad --config grad
bench grad_coherent --config grad --kind coherent --no-e2e
bench grad_lowrank --config grad --kind lowrank --no-e2e
bench smalln --config smalln
bench ls_transposed --config ls --layout t
bench grad_transposed --config grad --layout t
bench scaleout --config scaleout --steps 3 --warmup 3 --no-cpu-baseline
bench ls_affine --config ls --mode affine
bench grad_affine --config grad --mode affine
bench adjoint_ls --config ls --op adjoint
bench blockrow_ls --config ls --sketch blockrow
python bench.py --impl reference > $O/${TAG}_bench_reference.json 2>&1
fi
if [ -n "$NCU" ]; then
  for c in ls grad smalln; do
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bps -c 20 --csv \
       --log-file $O/${TAG}_launches_${c}.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1
    echo "ncu launches $c rc=$?"
  done
  for spec in "ls|--config ls|bps_tc_kernel" "grad|--config grad|bps_tc_kernel" "smalln|--config smalln|bps_tc_kernel" \
              "gradt|--config grad --layout t|bps_tc_kernel" "lst|--config ls --layout t|bps_tc_kernel" \
              "lscombine|--config ls|bps_tc_combine"; do
    IFS='|' read nm a k <<< "$spec"
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/${TAG}_prof_${nm} -f \
       python bench.py $a --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > $O/${TAG}_ncu_${nm}.log 2>&1
    echo "ncu full $nm rc=$?"
    python scripts/ncu_summary.py $O/${TAG}_prof_${nm}.ncu-rep $O/${TAG}_ncu_${nm}.txt > /dev/null 2>&1
    ncu -i $O/${TAG}_prof_${nm}.ncu-rep --page raw --csv > $O/${TAG}_ncu_${nm}_raw.csv 2>/dev/null
    [ -n "$KEEP_REP" ] || rm -f $O/${TAG}_prof_${nm}.ncu-rep   # gpurun copies back at most 64 MiB
  done
fi
if [ -n "$SANITIZE" ]; then
  TAG=$TAG bash scripts/sanitize.sh
fi
