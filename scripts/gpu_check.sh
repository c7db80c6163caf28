#!/bin/bash
# One gpurun session: build, smoke, gpu tests, bench, launch list, ncu capture. Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?"
  tail -25 gpurun_out/pytest_gpu.log
fi
for v in ${BENCH_VARIANTS:-auto}; do
  for c in ${BENCH_CONFIGS:-ls}; do
    timeout 900 python bench.py --config $c --variant $v ${BENCH_ARGS} > gpurun_out/bench_${c}_${v}.json 2> gpurun_out/bench_${c}_${v}.err
    echo "bench $c $v rc=$?"; head -c 2500 gpurun_out/bench_${c}_${v}.json; echo
  done
done
if [ -n "$NCU" ]; then
  for c in ${NCU_CONFIGS:-ls}; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_${c}.csv \
       python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1
    echo "ncu launches $c rc=$?"
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:bps_tc_kernel -s 3 -c 1 -o gpurun_out/prof_${c} -f \
       python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_full_${c}.log 2>&1
    echo "ncu full $c rc=$?"
  done
fi
