#!/bin/bash
# One gpurun session: build, smoke, gpu tests, bench, launch list. Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for v in ${BENCH_VARIANTS:-auto}; do
  for c in ${BENCH_CONFIGS:-ls}; do
    timeout 600 python bench.py --config $c --variant $v ${BENCH_ARGS} > gpurun_out/bench_${c}_${v}.json 2> gpurun_out/bench_${c}_${v}.err
    echo "bench $c $v rc=$?"; cat gpurun_out/bench_${c}_${v}.json | head -c 1500; echo
  done
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
     python bench.py --config ls --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1
  echo "ncu rc=$?"
fi
