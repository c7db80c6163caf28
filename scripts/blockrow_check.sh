#!/bin/bash
# gpurun session for FlashBlockRow: tests, bench lines, ncu launch list + full capture.
mkdir -p gpurun_out
python paper_2602_06071_b200/build.py > gpurun_out/br_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_blockrow.py -q -x > gpurun_out/br_pytest.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/br_pytest.log
for c in ${BR_CONFIGS:-ls grad smalln}; do
  timeout 600 python bench.py --sketch blockrow --config $c --steps 20 --warmup 5 > gpurun_out/br_bench_$c.json 2> gpurun_out/br_bench_$c.err
  echo "bench $c rc=$?"; python -c "import json;d=json.load(open('gpurun_out/br_bench_$c.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/br_launches_ls.csv \
     python bench.py --sketch blockrow --config ls --steps 3 --warmup 3 --no-clocks > /dev/null 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:blockrow -s 3 -c 1 -o gpurun_out/br_prof_ls -f \
     python bench.py --sketch blockrow --config ls --steps 2 --warmup 3 --no-clocks > gpurun_out/br_ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
