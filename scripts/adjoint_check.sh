#!/bin/bash
# gpurun session for the adjoint X = Sᵀ·Y: tests, bench lines, ncu (launch list + full capture).
mkdir -p gpurun_out
python paper_2602_06071_b200/build.py > gpurun_out/adj_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_adjoint.py -q -x > gpurun_out/adj_pytest.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/adj_pytest.log
for v in ${ADJ_VARIANTS:-tc sparse}; do
for c in ${ADJ_CONFIGS:-ls smalln sweep_k4_s4_bf16}; do
  timeout 600 python bench.py --op adjoint --variant $v --config $c --steps 10 --warmup 3 > gpurun_out/adj_bench_${c}_$v.json 2> gpurun_out/adj_bench_${c}_$v.err
  echo "bench $c $v rc=$?"; python -c "import json;d=json.load(open('gpurun_out/adj_bench_${c}_$v.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
done
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/adj_launches_ls.csv \
     python bench.py --op adjoint --config ls --steps 3 --warmup 3 --no-clocks > /dev/null 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:adjoint -s 3 -c 1 -o gpurun_out/adj_prof_ls -f \
     python bench.py --op adjoint --config ls --steps 2 --warmup 3 --no-clocks > gpurun_out/adj_ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
