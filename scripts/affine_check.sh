#!/bin/bash
# gpurun session for the AffineUnique mode: parity tests (both modes), bench lines.
mkdir -p gpurun_out
python paper_2602_06071_b200/build.py > gpurun_out/af_build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests/test_gpu_affine.py tests/test_gpu_parity.py tests/test_gpu_adjoint.py -q -x > gpurun_out/af_pytest.log 2>&1
echo "pytest rc=$?"; tail -6 gpurun_out/af_pytest.log
for m in rowpart affine; do
for c in ls grad; do
  timeout 600 python bench.py --mode $m --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/af_bench_${c}_$m.json 2> gpurun_out/af_bench_${c}_$m.err
  echo "bench $c $m rc=$?"; python -c "import json;d=json.load(open('gpurun_out/af_bench_${c}_$m.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'],d['clocks'])"
done
timeout 600 python bench.py --op adjoint --mode $m --config ls --steps 10 --warmup 3 > gpurun_out/af_bench_adj_ls_$m.json 2> gpurun_out/af_bench_adj_ls_$m.err
echo "bench adjoint ls $m rc=$?"; python -c "import json;d=json.load(open('gpurun_out/af_bench_adj_ls_$m.json'));print(d['value'],d['roofline']['frac'],d['ms_per_step'])"
done
