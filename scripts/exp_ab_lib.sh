#!/bin/bash
# A/B: production libbps.so vs a variant library (VAR=libname) on several configs; then a quick parity subset
L=$GRAFT_REPO_ROOT/paper_2602_06071_b200
mkdir -p gpurun_out
for c in ${CFGS:-smalln ls grad}; do
  CFG=$c TAG=${TAG:-ab} ENVS="new:X=1 old:BPS_LIB=$L/${VAR:-libbps_wa0.so}" BARGS="$BARGS" bash scripts/ab_env.sh
done
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -m gpu -q -x ${KEXPR:+-k "$KEXPR"} > gpurun_out/${TAG:-ab}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG:-ab}_pytest.log; fi
