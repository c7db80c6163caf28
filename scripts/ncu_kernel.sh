#!/bin/bash
# ncu --set full of one kernel (regex K) in a bench run; summary to gpurun_out
O=gpurun_out; T=${TAG:-nk}; C=${CFG:-ls}; K=${KREGEX:-bps_tc_kernel}
timeout 600 ncu --set full --clock-control none ${NCUX} --import-source on -k regex:$K -s ${SKIP:-3} -c 1 -o $O/${T}_${C} -f \
   env $LENV python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks $BARGS > $O/${T}_${C}.log 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py $O/${T}_${C}.ncu-rep $O/${T}_${C}.txt > /dev/null 2>&1; head -45 $O/${T}_${C}.txt
ncu -i $O/${T}_${C}.ncu-rep --page details --csv > $O/${T}_${C}_details.csv 2>/dev/null
[ -n "$KEEP_REP" ] || rm -f $O/${T}_${C}.ncu-rep
