#!/bin/bash
# ncu --set full of the tc kernel on one config, new library vs an old one (A/B)
O=gpurun_out; T=${TAG:-ncuab}; C=${CFG:-ls}
for v in new old; do
  L="X=1 $NEWENV"; [ $v = old ] && L="BPS_LIB=$PWD/ab_old/libbps_old.so"
  env $L timeout 600 ncu --set full --clock-control none --import-source on -k regex:bps_tc_kernel -s 3 -c 1 -o $O/${T}_${C}_$v -f \
     python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > $O/${T}_${C}_$v.log 2>&1
  echo "ncu $v rc=$?"
  python scripts/ncu_summary.py $O/${T}_${C}_$v.ncu-rep $O/${T}_${C}_$v.txt > /dev/null 2>&1
  head -20 $O/${T}_${C}_$v.txt
  [ -n "$KEEP_REP" ] || rm -f $O/${T}_${C}_$v.ncu-rep
done
