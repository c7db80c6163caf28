#!/bin/bash
# ncu launch list (kernel durations, cold cache, serialised) of a few bench steps
O=gpurun_out; T=${TAG:-ll}; C=${CFG:-ls}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none ${NCUX:--k regex:bps} -c ${NK:-40} --csv --log-file $O/${T}_launches_${C}.csv \
   env $LENV python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks $BARGS > /dev/null 2>&1
echo "ncu rc=$?"
python - "$O/${T}_launches_${C}.csv" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; iK = h.index("Kernel Name"); iM = h.index("Metric Name"); iV = h.index("Metric Value"); iID = h.index("ID")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    agg[r[iK][:60]][r[iM]].append(float(r[iV].replace(",", "")))
for k, m in agg.items():
    t = m.get("gpu__time_duration.sum", [0]); rd = m.get("dram__bytes_read.sum", [0]); wr = m.get("dram__bytes_write.sum", [0])
    print(f"{k:60s} n={len(t):3d} mean_us={sum(t)/len(t)/1e3:9.2f} read_MB={sum(rd)/len(rd)/1e6:9.1f} write_MB={sum(wr)/len(wr)/1e6:8.1f}")
PY
