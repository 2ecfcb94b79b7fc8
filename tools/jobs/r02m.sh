O=gpurun_out/r02m; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mcm_batch_warp -c 1 -f -o /tmp/ncu_mb python bench.py --workload c5a --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu -i /tmp/ncu_mb.ncu-rep --page details --csv > $O/ncu_mb.details.csv 2>/dev/null
ncu -i /tmp/ncu_mb.ncu-rep --page source --csv --print-source=sass > /tmp/src_mb.csv 2>/dev/null
python tools/ncu_hot.py /tmp/src_mb.csv 40 > $O/ncu_hot_mb.txt 2>&1; head -45 $O/ncu_hot_mb.txt
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r02m/ncu_mb.details.csv')))
h=rows[0]; ni=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
for r in rows[1:]:
    if r[ni] in ('Duration','Executed Instructions','Issue Slots Busy','Achieved Occupancy','Theoretical Occupancy','Block Limit Shared Mem','L1/TEX Cache Throughput','DRAM Throughput','Shared Memory Configuration Size'):
        print(f"  {r[ni]:40s} {r[vi]:>16s} {r[ui]}")
PY
