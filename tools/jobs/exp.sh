O=gpurun_out/exp; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bm_chain -c 1 -f -o /tmp/ncu_ch python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu -i /tmp/ncu_ch.ncu-rep --page source --csv --print-source=sass > /tmp/src_ch.csv 2>/dev/null
python tools/ncu_hot.py /tmp/src_ch.csv 25 > $O/ncu_hot_chain.txt 2>&1; head -30 $O/ncu_hot_chain.txt
ncu -i /tmp/ncu_ch.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|"Executed Instructions"|"Issue Slots Busy"' 
