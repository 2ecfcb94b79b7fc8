O=gpurun_out/r02f; mkdir -p $O
for m in 1 0; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sdp_batch_dom -s 2 -c 1 -f -o /tmp/ncu_m$m python tools/batch_modes.py $m > /dev/null 2>&1
ncu -i /tmp/ncu_m$m.ncu-rep --page details --csv > $O/ncu_m$m.details.csv 2>/dev/null
ncu -i /tmp/ncu_m$m.ncu-rep --page source --csv --print-source=sass > /tmp/src_m$m.csv 2>/dev/null
python tools/ncu_hot.py /tmp/src_m$m.csv 40 > $O/ncu_hot_m$m.txt 2>&1
done
