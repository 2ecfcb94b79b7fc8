# Round evidence run on one B200 (gpurun): GPU tests, every bench line, the
# reference arm, the ncu launch list and one `ncu --set full` capture per
# workload's hot kernel (CSV exports only; the .ncu-rep stays in /tmp).
# usage: bash tools/evidence.sh r01c
R=${1:-r01c}
O=gpurun_out/$R
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 300 $O/bench_c2.json
for w in c1 c3 c4 c5a c5b; do
  timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; tail -c 200 $O/bench_$w.json; echo
done
timeout 600 python bench.py --impl reference > $O/bench_ref_c2.json 2>&1; tail -c 200 $O/bench_ref_c2.json; echo
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
declare -A K=([c1]='regex:sdp_jump' [c2]='regex:sdp_pipeline_cta' [c3]='regex:mcm_tiled' [c4]='regex:mcm_tiled'
             [c5a]='regex:mcm_smem' [c5b]='regex:sdp_batch')
for w in c1 c2 c3 c4 c5a c5b; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "${K[$w]}" -c 1 -f -o /tmp/ncu_$w \
    python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  ncu -i /tmp/ncu_$w.ncu-rep --page raw --csv > $O/ncu_full_$w.raw.csv 2>/dev/null
  ncu -i /tmp/ncu_$w.ncu-rep --page details --csv > $O/ncu_full_$w.details.csv 2>/dev/null
  ncu -i /tmp/ncu_$w.ncu-rep --page source --csv --print-source=sass > /tmp/src_$w.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/src_$w.csv 40 > $O/ncu_hot_$w.txt 2>&1
  head -3 $O/ncu_hot_$w.txt
done
