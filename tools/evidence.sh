# Round evidence run on one B200 (gpurun): GPU tests, smoke, every bench line,
# the reference arm, the ncu launch list of the default bench, one
# `ncu --set full` capture per workload's dominant kernel (CSV exports only),
# Table I, the two-rank bench on the one GPU.  usage: bash tools/evidence.sh r02x
R=${1:-r02x}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=20 > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 300 $O/bench_c2.json; echo
for w in c1 c3 c4 c5a c5b; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; tail -c 200 $O/bench_$w.json; echo
done
timeout 600 python bench.py --workload c3 --mcm-kernel tournament --steps 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_c3_tournament.json 2>&1
PIPEDP_SDP_CHUNKED=0 timeout 900 python bench.py --steps 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_c2_pipeline_only.json 2>&1
timeout 900 python bench.py --impl reference > $O/bench_ref_c2.json 2>&1; tail -c 200 $O/bench_ref_c2.json; echo
timeout 900 python bench.py --gpus 2 --steps 3 > $O/bench_n2.json 2> $O/bench_n2.err; tail -c 300 $O/bench_n2.json; echo
timeout 900 python tools/table1.py --out $O/table1.csv > $O/table1.txt 2>&1; tail -6 $O/table1.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c2.csv 3 > $O/launches_c2_summary.txt 2>&1; head -8 $O/launches_c2_summary.txt
declare -A K=([c1]='regex:sdp_jump' [c2]='regex:chunk_rank' [c3]='regex:mcm_tiled' [c4]='regex:mcm_tiled'
             [c5a]='regex:mcm_batch_warp' [c5b]='regex:sdp_batch_dom')
for w in c1 c2 c3 c4 c5a c5b; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "${K[$w]}" -c 1 -f -o /tmp/ncu_$w \
    python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  ncu -i /tmp/ncu_$w.ncu-rep --page raw --csv > $O/ncu_full_$w.raw.csv 2>/dev/null
  ncu -i /tmp/ncu_$w.ncu-rep --page details --csv > $O/ncu_full_$w.details.csv 2>/dev/null
  ncu -i /tmp/ncu_$w.ncu-rep --page source --csv --print-source=sass > /tmp/src_$w.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/src_$w.csv 40 > $O/ncu_hot_$w.txt 2>&1
  head -3 $O/ncu_hot_$w.txt
done
# the cluster pipeline (one instance, C2 shape at 2^18 cells)
PIPEDP_SDP_CHUNKED=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sdp_cluster -c 1 -f -o /tmp/ncu_cl \
  python tools/cluster_probe.py 18 > /dev/null 2>&1
ncu -i /tmp/ncu_cl.ncu-rep --page details --csv > $O/ncu_full_cluster.details.csv 2>/dev/null
ncu -i /tmp/ncu_cl.ncu-rep --page source --csv --print-source=sass > /tmp/src_cl.csv 2>/dev/null
python tools/ncu_hot.py /tmp/src_cl.csv 40 > $O/ncu_hot_cluster.txt 2>&1
