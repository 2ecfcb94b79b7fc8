O=gpurun_out/r02c; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_sdp.py -m gpu -q -x -k "chunk or config2 or streamed" > $O/pytest_sdp.txt 2>&1; tail -5 $O/pytest_sdp.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; python -c "
import json; d=json.loads(open('$O/bench_c2.json').read().strip().splitlines()[-1]); print('c2 ms', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], d['parity'], d['roofline']['kernel'])"
PIPEDP_SDP_RANK=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_c2_norank.json 2>&1; python -c "
import json; d=json.loads(open('$O/bench_c2_norank.json').read().strip().splitlines()[-1]); print('c2 norank ms', d['ms_per_step'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c2.csv 3 2>&1 | head -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chunk_rank -c 1 -f -o /tmp/ncu_rank python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu -i /tmp/ncu_rank.ncu-rep --page raw --csv > $O/ncu_rank.raw.csv 2>/dev/null
ncu -i /tmp/ncu_rank.ncu-rep --page details --csv > $O/ncu_rank.details.csv 2>/dev/null
ncu -i /tmp/ncu_rank.ncu-rep --page source --csv --print-source=sass > /tmp/src_rank.csv 2>/dev/null
python tools/ncu_hot.py /tmp/src_rank.csv 40 > $O/ncu_hot_rank.txt 2>&1; head -30 $O/ncu_hot_rank.txt
