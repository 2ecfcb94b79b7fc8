timeout 600 python -m pytest tests/test_gpu_mcm.py -x -q > gpurun_out/pytest_mcm.txt 2>&1; tail -30 gpurun_out/pytest_mcm.txt
for w in c3 c4; do timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 0 --steps 3 > gpurun_out/bench_$w.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_$w.json').read().strip().splitlines()[-1]); print('$w', d['roofline']['kernel'], d['ms_per_step'], '%.3e'%d['value'], d['parity'])" || tail -5 gpurun_out/bench_$w.json; done
