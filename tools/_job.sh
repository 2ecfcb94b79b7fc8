mkdir -p gpurun_out/r01b
timeout 300 python -m pytest tests/test_gpu_mcm.py tests/test_gpu_batch.py tests/test_dropin.py -x -q > gpurun_out/r01b/pytest_mcm.txt 2>&1; tail -1 gpurun_out/r01b/pytest_mcm.txt
timeout 600 python bench.py --workload c5a > gpurun_out/r01b/bench_c5a.json 2> gpurun_out/r01b/bench_c5a.err; python -c "
import json; d=json.loads(open('gpurun_out/r01b/bench_c5a.json').read().strip().splitlines()[-1]); print('c5a', d['roofline']['kernel'], round(d['ms_per_step'],3), '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], 'cpu', d['cpu_baseline'] and '%.3e'%d['cpu_baseline']['value'])"
