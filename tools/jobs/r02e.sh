O=gpurun_out/r02e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_batch.py -m gpu -q -x > $O/pytest_batch.txt 2>&1; tail -5 $O/pytest_batch.txt
timeout 300 python tools/batch_modes.py > $O/modes.txt 2>&1; cat $O/modes.txt
timeout 300 python bench.py --workload c5b --no-cpu-baseline > $O/bench_c5b.json 2> $O/bench_c5b.err; python -c "
import json; d=json.loads(open('$O/bench_c5b.json').read().strip().splitlines()[-1]); print('c5b ms', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], d['parity'], d['roofline'])"
