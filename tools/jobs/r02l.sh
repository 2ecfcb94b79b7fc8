O=gpurun_out/r02l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_mcm.py -m gpu -q -x > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
timeout 300 python bench.py --workload c5a --no-cpu-baseline > $O/bench_c5a.json 2> $O/bench_c5a.err; python -c "
import json; d=json.loads(open('$O/bench_c5a.json').read().strip().splitlines()[-1]); print('c5a ms', d['ms_per_step'], d['parity'], d['roofline']['kernel'], d['roofline']['frac'])"
