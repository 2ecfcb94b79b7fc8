O=gpurun_out/r02n; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sdp.py tests/test_dropin.py -m gpu -q -x > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; python -c "
import json; d=json.loads(open('$O/bench_c2.json').read().strip().splitlines()[-1]); print('c2', d['ms_per_step'], 'e2e', d['e2e'], d['parity'])"
