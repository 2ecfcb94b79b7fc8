O=gpurun_out/r02o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_mcm.py -m gpu -q -x > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
for w in c3 c4; do timeout 600 python bench.py --workload $w --no-cpu-baseline --e2e-steps 0 > $O/b_$w.json 2>&1; python -c "
import json; d=json.loads(open('$O/b_$w.json').read().strip().splitlines()[-1]); print('$w', d['ms_per_step'], d['parity'])"; done
