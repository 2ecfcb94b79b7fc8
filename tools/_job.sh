timeout 900 python -m pytest tests/test_gpu_mcm.py tests/test_gpu_batch.py tests/test_dropin.py -x -q 2>&1 | tail -2
timeout 200 python bench.py --workload c5a --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5a', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],2))"
