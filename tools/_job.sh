timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_sdp.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --workload c5b --no-cpu-baseline --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5b', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), d.get('parity'))"
