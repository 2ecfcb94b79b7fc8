timeout 600 python -m pytest tests/test_gpu_sdp.py tests/test_gpu_batch.py tests/test_dropin.py -x -q 2>&1 | tail -3
PYTHONPATH=. timeout 200 python tools/e2e_probe.py
timeout 200 python bench.py --workload c2 --no-cpu-baseline --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', round(d['ms_per_step'],1), d['e2e']['ms_per_step'], d['parity']['match'])"
