timeout 900 python -m pytest tests/test_gpu_sdp.py -x -q -k "chunked" 2>&1 | tail -2
timeout 200 python bench.py --workload c2 --no-cpu-baseline --e2e-steps 0 --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', round(d['ms_per_step'],3), d['parity']['match'])"
