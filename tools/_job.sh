timeout 400 python -m pytest tests/test_gpu_sdp.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c1', d['ms_per_step'], d['value'], d['e2e']['value'], d['cpu_baseline']['value'], d['parity'], d['roofline']['kernel'], d.get('chain_roofline'))"
