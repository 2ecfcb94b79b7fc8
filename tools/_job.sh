timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 200 python bench.py --workload c2 --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', round(d['ms_per_step'],2), d['e2e']['ms_per_step'], d['parity']['match'])"
