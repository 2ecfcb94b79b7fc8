PYTHONPATH=. PIPEDP_TRACE_D2H=1 timeout 200 python tools/e2e_probe.py 2>&1 | tail -14
timeout 200 python bench.py --workload c2 --no-cpu-baseline --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', round(d['ms_per_step'],1), d['e2e']['ms_per_step'], d['parity']['match'])"
