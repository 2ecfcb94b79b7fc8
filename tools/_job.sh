timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for w in c2 c3 c4 c5a c5b; do timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), (d['parity'] or {}).get('match'))"; done
