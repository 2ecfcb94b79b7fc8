for w in c1 c3 c4 c5a c2; do python bench.py --workload $w --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); cb=d.get('cpu_baseline') or {}; print('$w', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), 'cpu', cb.get('value'))"; done
