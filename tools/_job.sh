timeout 900 python -m pytest tests/test_gpu_mcm.py -x -q 2>&1 | tail -2
for w in c3 c4; do timeout 200 python bench.py --workload $w --no-cpu-baseline --e2e-steps 0 --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],3), d['parity']['match'])"; done
