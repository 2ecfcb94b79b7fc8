timeout 30 ./tools/npt
PIPEDP_MCM_NEAR=2 timeout 40 python -m pytest tests/test_gpu_mcm.py -x -q -k "test_tiled_shapes and 33-100000" 2>&1 | tail -2
PIPEDP_MCM_NEAR=2 timeout 300 python -m pytest tests/test_gpu_mcm.py -x -q 2>&1 | tail -2
for m in 0 2; do for w in c3 c4; do PIPEDP_MCM_NEAR=$m timeout 100 python bench.py --workload $w --no-cpu-baseline --e2e-steps 0 --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('near $m $w', round(d['ms_per_step'],3), d['parity']['match'])"; done; done
