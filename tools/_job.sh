timeout 30 ./tools/npt
timeout 300 python -m pytest tests/test_gpu_mcm.py -x -q 2>&1 | tail -2
for w in c3 c4; do timeout 100 python bench.py --workload $w --no-cpu-baseline --e2e-steps 0 --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],3), d['parity']['match'])"; done
export PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so
timeout 120 python tools/mcm_profile.py 1024 2>&1 | tail -7 | head -6
timeout 120 python tools/mcm_profile.py 8192 2>&1 | tail -7 | head -6
