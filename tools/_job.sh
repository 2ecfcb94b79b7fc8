timeout 400 python -m pytest tests/test_gpu_sdp.py tests/test_gpu_batch.py -x -q 2>&1 | tail -2
b() { timeout 100 python bench.py --workload c2 --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step'],1), d['parity']['match'])"; }
b base
PIPEDP_SDP2_AREM=1024 b arem1024
PIPEDP_SDP_REMOTE_WARPS=24 b rw24
export PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so
timeout 120 python tools/v2_profile.py 24 1024 4096 2>&1 | tail -16
