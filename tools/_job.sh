./tools/near_bench
export PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so
python tools/v2_profile.py 22
unset PIPEDP_LIB
timeout 600 python -m pytest tests/test_gpu_sdp.py -x -q > gpurun_out/pytest_sm.txt 2>&1; tail -3 gpurun_out/pytest_sm.txt
for nc in 4 6; do for ng in 1 2 3; do PIPEDP_SDP2_COMB=$nc PIPEDP_SDP2_NEAR_GROUP=$ng timeout 300 python bench.py --workload c2 --no-cpu-baseline --e2e-steps 0 --steps 2 --warmup 1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nc $nc ng $ng', d['ms_per_step'], d['parity']['match'])"; done; done
