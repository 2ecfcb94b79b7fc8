mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_mcm.py -x -q > gpurun_out/pytest_m.txt 2>&1; tail -1 gpurun_out/pytest_m.txt; grep -E "^E |FAILED" gpurun_out/pytest_m.txt | head -5
export PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so
timeout 60 python tools/mcm_profile.py 1024 | head -6
PIPEDP_MCM_T32_MAXN=0 timeout 60 python tools/mcm_profile.py 1024 | head -6
unset PIPEDP_LIB
for w in c3 c4; do timeout 200 python bench.py --workload $w --no-cpu-baseline --steps 3 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', d['roofline']['kernel'], round(d['ms_per_step'],3), '%.3e'%d['value'], d['parity'])"; done
PIPEDP_MCM_T32_MAXN=0 timeout 200 python bench.py --workload c3 --no-cpu-baseline --steps 3 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 t64', d['roofline']['kernel'], round(d['ms_per_step'],3), d['parity'])"
PIPEDP_MCM_T32_MAXN=100000 timeout 200 python bench.py --workload c4 --no-cpu-baseline --steps 3 --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 t32', d['roofline']['kernel'], round(d['ms_per_step'],3), d['parity'])"
