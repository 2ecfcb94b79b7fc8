PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so python tools/mcm_profile.py 8192 > gpurun_out/p8192.txt 2>&1; head -6 gpurun_out/p8192.txt
PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so python tools/mcm_profile.py 1024 > gpurun_out/p1024.txt 2>&1; head -1 gpurun_out/p1024.txt
for w in c3 c4; do python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/$w.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/$w.json').read().strip().splitlines()[-1]); print('$w', d['ms_per_step'], d['parity'])"; done
python -m pytest tests/test_gpu_mcm.py -m gpu -x -q 2>&1 | tail -2
