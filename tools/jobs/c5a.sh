python -m pytest tests/test_gpu_mcm.py -m gpu -x -q -k "batch" 2>&1 | tail -2
python bench.py --workload c5a --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c5a.json 2> gpurun_out/c5a.err; python -c "
import json; d=json.loads(open('gpurun_out/c5a.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['parity']['match'])"
ncu --set full --import-source on -k regex:mcm_batch_warp -c 1 -o gpurun_out/c5a_warp3 python bench.py --workload c5a --steps 1 --warmup 1 --no-cpu-baseline --no-companion --e2e-steps 0 > /dev/null 2>&1
