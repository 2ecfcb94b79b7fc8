python -m pytest tests/test_gpu_mcm.py tests/test_gpu_batch.py -m gpu -x -q 2>&1 | tail -3
python bench.py --workload c5a --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c5a.json 2> gpurun_out/c5a.err; tail -c 600 gpurun_out/c5a.json; tail -3 gpurun_out/c5a.err
PIPEDP_MCM_BATCH_WARP=0 python bench.py --workload c5a --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c5a_sq.json 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/c5a_sq.json
