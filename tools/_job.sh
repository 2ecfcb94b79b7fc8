mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sdp.py tests/test_dropin.py -x -q > gpurun_out/pytest_s.txt 2>&1; tail -1 gpurun_out/pytest_s.txt; grep -E "^E |FAILED" gpurun_out/pytest_s.txt | head -5
timeout 100 python bench.py --workload c2 --no-cpu-baseline --e2e-steps 0 --steps 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', round(d['ms_per_step'],1), d['parity']['match'], d['roofline']['kernel'])"
timeout 1200 python tools/table1.py --out gpurun_out/table1.csv
