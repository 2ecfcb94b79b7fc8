O=gpurun_out/r02g; mkdir -p $O
timeout 600 python tools/sanitize_cases.py > $O/cases.txt 2>&1; tail -3 $O/cases.txt
timeout 900 python -m pytest tests/test_gpu_mcm.py tests/test_gpu_batch.py -m gpu -q -x > $O/pytest_mcm.txt 2>&1; tail -3 $O/pytest_mcm.txt
timeout 600 python bench.py --workload c3 --mcm-kernel tournament --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_c3t.json 2>&1; tail -c 400 $O/bench_c3t.json; echo
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -m gpu -q > $O/pytest_sanitizer.txt 2>&1; tail -5 $O/pytest_sanitizer.txt
cp gpurun_out/sanitizer_*.txt $O/ 2>/dev/null
