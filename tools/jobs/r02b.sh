O=gpurun_out/r02b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_dropin.py tests/test_gpu_mcm.py -m gpu -q -x --durations=10 > $O/pytest_engine.txt 2>&1; tail -15 $O/pytest_engine.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
