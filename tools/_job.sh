timeout 900 python -m pytest tests/test_gpu_mcm.py -x -q -k "packed" 2>&1 | tail -2
