timeout 300 python -m pytest tests/test_gpu_sdp.py -x -q -k "large_table" 2>&1 | tail -2
