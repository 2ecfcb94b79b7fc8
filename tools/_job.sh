timeout 600 python -m pytest tests/test_gpu_sdp.py -x -q -k "chunked_int64" 2>&1 | tail -2
