set -x
for v in 0 1 0 1; do echo PROG=$v; PIPEDP_D2H_PROGRESSIVE=$v python tools/e2e_breakdown.py 2>&1 | head -3; done
python -m pytest tests/test_gpu_sdp.py tests/test_dropin.py -m gpu -x -q 2>&1 | tail -3
