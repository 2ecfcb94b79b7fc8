timeout 300 python -m pytest tests/test_gpu_sdp.py tests/test_gpu_batch.py -x -q > gpurun_out/pytest_s.txt 2>&1; tail -2 gpurun_out/pytest_s.txt
export PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so
timeout 60 python tools/v2_profile.py 22
