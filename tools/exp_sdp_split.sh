export PIPEDP_LIB=paper_2008_01938_b200/_lib/libpipedp_cuda_prof.so
for ar in 256 512 1024; do for mw in 2 4; do echo "== AREMOTE=$ar MID=$mw"; PIPEDP_SDP_AREMOTE=$ar PIPEDP_SDP_MID_WARPS=$mw python tools/role_profile.py 22 | grep -E "ms|chain|mid.fold|far.fold"; done; done
unset PIPEDP_LIB
timeout 300 python -m pytest tests/test_gpu_sdp.py -x -q 2>&1 | tail -2
