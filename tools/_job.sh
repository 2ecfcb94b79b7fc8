for g in 256 444 512; do for fm in 3 4 6 8; do G=$g TAG="far$fm mid1" PIPEDP_SDP_FAR_MAX=$fm PIPEDP_SDP_MID_WARPS=1 PYTHONPATH=. timeout 100 python tools/chunk_probe.py 2>&1 | tail -1; done; done
