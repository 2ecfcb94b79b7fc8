# scratch job script for ad-hoc gpurun calls (the round evidence runs via tools/evidence.sh)
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
