# scratch job script for ad-hoc gpurun calls (the round evidence runs via tools/evidence.sh)
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -c 400
