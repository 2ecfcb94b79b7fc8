O=gpurun_out/r02j; mkdir -p $O
for ap in 256 512; do for mid in 2 4 6; do
PIPEDP_CLUSTER_AP=$ap PIPEDP_CLUSTER_MID=$mid PIPEDP_SDP_CHUNKED=0 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b_${ap}_${mid}.json 2>&1
echo "ap=$ap mid=$mid $(python -c "import json; d=json.loads(open('$O/b_${ap}_${mid}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['parity']['match'])")"
done; done
