O=gpurun_out/r02k; mkdir -p $O
PIPEDP_SDP_CHUNKED=0 timeout 120 python tools/cluster_probe.py 20
PIPEDP_SDP_CHUNKED=0 timeout 120 python tools/cluster_probe.py 20 modular-add
timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, paper_2008_01938_b200 as pd
from oracle import pyoracle
orc = pyoracle.load_c()
for (n,k,op,cap) in [(20000,512,'min',2048),(30000,300,'modular-add',1500),(50000,1024,'max',4096),(300000,2000,'modular-add',8000)]:
    inst = pd.generate_sdp(n=n,k=k,op=op,seed=5,a1_cap=cap)
    t = pd.solve_sequential(inst)
    w,_ = orc.sdp_solve(inst.offsets, inst.init, n, op)
    print(op, n, k, 'match', np.array_equal(t.cells, w), flush=True)
"
for ap in 256; do for mid in 4 6 8; do
PIPEDP_CLUSTER_AP=$ap PIPEDP_CLUSTER_MID=$mid PIPEDP_SDP_CHUNKED=0 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b_${ap}_${mid}.json 2>&1
echo "ap=$ap mid=$mid $(python -c "import json; d=json.loads(open('$O/b_${ap}_${mid}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['parity']['match'])" 2>&1 | tail -1)"
done; done
