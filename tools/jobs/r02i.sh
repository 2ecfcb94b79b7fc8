O=gpurun_out/r02i; mkdir -p $O
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, paper_2008_01938_b200 as pd
from oracle import pyoracle
orc = pyoracle.load_c()
for (n,k,op,cap) in [(20000,512,'min',2048),(30000,300,'modular-add',1500),(50000,1024,'max',4096)]:
    inst = pd.generate_sdp(n=n,k=k,op=op,seed=5,a1_cap=cap)
    plan = pd.SdpPlan(1, n, k, inst.a1, inst.offsets, inst.init, op, device=0)
    print(plan.describe(), flush=True)
    t = pd.solve_sequential(inst)
    w,_ = orc.sdp_solve(inst.offsets, inst.init, n, op)
    print(op, n, k, 'match', np.array_equal(t.cells, w), flush=True)
" > $O/quick.txt 2>&1; cat $O/quick.txt
timeout 900 python -m pytest tests/test_gpu_sdp.py tests/test_dropin.py -m gpu -q -x > $O/pytest_sdp.txt 2>&1; tail -3 $O/pytest_sdp.txt
PIPEDP_SDP_CHUNKED=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_c2_pipe.json 2>&1; tail -c 300 $O/bench_c2_pipe.json; echo
PIPEDP_SDP_CHUNKED=0 PIPEDP_SDP_CLUSTER=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_c2_v2.json 2>&1; tail -c 300 $O/bench_c2_v2.json; echo
