for m in 0 1; do for w in c2 c4 c5b; do PIPEDP_D2H_MODE=$m timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mode $m $w', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))"; done; done
python - <<'P'
import numpy as np, time, ctypes
a = np.ones(1 << 27, np.int64); b = np.empty_like(a)
for i in range(3):
    t = time.perf_counter(); b[:] = a; dt = time.perf_counter() - t
    print("numpy 1-thread copy GB/s", a.nbytes / dt / 1e9)
P
