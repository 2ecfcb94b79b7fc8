import sys
sys.path.insert(0, '.')
import numpy as np, torch, paper_2008_01938_b200 as pd
from oracle import pyoracle
orc = pyoracle.load_c()
n = 64
for B in (24, 1000):
    dims = pd.generate_mcm_batch(n, 300, B, 1, 100)
    plan = pd.McmPlan(B, n, dims.reshape(-1), device=0)
    size = pd.cell_count(n) + 1
    c = torch.full((B * size,), -1, dtype=torch.int64, device="cuda")
    s = torch.full((B * size,), -1, dtype=torch.int64, device="cuda")
    plan.execute(c.data_ptr(), s.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    c, s = c.cpu().numpy(), s.cpu().numpy()
    bad = 0
    for b in range(B):
        wc, _, ws = orc.mcm_solve(dims[b])
        if not (np.array_equal(c[b*size:(b+1)*size], wc) and np.array_equal(s[b*size:(b+1)*size], ws)):
            bad += 1
            if bad == 1:
                d = np.nonzero(c[b*size:(b+1)*size] != wc)[0]
                print("inst", b, "diff", d[:8], c[b*size + d[:4]], wc[d[:4]])
    print("B", B, plan.describe(), "bad", bad, flush=True)
