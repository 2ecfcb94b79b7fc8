"""C5b mode breakdown: classify the 65,536 instances the way sdp_batch_warp
does (1: offset 1; 2: S* covers [2, 127]; 0: general) and time the batch
kernel on 8,192 instances of each mode (GPU).  usage: python tools/batch_modes.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2008_01938_b200 as pd  # noqa: E402

N, K, B = 1 << 16, 64, 65536
offs, init = pd.generate_sdp_batch(N, K, 0, B)
S = np.zeros((B, 128), bool)  # S[b, d]: offset d present (d < 128)
rows = np.repeat(np.arange(B), K)
m = offs.reshape(-1) < 128
S[rows[m], offs.reshape(-1)[m]] = True
reach = np.zeros((B, 128), bool)
reach[:, 0] = True
for v in range(1, 128):  # v in S* iff v - d in S* for some offset d <= v
    reach[:, v] = (S[:, 1:v + 1] & reach[:, v - 1::-1][:, :v]).any(axis=1)
mode = np.where(S[:, 1], 1, np.where(reach[:, 2:].all(axis=1), 2, 0)).astype(np.int8)
print("modes:", {m: int((mode == m).sum()) for m in (0, 1, 2)}, flush=True)
for m in ([int(a) for a in sys.argv[1:]] or (0, 1, 2)):
    idx = np.nonzero(mode == m)[0][:8192]
    cnt = len(idx)
    if cnt == 0:
        continue
    o, i = offs[idx].copy(), init[idx].copy()
    plan = pd.SdpPlan(cnt, N, K, i.shape[1], o.reshape(-1), i.reshape(-1), "min", device=0)
    d_in = torch.from_numpy(i.reshape(-1)).cuda()
    d_out = torch.empty(cnt * N, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        plan.execute(d_in.data_ptr(), d_out.data_ptr(), st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3):
        plan.execute(d_in.data_ptr(), d_out.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"mode {m}: {cnt} instances {ms:.3f} ms -> {ms * 65536 / cnt:.1f} ms per 65536", flush=True)
