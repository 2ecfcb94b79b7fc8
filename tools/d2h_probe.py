"""Host<->device copy bandwidth probe (pinned and pageable), GB/s."""
import time
import torch

n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for pin in (True, False):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=pin)
    h.fill_(1)
    for name, fn in (("d2h", lambda: h.copy_(d)), ("h2d", lambda: d.copy_(h))):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        print(f"{'pinned' if pin else 'pageable'} {name}: {3 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
