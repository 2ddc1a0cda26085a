"""Raw pinned host<->device copy bandwidth on this box (context for the e2e number)."""
import time
import torch

n = 2 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(name, round(3 * n / (time.perf_counter() - t) / 1e9, 1), "GB/s")
