"""development: host<->device copy rates for the e2e path (pinned torch buffers, 25 MB)."""
import time

import torch

n = 25165824 // 8
h = torch.randn(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
print("pinned:", h.is_pinned())
for name, f in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))]:
    f()
    torch.cuda.synchronize()
    t0 = time.time()
    for _ in range(10):
        f()
    torch.cuda.synchronize()
    dt = (time.time() - t0) / 10
    print(f"{name}: {dt * 1e3:.2f} ms per 25 MB -> {25165824 / dt / 1e9:.1f} GB/s")
