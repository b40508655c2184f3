"""Host->device bandwidth probe (pinned), single vs chunked copies."""
import time

import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunks in (1, 8, 32):
    s = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for it in range(3):
        step = n // chunks
        for c in range(chunks):
            with torch.cuda.stream(s[c % 2]):
                d[c * step:(c + 1) * step].copy_(h[c * step:(c + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"chunks {chunks}: {n / dt / 1e9:.1f} GB/s")
