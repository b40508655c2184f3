"""HBM ceilings on this B200 for the kernels whose traffic is mostly writes
(K4's C~ store, K2's Gram store): write-only fill, read-only sum, and the
read+write copy MEASURED_PEAKS.json uses, each over 4 GiB (best of 10)."""
import torch

n = 1 << 30  # float32 elements: 4 GiB
a = torch.empty(n, dtype=torch.float32, device="cuda")
b = torch.empty(n, dtype=torch.float32, device="cuda")
a.fill_(1.0)


def best(fn, nbytes):
    ts = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return nbytes / (min(ts) / 1e3) / 1e9


print(f"write-only fill_: {best(lambda: b.fill_(2.0), 4 * n):.0f} GB/s")
print(f"write-only zero_ (memset): {best(lambda: b.zero_(), 4 * n):.0f} GB/s")
print(f"read-only sum: {best(lambda: a.sum(), 4 * n):.0f} GB/s")
print(f"copy (read+write bytes): {best(lambda: b.copy_(a), 8 * n):.0f} GB/s")
