import torch
x = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
y = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
z = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
def t(fn, nbytes, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    return nbytes / ms / 1e6
print("fill 4GB  GB/s %.0f" % t(lambda: x.fill_(1), 4 << 30))
print("zero 4GB  GB/s %.0f" % t(lambda: x.zero_(), 4 << 30))
print("copy 2GB  GB/s %.0f (r+w)" % t(lambda: y.copy_(z), 4 << 30))
xs = x.view(torch.float32).view(-1, 4096)
print("sum 4GB  GB/s %.0f (read)" % t(lambda: x.view(torch.float32).sum(), 4 << 30))
