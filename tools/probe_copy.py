import torch
n = 4096 * 262144
a = torch.empty(n, dtype=torch.uint8, device="cuda"); b = torch.empty_like(a)
a.random_(0, 255)
def t(fn, k=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(k): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / k
print("torch copy u8 1.07GB  %.3f ms" % t(lambda: b.copy_(a)))
a32, b32 = a.view(torch.int32), b.view(torch.int32)
print("torch copy i32        %.3f ms" % t(lambda: b32.copy_(a32)))
print("torch sum (read only) %.3f ms" % t(lambda: a32.sum()))
