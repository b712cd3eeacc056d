"""Streaming bandwidth probe on one B200 (context for the K4 roofline): read-only
sum over a large fp64 array, copy, and a 20-byte-per-element gather-free
stream (int32 + complex128) like the correction pairs."""
import torch

def t(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3

n = 2 * 1024**3 // 8 * 4          # 8 GiB of fp64
x = torch.ones(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
r = t(lambda: x.sum())
print(f"read (sum)  {x.numel() * 8 / r / 1e9:.0f} GB/s")
c = t(lambda: y.copy_(x))
print(f"copy        {2 * x.numel() * 8 / c / 1e9:.0f} GB/s")
