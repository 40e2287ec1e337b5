"""Effective HBM read bandwidth of short streaming reads (development tool):
how fast can a ~18 MB weight matrix (config 4 at g = 4) be read at all?
Times torch's own read-only reduction and a device-to-device copy per size,
L2 flushed before every launch, CUDA events around each launch (median)."""
import torch

dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def t_us(fn, reps=30):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for mb in (4, 8, 17.7, 32, 64, 128, 512):
    n = int(mb * (1 << 20)) // 4
    x = torch.ones(n, dtype=torch.int32, device=dev)
    y = torch.empty_like(x)
    r = t_us(lambda: x.sum())
    c = t_us(lambda: y.copy_(x))
    print(f"{mb:6.1f} MB  sum {r:8.2f} us ({n * 4 / r / 1e3:7.0f} GB/s read)   "
          f"copy {c:8.2f} us ({n * 4 / c / 1e3:7.0f} GB/s read)")
