"""HBM read-rate probe (dev tool): device time of reading N bytes once from a
flushed L2, for the decode layer sizes (torch reductions / copies as the
reference streams)."""
import torch

flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def t(fn, it=20):
    ts = []
    for _ in range(it):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for mb in (26.2, 104.9, 419.4):
    n = int(mb * 1e6) // 16 * 16
    a = torch.empty(n, dtype=torch.uint8, device="cuda").random_(0, 255)
    b = torch.empty_like(a)
    us_sum = t(lambda: a.view(torch.int32).sum())
    us_copy = t(lambda: b.copy_(a))
    w = torch.randn(5120, int(n // 5120 // 2), dtype=torch.float16, device="cuda")
    x = torch.randn(8, 5120, dtype=torch.float16, device="cuda")
    us_gemv = t(lambda: x @ w)
    print(f"{mb:7.1f} MB: int32 sum {us_sum:7.1f} us = {n / us_sum / 1e3:6.0f} GB/s | copy {us_copy:7.1f} us = "
          f"{2 * n / us_copy / 1e3:6.0f} GB/s | cuBLAS fp16 M=8 GEMV over {w.numel() * 2 / 1e6:.0f} MB "
          f"{us_gemv:7.1f} us = {w.numel() * 2 / us_gemv / 1e3:6.0f} GB/s")
