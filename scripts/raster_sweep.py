"""GROUP_M raster sweep of the prefill GEMM per layer shape (dev tool).

    python scripts/raster_sweep.py [shape ...]   shape = MxKxN

Prints, per shape and I8MM_GROUP_M value (0 = the library's heuristic), the
Int8Linear forward time and the GEMM alone (events around i8mm_linear_gemm).
"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2208_07339_b200 as pkg  # noqa: E402
from paper_2208_07339_b200.synthetic import planted_pair_device  # noqa: E402


class T:
    def __init__(self):
        self.p = []
        self.on = True

    def mark(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.p.append(e)


def t_ev(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]] or [
    (16384, 12288, 49152), (16384, 49152, 12288), (16384, 4096, 16384), (16384, 16384, 4096)]
groups = [int(g) for g in os.environ.get("GROUPS", "0,1,2,4,6,8,12,16").split(",")]
for (m, k, n) in shapes:
    x, w, _ = planted_pair_device(m, k, n, 6, 20.0, 0)
    lin = pkg.Int8Linear(w, 6.0)
    ops = 2 * m * n * k
    for g in groups:
        if g:
            os.environ["I8MM_GROUP_M"] = str(g)
        else:
            os.environ.pop("I8MM_GROUP_M", None)
        t = t_ev(lambda: lin(x))
        tm = T()
        for _ in range(5):
            lin.matmul(x, _timer=tm)
        torch.cuda.synchronize()
        g_ms = sum(tm.p[i].elapsed_time(tm.p[i + 1]) for i in range(0, len(tm.p), 2)) / 5
        print(f"M={m} K={k} N={n} GROUP_M={g or 'auto'}: layer {t:.3f} ms ({ops / t / 1e9:.0f} TOPS)"
              f" gemm {g_ms:.3f} ms ({ops / g_ms / 1e9:.0f} TOPS)", flush=True)
    del lin, x, w
    torch.cuda.empty_cache()
