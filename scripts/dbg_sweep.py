"""Debug: decode_sweep's exact pattern for fc1 M=16 then M=32, per-iteration times."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2208_07339_b200 as pkg
from paper_2208_07339_b200.synthetic import planted_pair_device


def t_ev(fn, iters=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    out = []
    for _ in range(iters):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        out.append(round(s.elapsed_time(e) * 1e3, 1))
    return out


k, n = 5120, 20480
x_all, w, _ = planted_pair_device(32, k, n, 6, 20.0, seed=3, device="cuda")
lin = pkg.Int8Linear(w, 6.0)
for m in (16, 32, 16, 32):
    x = x_all[:m].contiguous()
    r = t_ev(lambda: lin(x))
    print(m, lin.last_stats().get("decomposed_cols"), r, flush=True)
