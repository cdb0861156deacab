"""Single-shape driver for ncu captures (dev tool): runs Int8Linear forward."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2208_07339_b200 as pkg
from paper_2208_07339_b200.synthetic import planted_pair_device

m, k, n = (int(v) for v in (sys.argv[1:4] if len(sys.argv) >= 4 else (16384, 4096, 16384)))
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
x, w, _ = planted_pair_device(m, k, n, 6, 20.0, 0)
lin = pkg.Int8Linear(w, 6.0)
for _ in range(iters):
    y = lin(x)
torch.cuda.synchronize()
print("done", lin.last_stats())
