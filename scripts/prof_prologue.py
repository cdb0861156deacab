"""Driver for ncu captures of the prologue kernels (dev tool)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2208_07339_b200 import gemm as G
from paper_2208_07339_b200.synthetic import planted_pair_device

m, k, n = (int(v) for v in (sys.argv[1:4] if len(sys.argv) >= 4 else (16384, 16384, 256)))
x, w, _ = planted_pair_device(m, k, n, 6, 20.0, 0)
for _ in range(3):
    scan = G.scan_outliers(x, 6.0)
    G._quantize_rows(x, scan)
torch.cuda.synchronize()
print("done")
