"""Debug: qkvo M=64 Int8Linear forward (split-K GEMM) for ncu."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2208_07339_b200 as pkg
from paper_2208_07339_b200.synthetic import planted_pair_device

k, n = 5120, 5120
x_all, w, _ = planted_pair_device(64, k, n, 6, 20.0, seed=3, device="cuda")
lin = pkg.Int8Linear(w, 6.0)
x = x_all[:64].contiguous()
for _ in range(5):
    lin(x)
torch.cuda.synchronize()
