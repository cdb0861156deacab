"""Dev micro-benchmark: issue cost of decode-shape tcgen05 MMAs (M=128, small N)."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2208_07339_b200 import _native as nat  # noqa: E402

L = nat.lib()
f = L.i8mm_debug_mma_small
f.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_void_p]
cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
for n_tok, n_acc, per_commit in [(16, 4, 4), (16, 16, 0), (16, 4, 0), (32, 8, 0), (64, 4, 0), (256, 1, 0),
                                 (16, 16, 4)]:
    iters = 2000
    f(iters, n_tok, n_acc, per_commit, ctypes.c_void_p(cyc.data_ptr()), None)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    f(iters, n_tok, n_acc, per_commit, ctypes.c_void_p(cyc.data_ptr()), None)
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3
    mmas = iters * 4
    print(f"N={n_tok:3d} n_acc={n_acc:2d} commit/{per_commit:7d}: {us / mmas * 1e3:7.1f} ns/MMA wall")
