"""Per-CTA timeline of the swap-AB mid-M GEMM (dev tool; dev build):

    python scripts/swapab_timeline.py M K N
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2208_07339_b200 import _native as nat, build as _build  # noqa: E402
nat.load_library(_build.lib_path(devtools=True))
import paper_2208_07339_b200 as pkg  # noqa: E402
from paper_2208_07339_b200.synthetic import planted_pair_device  # noqa: E402

m, k, n = (int(v) for v in sys.argv[1:4])
x, w, _ = planted_pair_device(m, k, n, 6, 20.0, seed=3, device="cuda")
lin = pkg.Int8Linear(w, 6.0)
for _ in range(3):
    lin(x)
torch.cuda.synchronize()
g = torch.zeros(256 * 16, dtype=torch.int64, device="cuda")
torch.empty(256 << 20, dtype=torch.uint8, device="cuda").zero_()
nat.lib().i8mm_debug_swapab_timeline(g.data_ptr())
lin(x)
torch.cuda.synchronize()
nat.lib().i8mm_debug_swapab_timeline(None)
G = g.view(256, 16).cpu().double()
live = G[:, 0] > 0
G = G[live]
t0 = G[:, 0].min()
names = {0: "setup done", 1: "dependency released", 2: "MMAs seg0 issued", 3: "MMAs seg1 issued",
         5: "epi reaches seg0", 6: "epi reaches seg1", 8: "partials ready seg0", 9: "partials ready seg1",
         11: "acc ready seg0", 12: "acc ready seg1", 15: "epilogue done", 14: "end"}
print("CTAs", int(live.sum()))
for i, nm in names.items():
    v = G[:, i]
    v = v[v > 0]
    if v.numel():
        print(f"{nm:22s} min {(v.min() - t0) / 1e3:8.2f} med {(v.median() - t0) / 1e3:8.2f} max {(v.max() - t0) / 1e3:8.2f} us")
for c in range(0, G.shape[0], max(1, G.shape[0] // 6)):
    print("cta", c, " ".join(f"{i}:{(G[c, i] - t0) / 1e3:.2f}" for i in range(16) if G[c, i] > 0))
