"""Per-CTA timeline of the prefill GEMM (dev tool): %globaltimer stamps.

    python scripts/gemm_timeline.py qkvo 64
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2208_07339_b200 import _native as nat, build as _build  # noqa: E402
# the stamps are compiled only into the dev build (python -m paper_2208_07339_b200.build --devtools)
nat.load_library(_build.lib_path(devtools=True))
import paper_2208_07339_b200 as pkg  # noqa: E402
from paper_2208_07339_b200.synthetic import planted_pair_device  # noqa: E402

PROJ = {"qkvo": (5120, 5120), "fc1": (5120, 20480), "fc2": (20480, 5120),
        "cfg2fc1": (4096, 16384), "cfg2fc2": (16384, 4096)}
name, m = sys.argv[1], int(sys.argv[2])
k, n = PROJ[name]
L = nat.lib()
x, w, _ = planted_pair_device(m, k, n, 6, 20.0, seed=3, device="cuda")
lin = pkg.Int8Linear(w, 6.0)
g = torch.zeros(1024 * 16, dtype=torch.int64, device="cuda")
for _ in range(3):
    lin(x)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush.zero_()
L.i8mm_debug_decode_timeline(g.data_ptr())
lin(x)
torch.cuda.synchronize()
L.i8mm_debug_decode_timeline(None)
G = g.view(1024, 16).cpu().double()
live = G[:, 0] > 0
t0 = G[live, 0].min()
labels = {0: "start", 1: "setup+wait", 2: "1st TMA", 3: "1st MMA", 4: "MMA done(u0)",
          8: "epi wait", 5: "epi go", 6: "epi done(u0)", 9: "split fence", 10: "split count",
          11: "split emit", 7: "end"}
print(f"CTAs stamped: {int(live.sum())}")
for i, lab in labels.items():
    v = G[live, i]
    v = v[v > 0] - t0
    if v.numel() == 0:
        print(f"{lab:13s} -")
        continue
    print(f"{lab:13s} min {v.min() / 1e3:7.2f} med {v.median() / 1e3:7.2f} max {v.max() / 1e3:7.2f} us")

clk = torch.cuda.get_device_properties(0).clock_rate * 1e3 if hasattr(torch.cuda.get_device_properties(0), "clock_rate") else 1.9e9
for i, lab in {14: "producer waits (empty)", 12: "MMA waits (full)", 13: "MMA waits (tmem_empty)",
               15: "epilogue waits (tmem_full)"}.items():
    v = G[live, i]
    v = v[v > 0]
    if v.numel():
        print(f"{lab:28s} median {v.median() / 1e3:9.1f} kcycles  max {v.max() / 1e3:9.1f} kcycles")
