"""Per-CTA timeline of the decode kernels (dev tool): %globaltimer stamps.

    python scripts/decode_timeline.py fc1 1
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

PROJ = {"qkvo": (5120, 5120), "fc1": (5120, 20480), "fc2": (20480, 5120)}
name, m = sys.argv[1], int(sys.argv[2])
k, n = PROJ[name]
L = nat.lib()
L.i8mm_debug_set_decode_max_m(256)
x, w, _ = planted_pair_device(m, k, n, 6, 20.0, seed=3, device="cuda")
lin = pkg.Int8Linear(w, 6.0, check_finite=False)
sms = torch.cuda.get_device_properties(0).multi_processor_count
g = torch.zeros(sms * 64, dtype=torch.int64, device="cuda")
for _ in range(3):
    lin(x)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush.zero_()
x.sum()  # the tokens are L2-resident (written by the previous layer), the weights are not
L.i8mm_debug_decode_timeline(g.data_ptr())
lin(x)
torch.cuda.synchronize()
L.i8mm_debug_decode_timeline(None)
G = g.view(sms, 64).cpu().double()
t0 = G[:, 0][G[:, 0] > 0].min()


def col(i):
    v = G[:, i]
    v = v[v > 0] - t0
    if v.numel() == 0:
        return "-"
    return f"min {v.min() / 1e3:7.2f} med {v.median() / 1e3:7.2f} max {v.max() / 1e3:7.2f} us"


labels = {0: "start", 1: "waited", 2: "X landed", 3: "cluster barrier 1", 4: "panels ready",
          5: "first MMA", 6: "MMA issued", 7: "1st tmem_full", 8: "epi done", 9: "end"}
for i, lab in labels.items():
    v = G[:, i]
    arg = int(torch.argmax(v)) if (v > 0).any() else -1
    print(f"{lab:22s} {col(i)}  (max at CTA {arg})")
print(lin.last_stats())
