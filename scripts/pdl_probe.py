"""Dev probe: do two back-to-back decode launches overlap (programmatic
dependent launch)? Timeline stamps of both, eager, enqueued without a sync."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2208_07339_b200 import _native as nat, build as _build  # noqa: E402
nat.load_library(_build.lib_path(devtools=True))
import paper_2208_07339_b200 as pkg  # noqa: E402
from paper_2208_07339_b200.synthetic import planted_pair_device  # noqa: E402

L = nat.lib()
sms = torch.cuda.get_device_properties(0).multi_processor_count
x, w, _ = planted_pair_device(8, 5120, 5120, 6, 20.0, seed=3, device="cuda")
x2, w2, _ = planted_pair_device(8, 5120, 5120, 6, 20.0, seed=4, device="cuda")
l1 = pkg.Int8Linear(w, 6.0, check_finite=False)
l2 = pkg.Int8Linear(w2, 6.0, check_finite=False)
bufs = [torch.zeros(sms * 32, dtype=torch.int64, device="cuda") for _ in range(2)]
for _ in range(3):
    l1(x), l2(x2)
torch.cuda.synchronize()
big = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
big.zero_()  # keeps the GPU busy while the host enqueues both
L.i8mm_debug_decode_timeline(bufs[0].data_ptr())
l1(x)
L.i8mm_debug_decode_timeline(bufs[1].data_ptr())
l2(x2)
L.i8mm_debug_decode_timeline(None)
torch.cuda.synchronize()
G = [b.view(sms, 32).cpu().double() for b in bufs]
t0 = G[0][:, 0][G[0][:, 0] > 0].min()
for name, g in zip(("first", "second"), G):
    st = g[:, 0][g[:, 0] > 0] - t0
    en = g[:, 9][g[:, 9] > 0] - t0
    wt = g[:, 1][g[:, 1] > 0] - t0
    print(f"{name}: start {st.min() / 1e3:6.2f}..{st.max() / 1e3:6.2f}  waited {wt.min() / 1e3:6.2f}..{wt.max() / 1e3:6.2f}"
          f"  end {en.min() / 1e3:6.2f}..{en.max() / 1e3:6.2f} us")
