"""PCIe copy bandwidth on this box (dev tool): pinned host <-> device, each
direction alone and both at once, 512 MiB per copy, CUDA events."""
import json

import torch

n = 512 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


h2d = t(lambda: d1.copy_(h1, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
bi = t(both)
print(json.dumps({"h2d_gbs": n / h2d / 1e6, "d2h_gbs": n / d2h / 1e6,
                  "bidir_gbs_each": n / bi / 1e6}))
