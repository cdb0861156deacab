"""Debug: cfg2 step eager vs CUDA-graph replay (device time)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2208_07339_b200 as pkg
from paper_2208_07339_b200.synthetic import planted_pair_device

layers = [(16384, 4096, 16384), (16384, 16384, 4096)]
mods, xs = [], []
for li, (m, k, n) in enumerate(layers):
    x, w, _ = planted_pair_device(m, k, n, 6, 20.0, seed=li, device="cuda")
    mods.append(pkg.Int8Linear(w, alpha=6.0))
    xs.append(x)


def step():
    for mod, x in zip(mods, xs):
        mod(x)


def t(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


g = pkg.GraphedCall(lambda *xx: [m(x) for m, x in zip(mods, xx)], *xs)
for _ in range(3):
    print(f"eager {t(step):.4f} ms  graph {t(g.replay):.4f} ms", flush=True)
