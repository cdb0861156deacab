"""Debug: HostIOPipeline e2e step time, join=True vs join=False, cfg2 shapes."""
import sys
import time
import torch
sys.path.insert(0, ".")
import paper_2208_07339_b200 as pkg
from paper_2208_07339_b200.synthetic import planted_pair_device

dev = torch.device("cuda", 0)
layers = [(16384, 4096, 16384), (16384, 16384, 4096)]
mods, xh, yh = [], [], []
for li, (m, k, n) in enumerate(layers):
    x, w, _ = planted_pair_device(m, k, n, 6, 20.0, seed=li, device=dev)
    mods.append(pkg.Int8Linear(w, alpha=6.0))
    xh.append(x.cpu().pin_memory())
    yh.append(torch.empty((m, n), dtype=torch.float16).pin_memory())
torch.cuda.synchronize()
pipe = pkg.HostIOPipeline(dev, chunks=4)


def run(join, steps=6):
    for _ in range(2):
        pipe.run(list(zip(mods, xh, yh)), inputs_ready=True, join=join)
    pipe.join()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    for _ in range(steps):
        pipe.run(list(zip(mods, xh, yh)), inputs_ready=True, join=join)
    pipe.join()
    e.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"join={join}: {s.elapsed_time(e) / steps:.2f} ms/step (host enqueue {1e3 * (t1 - t0) / steps:.2f} ms/step, "
          f"wall {1e3 * (t2 - t0) / steps:.2f})", flush=True)


for j in (True, False, True, False):
    run(j)
