"""Debug: host enqueue cost vs device time of the cfg3 decode step."""
import sys
import time
import torch
sys.path.insert(0, ".")
import paper_2208_07339_b200 as pkg
from paper_2208_07339_b200.synthetic import planted_pair_device

layers = [(8, 5120, 5120)] * 4 + [(8, 5120, 20480), (8, 20480, 5120)]
mods, xs = [], []
for li, (m, k, n) in enumerate(layers):
    x, w, _ = planted_pair_device(m, k, n, 6, 20.0, seed=li, device="cuda")
    mods.append(pkg.Int8Linear(w, alpha=6.0))
    xs.append(x)


def step():
    for mod, x in zip(mods, xs):
        mod(x)


for _ in range(10):
    step()
torch.cuda.synchronize()
N = 200
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
s.record()
for _ in range(N):
    step()
e.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"device {s.elapsed_time(e) / N * 1e3:.1f} us/step, host enqueue {1e6 * (t1 - t0) / N:.1f} us/step")

# CUDA graph of the whole step (static inputs / workspaces / outputs)
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(st)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    step()
torch.cuda.synchronize()
for _ in range(10):
    g.replay()
torch.cuda.synchronize()
t0 = time.perf_counter()
s.record()
for _ in range(N):
    g.replay()
e.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"graph: device {s.elapsed_time(e) / N * 1e3:.1f} us/step, host {1e6 * (t1 - t0) / N:.1f} us/step")
