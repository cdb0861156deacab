"""Per-layer timeline of one cfg3 decode step (dev tool): the six OPT-13B
projections at M = 8 back to back, as bench.py --workload cfg3_decode runs them
(eager, PDL-chained), with %globaltimer stamps of every layer's prep and stream
kernels, relative to the first layer's prep start.

    python scripts/decode_chain_timeline.py
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2208_07339_b200 import _native as nat, build as _build  # noqa: E402
nat.load_library(_build.lib_path(devtools=True))
import bench  # noqa: E402

L = nat.lib()
run = bench.WorkloadRun("cfg3_decode", "cuda", False)
sms = torch.cuda.get_device_properties(0).multi_processor_count
bufs = [torch.zeros(sms * 64, dtype=torch.int64, device="cuda") for _ in run.layers]
for _ in range(5):
    run.step()
torch.cuda.synchronize()
graph = len(sys.argv) > 1 and sys.argv[1] == "graph"
if graph:  # the bench's form: one CUDA graph of the step (PDL edges between the layers)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):  # this stream's decode workspaces exist before the capture
            run.step()
        with torch.cuda.graph(g, stream=s):
            for mod, x, b in zip(run.mods, run.xs, bufs):
                L.i8mm_debug_decode_timeline(b.data_ptr())
                mod(x)
    L.i8mm_debug_decode_timeline(None)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for b in bufs:
        b.zero_()
    g.replay()
else:
    for mod, x, b in zip(run.mods, run.xs, bufs):
        L.i8mm_debug_decode_timeline(b.data_ptr())
        mod(x)
    L.i8mm_debug_decode_timeline(None)
torch.cuda.synchronize()
G = [b.view(sms, 64).cpu().double() for b in bufs]
t0 = G[0][:, 0][G[0][:, 0] > 0].min()


def stat(g, i, f=min):
    v = g[:, i]
    v = v[v > 0]
    if v.numel() == 0:
        return float("nan")
    return float((f(v) - t0) / 1e3)


names = ["q", "k", "v", "o", "fc1", "fc2"]
cols = [(0, "start", min), (0, "start (last CTA)", max), (1, "waited", max), (2, "X landed", max),
        (10, "flags", max), (11, "cluster wait", max), (12, "partials pushed", max), (13, "mask pushed", max),
        (3, "cluster barrier 1", max), (14, "row scales", max), (15, "codes pushed", max), (16, "proxy fence", max),
        (17, "w4 prefetch done", max), (28, "w4 codes done", max), (32, "t0 item0 start", max), (33, "t0 item0 codes", max), (34, "t0 item1 start", max), (18, "lead writes", max), (4, "panels ready", max), (5, "1st MMA", max),
        (6, "MMA issued", max)] + [(19, "setup: bars+W", max), (20, "setup: pdl wait", max), (21, "setup: X issued", max),
        (22, "setup: L2 pf+dst", max), (23, "setup: tmem alloc", max), (24, "setup: cand loads", max),
        (25, "setup: zeroing", max)] + [(35, "epi seg loop", max), (38, "epi W[O] staged", max), (37, "contrib release", max), (36, "fin spin done", max), (7, "1st tmem_full", max), (8, "epi done", max), (9, "end", max)]
print("us from layer q's prep start (min or max over CTAs); CTAs per layer:", [int((g[:, 0] > 0).sum()) for g in G])
print(f"{'':18s}" + "".join(f"{n:>8s}" for n in names))
med = lambda v: v.median()
for i, lab, f in cols:
    print(f"{lab:18s}" + "".join(f"{stat(g, i, f):8.2f}" for g in G) + "   med" +
          "".join(f"{stat(g, i, med):8.2f}" for g in G))

# the latest CTAs of each layer: what they did (patched entries per segment, role per segment: 0 contributor, 1 finisher, 2 full)
for name, g in zip(names, G):
    end = g[:, 9]
    order = torch.argsort(end, descending=True)[:6]
    rows = []
    for c in order.tolist():
        if end[c] <= 0:
            continue
        rows.append(f"cta {c:3d} end {(end[c] - t0) / 1e3:6.2f} 1st-tmem {(g[c, 7] - t0) / 1e3:6.2f} "
                    f"ents {[int(g[c, 26 + k]) for k in range(2)]} roles {[int(g[c, 29 + k]) for k in range(3)]} "
                    f"seg-loop {(g[c, 35] - t0) / 1e3:6.2f} W[O] {(g[c, 38] - t0) / 1e3:6.2f} spin {(g[c, 36] - t0) / 1e3:6.2f} "
                    f"MMA-issued {(g[c, 6] - t0) / 1e3:6.2f} 1stMMA {(g[c, 5] - t0) / 1e3:6.2f}")
    print(name, "latest:"); [print("   ", r) for r in rows]
    ents = g[:, 26:29].sum(1)
    print("    median end (no patched) {:.2f} / (patched) {:.2f}".format(
        float(((end[(ents == 0) & (end > 0)] - t0) / 1e3).median()) if ((ents == 0) & (end > 0)).any() else -1,
        float(((end[(ents > 0) & (end > 0)] - t0) / 1e3).median()) if ((ents > 0) & (end > 0)).any() else -1))
