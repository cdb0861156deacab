"""Nodes and edges of the captured cfg3 decode-step graph (dev tool): node
types in order and each edge's type (0 default, 1 programmatic launch,
2 programmatic event)."""
import sys
from pathlib import Path

import torch
from cuda.bindings import runtime as rt

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

run = bench.WorkloadRun("cfg3_decode", "cuda", False)
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    for _ in range(3):
        run.step()
torch.cuda.synchronize()
cg = torch.cuda.CUDAGraph(keep_graph=True)
# the GraphedCall form: captured on the warm-up stream
with torch.cuda.graph(cg, stream=side if "same" in sys.argv else None):
    run.step()
g = cg.raw_cuda_graph()
g = rt.cudaGraph_t(init_value=g)
err, nodes, n = rt.cudaGraphGetNodes(g, 0)
err, nodes, n = rt.cudaGraphGetNodes(g, n)
print("nodes:", n)
for i, nd in enumerate(nodes):
    err, t = rt.cudaGraphNodeGetType(nd)
    extra = ""
    if t == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel:
        extra = "kernel"
    print(i, t, extra)
res = rt.cudaGraphGetEdges_v2(g, 0)
print(res[0], len(res))
err, frm, to, data, ne = rt.cudaGraphGetEdges_v2(g, res[-1])
idx = {int(nd): i for i, nd in enumerate(nodes)}
for a, b, d in zip(frm, to, data):
    print(f"edge {idx[int(a)]} -> {idx[int(b)]} type {d.type} from_port {d.from_port} to_port {d.to_port}")
