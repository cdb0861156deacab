"""Time the prefill prologue (i8mm_linear_prologue: scan, compact, row scales,
codes, W[O,:] gather, column fixup) alone at the cfg2 layer shapes.

Dev tool (run under gpurun). Prints one JSON line per layer: mean us per call
over `iters` back-to-back calls (CUDA events), and the X-side HBM rate
(2 reads of X + one write of Xq, the algorithmic bytes of the two-pass row
quantizer). A/B kernel variants through the I8MM_* environment switches.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2208_07339_b200 as pkg  # noqa: E402
from paper_2208_07339_b200 import _native as nat  # noqa: E402
from paper_2208_07339_b200._tensors import stream_handle  # noqa: E402

SHAPES = {"fc1": (16384, 4096, 16384), "fc2": (16384, 16384, 4096)}


def main() -> None:
    names = sys.argv[1:] or list(SHAPES)
    iters = 20
    torch.cuda.set_device(0)
    L = nat.lib()
    for name in names:
        m, k, n = SHAPES[name]
        g = torch.Generator(device="cuda").manual_seed(0)
        x = torch.randn((m, k), generator=g, device="cuda", dtype=torch.float32).mul_(0.5)
        cols = torch.randperm(k, device="cuda", generator=g)[:6]
        x[:, cols] *= 20.0
        x = x.half()
        w = torch.randn((k, n), generator=g, device="cuda", dtype=torch.float32).mul_(0.05).half()
        lin = pkg.Int8Linear(w, alpha=6.0)
        ws = torch.empty(L.i8mm_linear_workspace_size(m, k, n), dtype=torch.uint8, device="cuda")
        st = stream_handle()

        def call():
            nat.check(L.i8mm_linear_prologue(x.data_ptr(), x.stride(0), m, w.data_ptr(),
                                             w.stride(0), lin.wbuf.data_ptr(), k, n, 6.0,
                                             ws.data_ptr(), ws.numel(), st), "prologue")

        for _ in range(3):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            call()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / iters
        xbytes = 2 * m * k * 2 + m * k
        print(json.dumps({"layer": name, "mkn": [m, k, n], "us": round(us, 2),
                          "x_side_gbs": round(xbytes / us / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
