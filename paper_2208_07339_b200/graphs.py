"""CUDA-graph capture of a fixed sequence of layer calls (decode serving).

A decode step is a handful of short launches (one cooperative decode kernel
per projection); from Python each costs ~30 us of host work, about as long as
the kernel itself. ``GraphedCall`` captures the step once on static tensors
(inputs, workspaces and outputs come from the graph's private memory pool) and
``replay()`` re-launches the whole sequence with one host call. Copy new
inputs into ``static_inputs`` (``copy_``) before a replay; the outputs are
overwritten in place.
"""

from __future__ import annotations

from typing import Callable

import torch

from . import _native as nat


class GraphedCall:
    def __init__(self, fn: Callable, *static_inputs: torch.Tensor, warmup: int = 3,
                 keep_graph: bool = False) -> None:
        self.fn = fn
        self.static_inputs = static_inputs
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up outside the graph: lazy init, allocator
            for _ in range(warmup):
                fn(*static_inputs)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph(keep_graph=keep_graph)  # keep: raw_cuda_graph() (tests)
        n0 = nat.launch_count()
        # captured on the warm-up stream: per-stream state the warm-up created
        # (decode workspaces, initialised once) is reused, so no initialisation
        # node (a memset between two kernels breaks their programmatic edge)
        # lands in the graph
        with torch.cuda.graph(self.graph, stream=side):
            self.output = fn(*static_inputs)
        self.kernels = nat.launch_count() - n0  # library kernels replayed per call

    def replay(self):
        self.graph.replay()
        return self.output
