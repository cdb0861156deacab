"""Host-buffer execution of Int8 linear layers with the PCIe copies overlapped.

The reference computes on host arrays (its DenseMatrix lives in host memory);
a drop-in caller hands host buffers in and expects host buffers back. Doing
that naively serialises host->device copy, compute and device->host copy.
``HostIOPipeline`` keeps the copy engines and the tensor cores busy at once:

* all inputs are copied host->device on one stream, in call order, so layer
  i+1's input streams in while layer i computes;
* each layer runs one prologue over all its rows, then the GEMM per row range
  (``Int8Linear.matmul_rows``), and every finished range is copied back
  device->host on a third stream while the next range computes. PCIe is full
  duplex, so the two directions overlap each other as well.

Results are bitwise those of ``Int8Linear.forward`` on device tensors.
"""

from __future__ import annotations

import torch

from .linear import Int8Linear
from .sharded import row_ranges


class HostIOPipeline:
    """Run ``[(module, x_host, y_host), ...]`` with overlapped transfers.

    ``x_host`` (M x K fp16) and ``y_host`` (M x N, the module's out dtype)
    should be pinned for the copies to be asynchronous. ``run`` returns once
    everything is enqueued; the host buffers are valid after the caller's
    current stream is synchronised.
    """

    def __init__(self, device=None, chunks: int = 4) -> None:
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.chunks = int(chunks)
        self.h2d = torch.cuda.Stream(device=self.device)
        self.d2h = torch.cuda.Stream(device=self.device)
        # device staging is persistent and double-buffered across runs (no
        # allocator traffic in a serving loop): set s of call i holds (x, y);
        # x_free[s][i] / y_free[s][i] mark when the previous use of the set's
        # buffers (compute reading x, the D2H copy reading y) is done
        self._sets = [[], []]
        self._x_free = [[], []]
        self._y_free = [[], []]
        self._parity = 0

    def _buffers(self, s: int, i: int, xh: torch.Tensor, mod: Int8Linear, yh: torch.Tensor):
        bufs = self._sets[s]
        while len(bufs) <= i:
            bufs.append(None)
            self._x_free[s].append(None)
            self._y_free[s].append(None)
        cur = bufs[i]
        if cur is None or cur[0].shape != xh.shape or cur[1].shape != yh.shape or cur[1].dtype != yh.dtype:
            cur = (torch.empty(xh.shape, dtype=xh.dtype, device=self.device),
                   torch.empty(yh.shape, dtype=yh.dtype, device=self.device))
            cur[0].record_stream(self.h2d)  # freed only after the side streams are done
            cur[1].record_stream(self.d2h)
            bufs[i] = cur
            self._x_free[s][i] = None
            self._y_free[s][i] = None
        return cur

    def run(self, calls: list[tuple[Int8Linear, torch.Tensor, torch.Tensor]],
            inputs_ready: bool = False, join: bool = True) -> None:
        """Enqueue the calls. By default the input copies wait for the caller's
        current stream (it may still be producing the host inputs, e.g. a D2H
        into ``x_host``). ``inputs_ready=True`` asserts the host inputs are
        already final, so this batch's input copies start at once and overlap
        the previous batch's compute and output copies (a serving loop over
        independent batches). ``join=False`` leaves the output copies running
        (the next batch's compute does not wait for them); call ``join()``
        before reading any ``y_host``."""
        compute = torch.cuda.current_stream(self.device)
        if not inputs_ready:
            self.h2d.wait_stream(compute)
        s = self._parity
        self._parity ^= 1
        staged = []
        for i, (mod, xh, yh) in enumerate(calls):
            xd, yd = self._buffers(s, i, xh, mod, yh)
            with torch.cuda.stream(self.h2d):
                if self._x_free[s][i] is not None:  # the compute that read this x is done
                    self.h2d.wait_event(self._x_free[s][i])
                xd.copy_(xh, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.h2d)
            staged.append((xd, yd, ev))
        for i, ((mod, _, yh), (xd, yd, ev)) in enumerate(zip(calls, staged)):
            compute.wait_event(ev)
            if self._y_free[s][i] is not None:  # the D2H copy that read this y is done
                compute.wait_event(self._y_free[s][i])

            def on_rows(r0: int, r1: int, y: torch.Tensor, yh=yh) -> None:
                done = torch.cuda.Event()
                done.record(compute)
                self.d2h.wait_event(done)
                with torch.cuda.stream(self.d2h):
                    yh[r0:r1].copy_(y[r0:r1], non_blocking=True)

            mod.matmul_rows(xd, row_ranges(xd.shape[0], self.chunks), on_rows, y=yd, ldy=yd.stride(0))
            xf = torch.cuda.Event()
            xf.record(compute)
            self._x_free[s][i] = xf
            yf = torch.cuda.Event()
            yf.record(self.d2h)
            self._y_free[s][i] = yf
        if join:
            compute.wait_stream(self.d2h)

    def join(self) -> None:
        """Make the caller's current stream wait for every output copy enqueued so far."""
        torch.cuda.current_stream(self.device).wait_stream(self.d2h)


def run_host_io(calls, chunks: int = 4) -> None:
    """Functional form of ``HostIOPipeline(...).run(calls)``."""
    HostIOPipeline(chunks=chunks).run(calls)
