"""Output-dimension (N) sharding of the LLM.int8() linear layer across GPUs.

One process per GPU. Rank r holds columns [lo_r, hi_r) of W (the layer's
output features) as a weight-stationary ``Int8Linear`` and computes
Y[:, lo_r:hi_r] with the single-GPU kernels; an NCCL all-gather over NVLink
reassembles Y. Parity survives sharding exactly: the outlier set O and the
row scales depend only on X (gemm.py:210, 242, identical on every rank), and
the column scales are per column (quantize.py:186), so every output element
is computed exactly as on one GPU.

The all-gather is pipelined behind the GEMM: after one
prologue over all rows, the GEMM runs per row range and each range's block is
gathered on a communication stream while the next range computes, so the
NVLink transfer overlaps the tensor-core work except for the last range.

The default (``fused_gather=None``) removes the collective altogether when the
process group supports symmetric memory: Y lives in symmetric memory and the
GEMM epilogue stores each output tile into every rank's Y over NVLink
(``forward_fused``); otherwise the NCCL pipeline runs. Validated on one GPU
(world size 1 through symmetric memory, and peers emulated by extra buffers in
``i8mm_linear_forward_peers``); no multi-GPU box was available to this round.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict

import torch
import torch.distributed as dist

from ._tensors import as_f16_matrix
from .linear import Int8Linear


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced column range of ``rank`` (first n % world ranks get one more)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} for world size {world}")
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def gather_columns(y_local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather the per-rank column blocks Y[:, lo_r:hi_r] into Y (M x n_total).

    One ``all_gather_into_tensor`` over equal-size (padded) blocks, then the
    blocks are placed. Works with NCCL (GPU) and gloo (CPU).
    """
    world = dist.get_world_size(group)
    m, n_loc = y_local.shape
    width = -(-n_total // world)
    if n_loc != width:
        pad = torch.zeros((m, width), dtype=y_local.dtype, device=y_local.device)
        pad[:, :n_loc] = y_local
        y_local = pad
    flat = torch.empty((world * m, width), dtype=y_local.dtype, device=y_local.device)
    if dist.get_backend(group) == "gloo":
        parts = list(flat.view(world, m, width).unbind(0))
        dist.all_gather(parts, y_local.contiguous(), group=group)
    else:
        dist.all_gather_into_tensor(flat, y_local.contiguous(), group=group)
    blocks = flat.view(world, m, width)
    out = torch.empty((m, n_total), dtype=y_local.dtype, device=y_local.device)
    for r in range(world):
        lo, hi = shard_bounds(n_total, world, r)
        out[:, lo:hi] = blocks[r, :, : hi - lo]
    return out


def row_ranges(m: int, chunks: int) -> list[tuple[int, int]]:
    """Balanced contiguous row ranges; multiples of 256 (a CTA-pair tile) when possible."""
    chunks = max(1, min(int(chunks), -(-m // 256)))
    step = -(-m // chunks)
    step = -(-step // 256) * 256 if m >= 256 * chunks else step
    out, r = [], 0
    while r < m:
        out.append((r, min(m, r + step)))
        r += step
    return out


class _GatherPipeline:
    """Gathers row ranges of the padded per-rank blocks as they are produced.

    ``push(r0, r1, y_pad)`` (called right after range r0:r1 is enqueued on the
    compute stream) all-gathers those rows on the communication stream and
    places every rank's block into ``out``; ``finish()`` joins the streams.
    """

    def __init__(self, m: int, n_total: int, width: int, dtype, device, group):
        self.group = group
        self.world = dist.get_world_size(group)
        self.n_total, self.width = n_total, width
        self.out = torch.empty((m, n_total), dtype=dtype, device=device)
        self.cuda = device.type == "cuda"
        self.comm = torch.cuda.Stream(device=device) if self.cuda else None
        self.gloo = dist.get_backend(group) == "gloo"

    def push(self, r0: int, r1: int, y_pad: torch.Tensor) -> None:
        rows = r1 - r0
        src = y_pad[r0:r1]
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record()
            self.comm.wait_event(ev)
            ctx = torch.cuda.stream(self.comm)
        else:
            import contextlib

            ctx = contextlib.nullcontext()
        with ctx:
            buf = torch.empty((self.world, rows, self.width), dtype=src.dtype, device=src.device)
            if self.gloo:
                dist.all_gather(list(buf.unbind(0)), src.contiguous(), group=self.group)
            else:
                dist.all_gather_into_tensor(buf, src, group=self.group)
            for r in range(self.world):
                lo, hi = shard_bounds(self.n_total, self.world, r)
                self.out[r0:r1, lo:hi].copy_(buf[r, :, : hi - lo])
        if self.cuda:
            src.record_stream(self.comm)
            buf.record_stream(self.comm)

    def finish(self) -> torch.Tensor:
        if self.cuda:
            torch.cuda.current_stream().wait_stream(self.comm)
            self.out.record_stream(torch.cuda.current_stream())
        return self.out


class ShardedInt8Linear(torch.nn.Module):
    """LLM.int8() linear layer with W split along its output dimension.

    ``weight`` is the full K x N weight (each rank keeps only its slice) or,
    with ``local=True``, this rank's K x (hi-lo) slice and ``n_total``.
    """

    def __init__(self, weight, n_total: int | None = None, alpha: float = 6.0,
                 group=None, local: bool = False, out_dtype: torch.dtype = torch.float16,
                 weight_stationary: bool = True, fused_gather: bool | None = None,
                 check_finite: bool = True):
        super().__init__()
        # forward() -> forward_fused (symmetric memory) when True; None = use it
        # when the process group supports symmetric memory, else the NCCL pipeline
        self.fused_gather = fused_gather
        self.gather_path = None  # "fused-epilogue" | "nccl-pipelined", set by forward()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        w = as_f16_matrix(weight, "weight")
        self.n_total = int(n_total if n_total is not None else w.shape[1])
        self.lo, self.hi = shard_bounds(self.n_total, self.world, self.rank)
        if not local:
            w = w[:, self.lo:self.hi].contiguous()
        self.local = Int8Linear(w, alpha, out_dtype=out_dtype, weight_stationary=weight_stationary,
                                check_finite=check_finite)
        # forward_fused: (M, device) -> symmetric Y buffer and peer handles, LRU-bounded
        self._symm: "OrderedDict[tuple, tuple]" = OrderedDict()
        self.symm_cache_size = 4
        self._fused_ok: bool | None = None  # agreed by all ranks on first use

    def forward_local(self, x: torch.Tensor, _timer=None) -> torch.Tensor:
        """This rank's column block Y[:, lo:hi] (no communication)."""
        return self.local(x, _timer=_timer)

    def fused_supported(self, x2: torch.Tensor) -> bool:
        """Whether the fused peer-store gather can run, decided ONCE and agreed
        by every rank (an all-reduce MIN of each rank's probe), so no rank
        takes a different path than its peers (which would hang the job)."""
        if self._fused_ok is None:
            ok = int(self.local.out_dtype == torch.float16 and self.local.weight_stationary
                     and x2.is_cuda and dist.get_backend(self.group) == "nccl")
            if ok:
                try:  # probe: symmetric memory allocation + rendezvous on a tiny buffer
                    import torch.distributed._symmetric_memory as symm_mem

                    group = self.group if self.group is not None else dist.group.WORLD
                    t = symm_mem.empty((8,), dtype=torch.float16, device=x2.device)
                    symm_mem.rendezvous(t, group.group_name)
                except (ImportError, NotImplementedError, AttributeError, RuntimeError):
                    ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device=x2.device if x2.is_cuda else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
            self._fused_ok = bool(flag.item())
        return self._fused_ok

    def forward(self, x: torch.Tensor, _timer=None, chunks: int | None = None,
                out: torch.Tensor | None = None, alias: bool = False) -> torch.Tensor:
        """Y = x @ W over all ranks. ``chunks`` row ranges pipeline the NCCL
        all-gather behind the GEMM (default 4 when world > 1, else 1).

        With the fused gather, Y is assembled in a symmetric-memory buffer that
        the next call with the same M overwrites: by default it is copied into
        ``out`` (or a fresh tensor); ``alias=True`` returns the buffer itself
        (valid until the next call -- for callers that consume Y at once)."""
        lead = x.shape[:-1]
        x2 = x.reshape(-1, x.shape[-1])
        want_fused = self.fused_gather is not False and _timer is None and chunks is None
        if want_fused and self.fused_supported(x2):
            y = self.forward_fused(x2)
            self.gather_path = "fused-epilogue"
            if not alias:
                y = y.clone() if out is None else out.view(-1, self.n_total).copy_(y)
            return y.reshape(*lead, self.n_total)
        if self.fused_gather:
            raise ValueError("fused_gather needs CUDA tensors, NCCL with symmetric memory, fp16 "
                             "output and a weight-stationary layer")
        self.gather_path = "nccl-pipelined"
        if chunks is None:
            chunks = 4 if self.world > 1 else 1
        if chunks <= 1 or _timer is not None:
            y = self.forward_local(x2, _timer)
            y = gather_columns(y, self.n_total, self.group)
        else:
            y = self.forward_pipelined(x2, chunks)
        if out is not None:
            y = out.view(-1, self.n_total).copy_(y)
        return y.reshape(*lead, self.n_total)

    def forward_fused(self, x2: torch.Tensor) -> torch.Tensor:
        """Y = x @ W with the all-gather fused into the GEMM epilogue.

        Y lives in symmetric memory (``torch.distributed._symmetric_memory``):
        every rank's epilogue stores its column block into its own Y and, over
        NVLink, into every peer's Y (``i8mm_linear_forward_peers``); one
        device-side barrier then orders the peers' stores before the reads. No
        NCCL collective runs. The returned tensor is a persistent buffer per
        row count (at most ``symm_cache_size`` row counts are kept, least
        recently used evicted), overwritten by the next call with the same M.
        """
        import torch.distributed._symmetric_memory as symm_mem

        from . import _native as nat
        from ._tensors import stream_handle

        if self.local.out_dtype != torch.float16 or not self.local.weight_stationary:
            raise ValueError("forward_fused needs fp16 output and a weight-stationary layer")
        x16 = as_f16_matrix(x2, "x")
        m, k = x16.shape
        key = (m, x16.device.index)
        if key in self._symm:
            self._symm.move_to_end(key)
        else:
            while len(self._symm) >= self.symm_cache_size:
                self._symm.popitem(last=False)  # the buffer is freed with its last reference
            out = symm_mem.empty((m, self.n_total), dtype=torch.float16, device=x16.device)
            group = self.group if self.group is not None else dist.group.WORLD
            hdl = symm_mem.rendezvous(out, group.group_name)
            peers = [hdl.get_buffer(r, out.shape, out.dtype) for r in range(self.world) if r != self.rank]
            ptrs = (ctypes.c_void_p * max(1, len(peers)))(*[t.data_ptr() for t in peers])
            self._symm[key] = (out, hdl, peers, ptrs)
        out, hdl, peers, ptrs = self._symm[key]
        # every rank is done with the previous contents of its Y (work enqueued
        # before this call) before any peer overwrites them
        hdl.barrier(channel=1)
        L = nat.lib()
        lin = self.local
        n = self.hi - self.lo
        ws = lin.workspace(m)
        y_loc = out[:, self.lo:self.hi]  # this rank's block, written in place (ldy = n_total)
        nat.check(L.i8mm_linear_forward_peers(
            x16.data_ptr(), x16.stride(0), m, lin.weight.data_ptr(), lin.weight.stride(0),
            lin.wbuf.data_ptr(), k, n, lin.alpha, y_loc.data_ptr(), self.n_total, ws.data_ptr(),
            ws.numel(), ptrs, len(peers), self.n_total, self.lo, stream_handle()), "linear_forward_peers")
        hdl.barrier()
        return out

    def forward_pipelined(self, x2: torch.Tensor, chunks: int) -> torch.Tensor:
        m = x2.shape[0]
        width = -(-self.n_total // self.world)
        dt = self.local.out_dtype
        y_pad = torch.zeros((m, width), dtype=dt, device=x2.device)
        pipe = _GatherPipeline(m, self.n_total, width, dt, x2.device, self.group)
        self.local.matmul_rows(as_f16_matrix(x2, "x"), row_ranges(m, chunks), pipe.push,
                               y=y_pad, ldy=width)
        return pipe.finish()
