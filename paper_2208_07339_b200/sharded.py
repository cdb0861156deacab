"""Output-dimension (N) sharding of the LLM.int8() linear layer across GPUs.

One process per GPU. Rank r holds columns [lo_r, hi_r) of W (the layer's
output features) as a weight-stationary ``Int8Linear`` and computes
Y[:, lo_r:hi_r] with the single-GPU kernels; an NCCL all-gather over NVLink
reassembles Y. Parity survives sharding exactly: the outlier set O and the
row scales depend only on X (gemm.py:210, 242, identical on every rank), and
the column scales are per column (quantize.py:186), so every output element
is computed exactly as on one GPU.
"""

from __future__ import annotations

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


class ShardedInt8Linear(torch.nn.Module):
    """LLM.int8() linear layer with W split along its output dimension.

    ``weight`` is the full K x N weight (each rank keeps only its slice) or,
    with ``local=True``, this rank's K x (hi-lo) slice and ``n_total``.
    """

    def __init__(self, weight, n_total: int | None = None, alpha: float = 6.0,
                 group=None, local: bool = False, out_dtype: torch.dtype = torch.float16,
                 weight_stationary: bool = True):
        super().__init__()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        w = as_f16_matrix(weight, "weight")
        self.n_total = int(n_total if n_total is not None else w.shape[1])
        self.lo, self.hi = shard_bounds(self.n_total, self.world, self.rank)
        if not local:
            w = w[:, self.lo:self.hi].contiguous()
        self.local = Int8Linear(w, alpha, out_dtype=out_dtype, weight_stationary=weight_stationary)

    def forward_local(self, x: torch.Tensor, _timer=None) -> torch.Tensor:
        """This rank's column block Y[:, lo:hi] (no communication)."""
        return self.local(x, _timer=_timer)

    def forward(self, x: torch.Tensor, _timer=None) -> torch.Tensor:
        lead = x.shape[:-1]
        y = self.forward_local(x.reshape(-1, x.shape[-1]), _timer)
        return gather_columns(y, self.n_total, self.group).reshape(*lead, self.n_total)
