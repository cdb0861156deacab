"""Synthetic inputs of the reference's accuracy sweeps and benchmark.

``planted_pair`` restates the reference generator (sweep.py:60-77, used by
bench.py:134): Gaussian X with ``outlier_cols`` seeded columns scaled by
``outlier_scale``, Gaussian W, PCG64 streams -- bit-identical values on the
host (numpy). ``planted_pair_device`` draws the same distribution directly
in HBM with a seeded ``torch.Generator`` for shapes too large to generate on
the host; its outlier columns are returned so callers can
check the detected set.
"""

from __future__ import annotations

import numpy as np
import torch


def planted_pair(rows: int, inner: int, cols: int, outlier_cols: int, outlier_scale: float,
                 seed: int) -> tuple[np.ndarray, np.ndarray]:
    """float32 (X, W) exactly as the reference's planted_pair (sweep.py:60-77)."""
    if outlier_cols > inner:
        raise ValueError(f"cannot plant {outlier_cols} outlier columns in {inner}")
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((rows, inner), dtype=np.float32)
    if outlier_cols:
        idx = rng.choice(inner, size=outlier_cols, replace=False)
        x[:, idx] *= np.float32(outlier_scale)
    w = rng.standard_normal((inner, cols), dtype=np.float32)
    return x, w


def planted_pair_device(rows: int, inner: int, cols: int, outlier_cols: int,
                        outlier_scale: float, seed: int, device=None,
                        dtype: torch.dtype = torch.float16):
    """Same distribution as ``planted_pair`` generated on the GPU.

    Returns (x, w, planted_columns) with x rows x inner, w inner x cols.
    """
    dev = torch.device(device) if device is not None else torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    x = torch.randn((rows, inner), generator=g, device=dev, dtype=torch.float32)
    idx = torch.randperm(inner, generator=g, device=dev)[:outlier_cols]
    if outlier_cols:
        x[:, idx] *= float(outlier_scale)
    x = x.to(dtype)
    w = torch.randn((inner, cols), generator=g, device=dev, dtype=torch.float32).to(dtype)
    return x, w, torch.sort(idx).values
