"""Row-wise / column-wise (vector-wise) int8 quantization on B200, mirroring
``int8mm.quantize`` (pkg/src/int8mm/quantize.py:168-202).

Codes are bit-identical to the reference: scale = 127/amax in float64
(amax 0 -> scale 1) and codes = clip(copysign(floor(|x*scale| + 0.5), x), +-127)
with every float64 operation a single IEEE round-to-nearest op.
"""

from __future__ import annotations

import torch

from ._tensors import as_f16_matrix
from .errors import ShapeMismatchError
from .gemm import _quantize_cols_t, _quantize_rows
from .types import ColwiseParams, QuantizedTensor, RowwiseParams

__all__ = ["rowwise_quantize", "colwise_quantize", "vectorwise_params", "RowwiseParams",
           "ColwiseParams", "QuantizedTensor"]


def rowwise_quantize(x) -> QuantizedTensor:
    """Absmax quantization applied independently to each row (quantize.py:174-179)."""
    x16 = as_f16_matrix(x, "x")
    xq, _, amax, _ = _quantize_rows(x16, None)
    return QuantizedTensor(xq[:, : x16.shape[1]], RowwiseParams(amax=amax))


def colwise_quantize(w) -> QuantizedTensor:
    """Absmax quantization applied independently to each column (quantize.py:182-187).

    The codes are returned in the reference orientation (K x N) as a transposed
    view of the K-major buffer the tensor-core GEMM consumes.
    """
    w16 = as_f16_matrix(w, "w")
    wq_t, _, amax = _quantize_cols_t(w16, None)
    codes: torch.Tensor = wq_t[:, : w16.shape[0]].t()
    return QuantizedTensor(codes, ColwiseParams(amax=amax))


def vectorwise_params(x, w) -> tuple[QuantizedTensor, QuantizedTensor]:
    """Quantize an (X, W) pair with per-row / per-column constants (quantize.py:190-202)."""
    xs = x.shape if hasattr(x, "shape") else None
    ws = w.shape if hasattr(w, "shape") else None
    if xs is not None and ws is not None and xs[1] != ws[0]:
        raise ShapeMismatchError(
            f"inner dimensions differ: X is {xs[0]}x{xs[1]}, W is {ws[0]}x{ws[1]}")
    return rowwise_quantize(x), colwise_quantize(w)
