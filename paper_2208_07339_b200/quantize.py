"""Int8 quantization on B200, mirroring ``int8mm.quantize``: row-wise /
column-wise (vector-wise, quantize.py:168-202) and the tensor-wise absmax and
zeropoint schemes (quantize.py:120-165).

Codes are bit-identical to the reference: scale = 127/amax in float64
(amax 0 -> scale 1) and codes = clip(copysign(floor(|x*scale| + 0.5), x), +-127)
with every float64 operation a single IEEE round-to-nearest op.
"""

from __future__ import annotations

import torch

from ._tensors import as_f16_matrix
from .errors import ShapeMismatchError
from .gemm import _absmax_codes, _quantize_cols_t, _quantize_rows, _zeropoint_codes
from .types import AbsmaxParams, ColwiseParams, QuantizedTensor, RowwiseParams, ZeropointParams

__all__ = ["rowwise_quantize", "colwise_quantize", "vectorwise_params", "absmax_quantize",
           "zeropoint_quantize", "RowwiseParams", "ColwiseParams", "AbsmaxParams",
           "ZeropointParams", "QuantizedTensor"]


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


def absmax_quantize(x) -> QuantizedTensor:
    """Symmetric tensor-wise quantization by 127 over max|x| (quantize.py:137-151).

    An all-zero input uses scale 1 and all-zero codes. Reads max|x| back to the
    host for ``AbsmaxParams`` (one 4-byte copy).
    """
    x16 = as_f16_matrix(x, "x")
    codes, amax = _absmax_codes(x16, transpose=False)
    a = float(amax.item())
    return QuantizedTensor(codes[:, : x16.shape[1]], AbsmaxParams(1.0 if a == 0.0 else 127.0 / a))


def zeropoint_quantize(x) -> QuantizedTensor:
    """Asymmetric quantization spanning [-127, 127] over the input range
    (quantize.py:153-171): nd = 254/(max-min), zp = round(nd*min) + 127, stored
    codes round(nd*x) - zp. A constant tensor keeps its value as ``offset``
    with zero codes; an offset beyond a 16-bit zeropoint raises ValueError.
    """
    x16 = as_f16_matrix(x, "x")
    codes, params = _zeropoint_codes(x16, transpose=False)
    return QuantizedTensor(codes[:, : x16.shape[1]], params)
