"""Int8 quantization on B200, mirroring ``int8mm.quantize``: row-wise /
column-wise (vector-wise, quantize.py:168-202), the tensor-wise absmax and
zeropoint schemes (quantize.py:120-165), ``dequantize`` (quantize.py:205-227)
and ``round_half_away`` (quantize.py:26-29).

Codes are bit-identical to the reference: scale = 127/amax in float64
(amax 0 -> scale 1) and codes = clip(copysign(floor(|x*scale| + 0.5), x), +-127)
with every float64 operation a single IEEE round-to-nearest op. fp16 and
float32 operands are both exact (``_tensors.as_operand``).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from ._tensors import as_operand, device, stream_handle
from .errors import ShapeMismatchError
from .gemm import _absmax_codes, _quantize_cols_t, _quantize_rows, _zeropoint_codes
from .types import (AbsmaxParams, ColwiseParams, QuantizedTensor, QuantParams, RowwiseParams,
                    ZeropointParams)

__all__ = ["rowwise_quantize", "colwise_quantize", "vectorwise_params", "absmax_quantize",
           "zeropoint_quantize", "dequantize", "round_half_away", "RowwiseParams",
           "ColwiseParams", "AbsmaxParams", "ZeropointParams", "QuantizedTensor", "QuantParams"]


def round_half_away(x) -> torch.Tensor:
    """Round to the nearest integer with ties away from zero, in float64
    (quantize.py:26-29). float32/float64 input (tensor or array); returns a
    float64 CUDA tensor of the same shape."""
    dev = device()
    if isinstance(x, torch.Tensor):
        t = x.detach().to(dev)
        if t.dtype not in (torch.float32, torch.float64):
            t = t.double()
    else:
        arr = np.asarray(x)
        arr = arr if arr.dtype in (np.float32, np.float64) else arr.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
    t = t.contiguous()
    out = torch.empty(t.shape, dtype=torch.float64, device=dev)
    nat.check(nat.lib().i8mm_round_half_away(t.data_ptr(), t.numel(), t.element_size(),
                                             out.data_ptr(), stream_handle()), "round_half_away")
    return out


def rowwise_quantize(x, validate: bool = True) -> QuantizedTensor:
    """Absmax quantization applied independently to each row (quantize.py:174-179)."""
    xt = as_operand(x, "x", validate)
    xq, _, amax, _ = _quantize_rows(xt, None)
    return QuantizedTensor(xq[:, : xt.shape[1]], RowwiseParams(amax=amax))


def colwise_quantize(w, validate: bool = True) -> QuantizedTensor:
    """Absmax quantization applied independently to each column (quantize.py:182-187).

    The codes are returned in the reference orientation (K x N) as a transposed
    view of the K-major buffer the tensor-core GEMM consumes.
    """
    wt = as_operand(w, "w", validate)
    wq_t, _, amax = _quantize_cols_t(wt, None)
    codes: torch.Tensor = wq_t[:, : wt.shape[0]].t()
    return QuantizedTensor(codes, ColwiseParams(amax=amax))


def vectorwise_params(x, w) -> tuple[QuantizedTensor, QuantizedTensor]:
    """Quantize an (X, W) pair with per-row / per-column constants (quantize.py:190-202)."""
    xs = tuple(x.shape) if hasattr(x, "shape") else np.shape(x)
    ws = tuple(w.shape) if hasattr(w, "shape") else np.shape(w)
    if len(xs) == 2 and len(ws) == 2 and xs[1] != ws[0]:
        raise ShapeMismatchError(
            f"inner dimensions differ: X is {xs[0]}x{xs[1]}, W is {ws[0]}x{ws[1]}")
    return rowwise_quantize(x), colwise_quantize(w)


def absmax_quantize(x, validate: bool = True) -> QuantizedTensor:
    """Symmetric tensor-wise quantization by 127 over max|x| (quantize.py:137-151).

    An all-zero input uses scale 1 and all-zero codes. Reads max|x| back to the
    host for ``AbsmaxParams`` (one 4-byte copy).
    """
    xt = as_operand(x, "x", validate)
    codes, amax = _absmax_codes(xt, transpose=False)
    a = float(amax.item())
    return QuantizedTensor(codes[:, : xt.shape[1]], AbsmaxParams(1.0 if a == 0.0 else 127.0 / a))


def zeropoint_quantize(x, validate: bool = True) -> QuantizedTensor:
    """Asymmetric quantization spanning [-127, 127] over the input range
    (quantize.py:153-171): nd = 254/(max-min), zp = round(nd*min) + 127, stored
    codes round(nd*x) - zp. A constant tensor keeps its value as ``offset``
    with zero codes; an offset beyond a 16-bit zeropoint raises ValueError.
    """
    xt = as_operand(x, "x", validate)
    codes, params = _zeropoint_codes(xt, transpose=False)
    return QuantizedTensor(codes[:, : xt.shape[1]], params)


def dequantize(q: QuantizedTensor) -> torch.Tensor:
    """Invert a quantization up to the scheme's rounding error (quantize.py:205-227):
    float32(codes / scale) per params kind, in float64 on the device."""
    from ._tensors import as_i8_matrix

    codes = as_i8_matrix(q.codes, "codes", validate=False)
    if codes.stride(1) != 1:  # colwise codes are a transposed view
        codes = codes.contiguous()
    rows, cols = codes.shape
    dev = codes.device
    p = q.params
    sr = sc = None
    scale, zp, nd, off = 1.0, 0, 1.0, 0.0
    if isinstance(p, AbsmaxParams):
        mode, scale = nat.DEQ_ABSMAX, float(p.scale)
    elif isinstance(p, ZeropointParams):
        mode, zp, nd, off = nat.DEQ_ZEROPOINT, int(p.zp), float(p.nd), float(p.offset)
    elif isinstance(p, RowwiseParams):
        mode = nat.DEQ_ROWWISE
        sr = torch.from_numpy(np.array(p.scales, dtype=np.float64)).to(dev)
    elif isinstance(p, ColwiseParams):
        mode = nat.DEQ_COLWISE
        sc = torch.from_numpy(np.array(p.scales, dtype=np.float64)).to(dev)
    else:
        raise TypeError(f"unknown params type {type(p)!r}")
    out = torch.empty((rows, cols), dtype=torch.float32, device=dev)
    nat.check(nat.lib().i8mm_dequantize_codes(
        codes.data_ptr(), rows, cols, codes.stride(0), mode,
        sr.data_ptr() if sr is not None else None, sc.data_ptr() if sc is not None else None,
        scale, zp, nd, off, out.data_ptr(), cols, stream_handle()), "dequantize")
    return out
