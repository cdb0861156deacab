"""Result / parameter types of the operator API, mirroring the reference.

* ``OutlierSet``      -- outliers.py:27-50
* ``RowwiseParams``   -- quantize.py:74-81 (scales = 127/amax per row, f64)
* ``ColwiseParams``   -- quantize.py:84-91 (scales = 127/amax per column, f64)
* ``AbsmaxParams``    -- quantize.py:32-41 (tensor-wise scale)
* ``ZeropointParams`` -- quantize.py:44-61 (nd, zp, offset)
* ``QuantizedTensor`` -- quantize.py:97-112
* ``MatmulResult``    -- gemm.py:49-60

Device results stay on the GPU. Host values of the reference result
(``decomposed_cols``, ``int8_fraction``, ``OutlierSet.dims``) are materialised
lazily from device counters, so a call never synchronises unless the caller
reads them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class OutlierSet:
    """Sorted, duplicate-free feature indices plus the threshold (outliers.py:27-50)."""

    dims: tuple[int, ...]
    alpha: float

    def __post_init__(self) -> None:
        dims = tuple(int(d) for d in self.dims)
        if any(d < 0 for d in dims):
            raise ValueError("feature indices must be non-negative")
        if len(set(dims)) != len(dims):
            raise ValueError("feature indices must be unique")
        object.__setattr__(self, "dims", tuple(sorted(dims)))
        if not (self.alpha > 0) or not np.isfinite(self.alpha):
            raise ValueError(f"alpha must be positive and finite, got {self.alpha}")

    def __len__(self) -> int:
        return len(self.dims)

    def __contains__(self, dim: int) -> bool:
        return dim in self.dims


def _scales_from_amax(amax: torch.Tensor) -> np.ndarray:
    """quantize.py:168-171: amax == 0 -> 127 -> scale 1; 127/amax in float64.

    Computed on the host with numpy's IEEE true_divide, exactly as the
    reference (torch's CUDA ``scalar / tensor`` is a reciprocal-multiply and is
    not correctly rounded). The device kernels carry amax, never the scale.
    """
    a = amax.detach().cpu().numpy().astype(np.float64)  # D2H copy, widened on the host
    a[a == 0.0] = 127.0
    return 127.0 / a


class _VectorParams:
    __slots__ = ("amax", "_scales")
    _what = "scales"

    def __init__(self, scales=None, *, amax: torch.Tensor | None = None) -> None:
        if (amax is None) == (scales is None):
            raise ValueError("give exactly one of amax or scales")
        if amax is not None:
            self.amax = amax
            self._scales = None
        else:
            s = np.array(scales, dtype=np.float64, copy=True)
            if s.ndim != 1 or s.size < 1:
                raise ValueError(f"{self._what} must be a non-empty vector")
            if not np.isfinite(s).all() or (s <= 0).any():
                raise ValueError(f"{self._what} must all be positive and finite")
            s.setflags(write=False)
            self.amax = None
            self._scales = s

    @property
    def scales(self) -> np.ndarray:
        """float64 scales 127/amax (quantize.py:171) as a host numpy array."""
        if self._scales is None:
            self._scales = _scales_from_amax(self.amax)
        return self._scales

    @property
    def size(self) -> int:
        return int(self.amax.numel() if self.amax is not None else self._scales.size)


class RowwiseParams(_VectorParams):
    """One absmax scale per row (quantize.py:74-81). ``RowwiseParams(scales)``
    as in the reference, or ``RowwiseParams(amax=device_tensor)`` from a kernel."""

    __slots__ = ()
    _what = "row scales"


class ColwiseParams(_VectorParams):
    """One absmax scale per column (quantize.py:84-91)."""

    __slots__ = ()
    _what = "column scales"


ZP_INT16_MIN = -(1 << 15)  # quantize.py:22-23
ZP_INT16_MAX = (1 << 15) - 1


@dataclass(frozen=True)
class AbsmaxParams:
    """Tensor-wise symmetric scale: codes = round(scale * x), scale = 127 / max|x|
    (quantize.py:32-41)."""

    scale: float

    def __post_init__(self) -> None:
        if not np.isfinite(self.scale) or self.scale <= 0:
            raise ValueError(f"scale must be positive and finite, got {self.scale}")


@dataclass(frozen=True)
class ZeropointParams:
    """Affine scale/shift: stored code = round(nd * x) - zp, zp a 16-bit integer;
    ``offset`` carries a constant tensor's value (quantize.py:44-61)."""

    nd: float
    zp: int
    offset: float = 0.0

    def __post_init__(self) -> None:
        if not np.isfinite(self.nd) or self.nd <= 0:
            raise ValueError(f"nd must be positive and finite, got {self.nd}")
        if not (ZP_INT16_MIN <= self.zp <= ZP_INT16_MAX):
            raise ValueError(f"zeropoint {self.zp} outside the signed 16-bit range")
        if not np.isfinite(self.offset):
            raise ValueError("offset must be finite")


QuantParams = AbsmaxParams | ZeropointParams | RowwiseParams | ColwiseParams  # quantize.py:94


@dataclass(frozen=True, eq=False)
class QuantizedTensor:
    """Int8 codes with the constants that dequantize them (quantize.py:97-112)."""

    codes: torch.Tensor
    params: RowwiseParams | ColwiseParams | AbsmaxParams | ZeropointParams

    def __post_init__(self) -> None:
        if isinstance(self.params, RowwiseParams) and self.params.size != self.codes.shape[0]:
            raise ValueError("row scale count must equal the number of rows")
        if isinstance(self.params, ColwiseParams) and self.params.size != self.codes.shape[1]:
            raise ValueError("column scale count must equal the number of columns")

    @property
    def source_shape(self) -> tuple[int, int]:
        return tuple(self.codes.shape)


class MatmulResult:
    """Output of a quantized matmul pipeline (gemm.py:49-60).

    ``decomposed_cols`` / ``int8_fraction`` are read from the device counter on
    first access (one 4-byte D2H copy).
    """

    __slots__ = ("output", "scheme", "_count", "_h", "_decomposed")

    def __init__(self, output: torch.Tensor, scheme: str, count: torch.Tensor | int | None,
                 h: int) -> None:
        self.output = output
        self.scheme = scheme
        self._count = count
        self._h = h
        self._decomposed: int | None = None

    @property
    def decomposed_cols(self) -> int:
        if self._decomposed is None:
            c = self._count
            if c is None:
                self._decomposed = 0
            elif isinstance(c, torch.Tensor):
                self._decomposed = int(c.reshape(-1)[0].item())
            else:
                self._decomposed = int(c)
        return self._decomposed

    @property
    def int8_fraction(self) -> float:
        n = self.decomposed_cols
        return 1.0 - n / self._h if n else 1.0

    def __repr__(self) -> str:
        return f"MatmulResult(scheme={self.scheme!r}, output={tuple(self.output.shape)})"
