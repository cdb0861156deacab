"""Device-backed matrix containers mirroring ``int8mm.tensors``.

``DenseMatrix`` / ``Int8Matrix`` / ``Int32Matrix`` keep the reference's
constructor contract (pkg/src/int8mm/tensors.py:31-170): rank-2, non-empty,
copied on construction, immutable, the same ValueError messages, bitwise
equality. The values live in HBM; the validation a constructor performs
(NaN/Inf for DenseMatrix, the int8 code range) runs on the GPU, and
``.data`` materialises a read-only host numpy copy on first access (the
reference's attribute), so code written against the reference keeps working.

``DenseMatrix`` also records whether its float32 values are all exactly fp16
values; the operators then run the fp16 production kernels on an fp16 copy
(bit-identical results) and otherwise the float32 kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from ._tensors import (_check_rank2, _device_f32, as_i8_matrix, device, raise_for_flags, scan_f32)
from .errors import ShapeMismatchError

INT8_CODE_MIN = -127
INT8_CODE_MAX = 127

__all__ = ["DenseMatrix", "Int8Matrix", "Int32Matrix", "ShapeMismatchError",
           "seeded_random_matrix", "INT8_CODE_MIN", "INT8_CODE_MAX"]


def _frozen_host(t: torch.Tensor) -> np.ndarray:
    a = t.detach().cpu().numpy().copy()
    a.setflags(write=False)
    return a


class _DeviceMatrix:
    __slots__ = ("_t", "_host")

    @property
    def tensor(self) -> torch.Tensor:
        """The device tensor (do not mutate: containers are immutable)."""
        return self._t

    @property
    def data(self) -> np.ndarray:
        """Read-only host copy (tensors.py: ``.data``)."""
        if self._host is None:
            self._host = _frozen_host(self._t)
        return self._host

    @property
    def rows(self) -> int:
        return int(self._t.shape[0])

    @property
    def cols(self) -> int:
        return int(self._t.shape[1])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)

    def __eq__(self, other) -> bool:
        if type(other) is not type(self):
            return NotImplemented
        return np.array_equal(self.data, other.data)

    __hash__ = None  # type: ignore[assignment]

    def __repr__(self) -> str:
        return f"{type(self).__name__}({self.rows}x{self.cols})"


class DenseMatrix(_DeviceMatrix):
    """Row-major matrix of finite 32-bit floats (tensors.py:31-76)."""

    __slots__ = ("_t16",)

    def __init__(self, data) -> None:
        if isinstance(data, DenseMatrix):
            self._t, self._t16, self._host = data._t, data._t16, data._host
            return
        t = _device_f32(data, "data")
        if isinstance(data, torch.Tensor) and t.data_ptr() == data.data_ptr():
            t = t.clone()  # the constructor copies its input (tensors.py:25-28)
        if not t.is_contiguous():
            t = t.contiguous()
        flags, t16 = scan_f32(t)
        raise_for_flags(flags & nat.FLAG_NONFINITE)
        self._t = t
        self._t16 = t16
        self._host = None

    @property
    def tensor16(self) -> torch.Tensor | None:
        """fp16 copy when every value is exactly an fp16 value, else None."""
        return self._t16

    def to_f16_precision(self) -> "DenseMatrix":
        """Round every entry to the nearest 16-bit float (tensors.py:64-66);
        values beyond the fp16 range become Inf and are rejected, as in the
        reference."""
        if self._t16 is not None:
            return self
        rows, cols = self._t.shape
        y16 = torch.empty((rows, cols), dtype=torch.float16, device=self._t.device)
        from ._tensors import new_flags, stream_handle

        flags = new_flags(1)
        nat.check(nat.lib().i8mm_f32_scan(self._t.data_ptr(), rows, cols, cols, 0.0, None,
                                          flags.data_ptr(), y16.data_ptr(), cols, stream_handle()))
        return DenseMatrix(y16)


class Int8Matrix(_DeviceMatrix):
    """Row-major int8 codes restricted to [-127, 127] (tensors.py:79-122)."""

    __slots__ = ()

    def __init__(self, data) -> None:
        if isinstance(data, Int8Matrix):
            self._t, self._host = data._t, data._host
            return
        if isinstance(data, torch.Tensor) and data.dtype != torch.int8:
            if data.dtype.is_floating_point:
                raise ValueError(f"Int8Matrix requires integer data, got dtype {data.dtype}")
            data = data.detach().cpu().numpy()
        t = as_i8_matrix(data, "data", validate=True)
        if isinstance(data, torch.Tensor) and t.data_ptr() == data.data_ptr():
            t = t.clone()
        self._t = t.contiguous()
        self._host = None


class Int32Matrix(_DeviceMatrix):
    """Row-major int32 accumulator values (tensors.py:125-170)."""

    __slots__ = ()

    def __init__(self, data) -> None:
        if isinstance(data, Int32Matrix):
            self._t, self._host = data._t, data._host
            return
        if isinstance(data, torch.Tensor) and data.dtype == torch.int32:
            _check_rank2(data.shape, "data", "Int32Matrix")
            t = data.detach().to(device())
            self._t = t.clone() if t.data_ptr() == data.data_ptr() else t.contiguous()
            self._host = None
            return
        arr = np.asarray(data.detach().cpu().numpy() if isinstance(data, torch.Tensor) else data)
        if arr.dtype.kind not in "iu":
            raise ValueError(f"Int32Matrix requires integer data, got dtype {arr.dtype}")
        _check_rank2(arr.shape, "data", "Int32Matrix")
        info = np.iinfo(np.int32)
        if arr.size and (arr.min() < info.min or arr.max() > info.max):
            raise ValueError("Int32Matrix values exceed the signed 32-bit range")
        self._t = torch.from_numpy(np.ascontiguousarray(arr.astype(np.int32))).to(device())
        self._host = None

    @classmethod
    def _wrap(cls, t: torch.Tensor) -> "Int32Matrix":
        obj = cls.__new__(cls)
        obj._t = t
        obj._host = None
        return obj


def _wrap_dense(t: torch.Tensor) -> DenseMatrix:
    """Container around a float32 result tensor the library produced (finite by
    construction of the operators; no re-scan)."""
    obj = DenseMatrix.__new__(DenseMatrix)
    obj._t = t
    obj._t16 = None
    obj._host = None
    return obj


def _wrap_int8(t: torch.Tensor) -> Int8Matrix:
    obj = Int8Matrix.__new__(Int8Matrix)
    obj._t = t
    obj._host = None
    return obj


def seeded_random_matrix(rows: int, cols: int, seed: int, stddev: float = 1.0) -> DenseMatrix:
    """Gaussian matrix, a pure function of its arguments (tensors.py:221-236):
    PCG64 seeded with ``seed``, numpy's float32 ziggurat, scaled by
    float32(stddev). Input generation, not part of the operator path."""
    if rows < 1 or cols < 1:
        raise ValueError(f"matrix dimensions must be >= 1, got {rows}x{cols}")
    if not (seed >= 0):
        raise ValueError("seed must be a non-negative integer")
    if not np.isfinite(stddev) or stddev <= 0:
        raise ValueError(f"stddev must be positive and finite, got {stddev}")
    rng = np.random.Generator(np.random.PCG64(seed))
    vals = rng.standard_normal((rows, cols), dtype=np.float32) * np.float32(stddev)
    return DenseMatrix(vals)
