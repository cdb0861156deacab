"""The reference package's API with the reference's own types (import swap).

    import paper_2208_07339_b200.int8mm as int8mm   # instead of: import int8mm

Every LLM.int8()-path name of ``int8mm/__init__.py`` (pkg/src/int8mm/
__init__.py:11-76) with the same signature, the same return types
(``DenseMatrix`` / ``Int8Matrix`` / ``Int32Matrix`` containers whose ``.data`` is
a read-only host numpy array, ``QuantizedTensor``, ``MatmulResult`` with plain
ints, ``OutlierSet``) and the same exceptions, so code and tests written
against the reference run unchanged. The arithmetic is the B200 kernels of
this package (fp16 production kernels when the operands' values are all
exactly fp16, otherwise the float32 kernels); results are bit-identical to the
reference's: float32 outputs come from the exact epilogues.

The top-level ``paper_2208_07339_b200`` namespace is the device-native form of
the same operators (CUDA tensors in and out, no host round trips).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import gemm as _g
from . import quantize as _q
from .errors import GemmOverflowError, ParamsMismatchError, ShapeMismatchError
from .gemm import MAX_INNER_DIM
from .linear import (ABSMAX, BACKEND_KINDS, EXACT, VECTORWISE, ZEROPOINT, LinearBackend,
                     llm_int8_backend)
from .synthetic import planted_pair
from .tensors import (DenseMatrix, Int8Matrix, Int32Matrix, _wrap_dense, _wrap_int8,
                      seeded_random_matrix)
from .types import (AbsmaxParams, ColwiseParams, OutlierSet, QuantizedTensor, QuantParams,
                    RowwiseParams, ZeropointParams)

__all__ = [
    "MAX_INNER_DIM", "GemmOverflowError", "ParamsMismatchError", "ShapeMismatchError",
    "MatmulResult", "absmax_matmul", "dequantize_output", "extract_outlier_columns",
    "int8_gemm_i32", "llm_int8_matmul", "ordered_matmul_f64", "vectorwise_matmul",
    "zeropoint_gemm_i32", "zeropoint_matmul", "AbsmaxParams", "ColwiseParams",
    "QuantizedTensor", "QuantParams", "RowwiseParams", "ZeropointParams", "absmax_quantize",
    "colwise_quantize", "dequantize", "rowwise_quantize", "round_half_away",
    "vectorwise_params", "zeropoint_quantize", "DenseMatrix", "Int8Matrix", "Int32Matrix",
    "seeded_random_matrix", "OutlierSet", "LinearBackend", "BACKEND_KINDS", "EXACT", "ABSMAX",
    "ZEROPOINT", "VECTORWISE", "llm_int8_backend", "planted_pair",
]


@dataclass(frozen=True, eq=False)
class MatmulResult:
    """gemm.py:49-60: output DenseMatrix, scheme, decomposed_cols, int8_fraction."""

    output: DenseMatrix
    scheme: str
    decomposed_cols: int = 0
    int8_fraction: float = 1.0


def _dense(x) -> DenseMatrix:
    return x if isinstance(x, DenseMatrix) else DenseMatrix(x)


def _int8(a) -> Int8Matrix:
    return a if isinstance(a, Int8Matrix) else Int8Matrix(a)


def _result(r, scheme: str) -> MatmulResult:
    n = r.decomposed_cols
    return MatmulResult(_wrap_dense(r.output), scheme, n, r.int8_fraction)


# ---------------------------------------------------------------- gemm.py
def int8_gemm_i32(a: Int8Matrix, b: Int8Matrix) -> Int32Matrix:
    """gemm.py:78-82"""
    return Int32Matrix._wrap(_g.int8_gemm_i32(_int8(a), _int8(b), validate=False))


def zeropoint_gemm_i32(a: Int8Matrix, b: Int8Matrix, zp_a: int, zp_b: int,
                       unrolled: bool = False) -> Int32Matrix:
    """gemm.py:85-104"""
    return Int32Matrix._wrap(_g.zeropoint_gemm_i32(_int8(a), _int8(b), zp_a, zp_b, unrolled))


def ordered_matmul_f64(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """gemm.py:110-117 (host arrays in and out; computed on the GPU)."""
    return _g.ordered_matmul_f64(x, w).cpu().numpy()


def dequantize_output(c: Int32Matrix, params_x: QuantParams, params_w: QuantParams) -> DenseMatrix:
    """gemm.py:120-147"""
    return _wrap_dense(_g.dequantize_output(c, params_x, params_w))


def absmax_matmul(x: DenseMatrix, w: DenseMatrix) -> MatmulResult:
    """gemm.py:150-156"""
    return _result(_g.absmax_matmul(_dense(x), _dense(w), validate=False), "absmax")


def zeropoint_matmul(x: DenseMatrix, w: DenseMatrix, unrolled: bool = False) -> MatmulResult:
    """gemm.py:159-187"""
    return _result(_g.zeropoint_matmul(_dense(x), _dense(w), unrolled, validate=False),
                   "zeropoint")


def vectorwise_matmul(x: DenseMatrix, w: DenseMatrix) -> MatmulResult:
    """gemm.py:197-200 (float32 output bit-identical: exact epilogue)."""
    return _result(_g.vectorwise_matmul(_dense(x), _dense(w), exact=True, validate=False),
                   "vectorwise")


def extract_outlier_columns(x: DenseMatrix, alpha: float = 6.0) -> OutlierSet:
    """gemm.py:203-211"""
    if not (alpha > 0) or not np.isfinite(alpha):
        raise ValueError(f"alpha must be positive and finite, got {alpha}")
    return _g.extract_outlier_columns(_dense(x), alpha, validate=False)


def llm_int8_matmul(x: DenseMatrix, w: DenseMatrix, alpha: float = 6.0) -> MatmulResult:
    """gemm.py:214-247 (float32 output bit-identical: exact epilogue)."""
    xd, wd = _dense(x), _dense(w)
    r = _g.llm_int8_matmul(xd, wd, alpha, exact=True, validate=False)
    n = r.decomposed_cols
    return MatmulResult(_wrap_dense(r.output), "llm_int8", n, 1.0 - n / xd.cols if n else 1.0)


# ---------------------------------------------------------------- quantize.py
def round_half_away(x: np.ndarray) -> np.ndarray:
    """quantize.py:26-29 (host array in and out; computed on the GPU)."""
    arr = np.asarray(x, dtype=np.float64)
    return _q.round_half_away(arr).cpu().numpy().reshape(arr.shape)


def _qt(q) -> QuantizedTensor:
    codes = q.codes
    if isinstance(codes, torch.Tensor):
        codes = _wrap_int8(codes if codes.is_contiguous() else codes.contiguous())
    params = q.params
    if isinstance(params, (RowwiseParams, ColwiseParams)):  # plain host scales, like the reference
        params = type(params)(params.scales)
    return QuantizedTensor(codes, params)


def absmax_quantize(x: DenseMatrix) -> QuantizedTensor:
    """quantize.py:137-151"""
    return _qt(_q.absmax_quantize(_dense(x), validate=False))


def zeropoint_quantize(x: DenseMatrix) -> QuantizedTensor:
    """quantize.py:153-171"""
    return _qt(_q.zeropoint_quantize(_dense(x), validate=False))


def rowwise_quantize(x: DenseMatrix) -> QuantizedTensor:
    """quantize.py:174-179"""
    return _qt(_q.rowwise_quantize(_dense(x), validate=False))


def colwise_quantize(w: DenseMatrix) -> QuantizedTensor:
    """quantize.py:182-187"""
    return _qt(_q.colwise_quantize(_dense(w), validate=False))


def vectorwise_params(x: DenseMatrix, w: DenseMatrix) -> tuple[QuantizedTensor, QuantizedTensor]:
    """quantize.py:190-202"""
    if x.cols != w.rows:
        raise ShapeMismatchError(
            f"inner dimensions differ: X is {x.rows}x{x.cols}, W is {w.rows}x{w.cols}")
    return rowwise_quantize(x), colwise_quantize(w)


def dequantize(q: QuantizedTensor) -> DenseMatrix:
    """quantize.py:205-227"""
    return _wrap_dense(_q.dequantize(q))
