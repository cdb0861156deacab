"""B200-native (sm_100a) LLM.int8() linear layer (arXiv 2208.07339).

Drop-in for the reference package ``int8mm``'s operator API on the
LLM.int8() path: quantize (row-/column-wise), the outlier-decomposed int8
matmul, and the Int8 linear module / backend plugin. Hot ops are hand-written
CUDA kernels for sm_100a (tcgen05 + TMA + TMEM) behind the C ABI in
``include/llmint8.h``; PyTorch provides device memory and streams only.
"""

from .errors import GemmOverflowError, ParamsMismatchError, ShapeMismatchError
from .gemm import (MAX_INNER_DIM, MatmulResult, absmax_matmul, dequantize_output,
                   extract_outlier_columns, int8_gemm_i32, llm_int8_matmul, ordered_matmul_f64,
                   vectorwise_matmul, zeropoint_gemm_i32, zeropoint_matmul)
from .linear import (ABSMAX, BACKEND_KINDS, EXACT, VECTORWISE, ZEROPOINT, Int8Linear,
                     LinearBackend, _linear, linear, llm_int8_backend)
from .quantize import (absmax_quantize, colwise_quantize, dequantize, round_half_away,
                       rowwise_quantize, vectorwise_params, zeropoint_quantize)
from .graphs import GraphedCall
from .pipeline import HostIOPipeline, run_host_io
from .synthetic import planted_pair
from .tensors import DenseMatrix, Int8Matrix, Int32Matrix, seeded_random_matrix
from .types import (AbsmaxParams, ColwiseParams, OutlierSet, QuantizedTensor, QuantParams,
                    RowwiseParams, ZeropointParams)
from . import int8mm  # the reference-typed API (import swap)

__version__ = "0.1.0"

__all__ = [
    "MAX_INNER_DIM", "GemmOverflowError", "ParamsMismatchError", "ShapeMismatchError",
    "MatmulResult", "OutlierSet", "QuantizedTensor", "RowwiseParams", "ColwiseParams",
    "extract_outlier_columns", "int8_gemm_i32", "dequantize_output", "llm_int8_matmul",
    "vectorwise_matmul", "rowwise_quantize", "colwise_quantize", "vectorwise_params",
    "BACKEND_KINDS", "LinearBackend", "EXACT", "ABSMAX", "ZEROPOINT", "VECTORWISE",
    "llm_int8_backend", "linear", "_linear", "Int8Linear", "planted_pair",
    "AbsmaxParams", "ZeropointParams", "absmax_quantize", "zeropoint_quantize",
    "absmax_matmul", "zeropoint_matmul", "zeropoint_gemm_i32", "HostIOPipeline", "run_host_io",
    "GraphedCall", "ordered_matmul_f64", "round_half_away", "dequantize", "QuantParams",
    "DenseMatrix", "Int8Matrix", "Int32Matrix", "seeded_random_matrix", "int8mm",
]
