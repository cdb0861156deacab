"""ctypes binding of the in-tree sm_100a library (include/llmint8.h).

There is no fallback: if the library is missing, fails to load, or the
device is not a B200 (sm_100), every call raises. Status codes map onto the
reference's exception classes (gemm.py:41-46, tensors.py:21).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import GemmOverflowError, ParamsMismatchError, ShapeMismatchError

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libllmint8_sm100.so"

I8MM_OK = 0
I8MM_ERR_SHAPE = 1
I8MM_ERR_OVERFLOW = 2
I8MM_ERR_ALPHA = 3
I8MM_ERR_PARAMS = 4
I8MM_ERR_ARGUMENT = 5
I8MM_ERR_CUDA = 6
I8MM_ERR_UNSUPPORTED = 7
I8MM_ERR_ZEROPOINT = 8

FLAG_NONFINITE = 1
FLAG_NOT_F16 = 2
FLAG_CODE_128 = 4

DEQ_ABSMAX = 0
DEQ_ZEROPOINT = 1
DEQ_ROWWISE = 2
DEQ_COLWISE = 3

OUT_F16 = 0
OUT_F32 = 1
OUT_F32_EXACT = 2

# Every symbol include/llmint8.h declares (tests check the .so exports them all).
EXPORTED_SYMBOLS = (
    "i8mm_version",
    "i8mm_status_string",
    "i8mm_launch_count",
    "i8mm_debug_set_gemm_variant",
    "i8mm_outlier_scan",
    "i8mm_outlier_compact",
    "i8mm_quantize_rows",
    "i8mm_quantize_cols_t",
    "i8mm_gemm_i32",
    "i8mm_gemm_dequant",
    "i8mm_dequantize_output",
    "i8mm_transpose_i8",
    "i8mm_llm_int8_workspace_size",
    "i8mm_llm_int8_matmul",
    "i8mm_llm_int8_matmul_checked",
    "i8mm_gather_outlier_rows",
    "i8mm_linear_weight_bytes",
    "i8mm_linear_prepare_scratch_bytes",
    "i8mm_linear_prepare",
    "i8mm_linear_workspace_size",
    "i8mm_linear_prologue",
    "i8mm_linear_gemm",
    "i8mm_linear_gemm_rows",
    "i8mm_linear_forward",
    "i8mm_linear_forward_peers",
    "i8mm_linear_workspace_views",
    "i8mm_linear_weight_views",
    "i8mm_linear_workspace_init",
    "i8mm_linear_patch_stats",
    "i8mm_debug_set_decode_max_m",
    "i8mm_debug_set_swapab",
    "i8mm_debug_swapab_timeline",
    "i8mm_debug_set_pdl",
    "i8mm_linear_uses_decode",
    "i8mm_debug_decode_timeline",
    "i8mm_tensor_stats",
    "i8mm_absmax_quantize",
    "i8mm_zeropoint_params",
    "i8mm_zeropoint_quantize",
    "i8mm_rowsum_i8",
    "i8mm_dequantize_absmax",
    "i8mm_zeropoint_combine",
    "i8mm_scalar_workspace_size",
    "i8mm_absmax_matmul",
    "i8mm_zeropoint_matmul",
    "i8mm_f32_scan",
    "i8mm_f32_quantize_rows",
    "i8mm_f32_quantize_cols_t",
    "i8mm_f32_llm_int8_combine",
    "i8mm_f32_workspace_size",
    "i8mm_llm_int8_matmul_f32",
    "i8mm_ordered_matmul_f64",
    "i8mm_round_half_away",
    "i8mm_dequantize_codes",
    "i8mm_check_codes",
    "i8mm_f16_check",
    "i8mm_f16_to_f32",
    "i8mm_zero",
    "i8mm_tensor_stats_f32",
    "i8mm_absmax_quantize_f32",
    "i8mm_zeropoint_quantize_f32",
    "i8mm_peak_mma_launch",
    "i8mm_peak_mma_ops",
)

_lib = None


class NativeLibraryError(RuntimeError):
    """The sm_100a CUDA library is missing or unusable (no CPU fallback exists)."""


def _declare(lib: ctypes.CDLL) -> None:
    P, I64, I32, F32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
    F64 = ctypes.c_double
    SZ = ctypes.c_size_t
    sigs = {
        "i8mm_version": ([], I32),
        "i8mm_status_string": ([I32], ctypes.c_char_p),
        "i8mm_launch_count": ([], ctypes.c_uint64),
        "i8mm_debug_set_gemm_variant": ([I32, I32], None),
        "i8mm_debug_set_decode_max_m": ([I32], None),
        "i8mm_debug_set_swapab": ([I32], None),
        "i8mm_debug_swapab_timeline": ([P], None),
        "i8mm_debug_set_pdl": ([I32], None),
        "i8mm_linear_uses_decode": ([I64, I64, I64], I32),
        "i8mm_debug_decode_timeline": ([P], None),
        "i8mm_outlier_scan": ([P, I64, I64, I64, F32, P, P, P], I32),
        "i8mm_outlier_compact": ([P, I64, P, P, P], I32),
        "i8mm_quantize_rows": ([P, I64, I64, I64, P, P, P, P, I64, P, P, I64, P], I32),
        "i8mm_quantize_cols_t": ([P, I64, I64, I64, P, P, I64, P, P], I32),
        "i8mm_gemm_i32": ([P, I64, P, I64, P, I64, I64, I64, I64, P], I32),
        "i8mm_gemm_dequant": ([P, P, I64, I64, I64, I64, P, P, P, I64, P, I64, P, I64, P, I64, P,
                               P, P, I64, I32, P], I32),
        "i8mm_gather_outlier_rows": ([P, I64, I64, P, P, I64, P, I64, P], I32),
        "i8mm_linear_weight_bytes": ([I64, I64], ctypes.c_size_t),
        "i8mm_linear_prepare_scratch_bytes": ([I64, I64], ctypes.c_size_t),
        "i8mm_linear_prepare": ([P, I64, I64, I64, P, ctypes.c_size_t, P, ctypes.c_size_t, P], I32),
        "i8mm_linear_workspace_size": ([I64, I64, I64], ctypes.c_size_t),
        "i8mm_linear_prologue": ([P, I64, I64, P, I64, P, I64, I64, F32, P, ctypes.c_size_t, P],
                                 I32),
        "i8mm_linear_gemm": ([P, I64, I64, P, I64, P, I64, I64, P, I64, I32, P, ctypes.c_size_t,
                              P], I32),
        "i8mm_linear_gemm_rows": ([P, I64, I64, P, I64, P, I64, I64, P, I64, I32, P,
                                   ctypes.c_size_t, I64, I64, P], I32),
        "i8mm_linear_forward": ([P, I64, I64, P, I64, P, I64, I64, F32, P, I64, I32, P,
                                 ctypes.c_size_t, P, P], I32),
        "i8mm_linear_forward_peers": ([P, I64, I64, P, I64, P, I64, I64, F32, P, I64, P,
                                       ctypes.c_size_t, P, I32, I64, I64, P], I32),
        "i8mm_linear_workspace_views": ([P, I64, I64, I64, P, I32], I32),
        "i8mm_linear_weight_views": ([P, I64, I64, P, I32], I32),
        "i8mm_linear_workspace_init": ([P, ctypes.c_size_t, I64, I64, I64, P], I32),
        "i8mm_linear_patch_stats": ([P, I64, P, I64, I64, I64, P, ctypes.c_size_t, P], I32),
        "i8mm_dequantize_output": ([P, I64, I64, I64, P, P, P, I64, P], I32),
        "i8mm_transpose_i8": ([P, I64, I64, I64, P, I64, P], I32),
        "i8mm_llm_int8_workspace_size": ([I64, I64, I64], ctypes.c_size_t),
        "i8mm_llm_int8_matmul": ([P, I64, P, I64, I64, I64, I64, F32, P, I64, I32, P,
                                  ctypes.c_size_t, P, P], I32),
        "i8mm_llm_int8_matmul_checked": ([P, I64, P, I64, I64, I64, I64, F32, P, I64, I32, P,
                                          ctypes.c_size_t, P, P, P], I32),
        "i8mm_tensor_stats": ([P, I64, I64, I64, P, P, P], I32),
        "i8mm_absmax_quantize": ([P, I64, I64, I64, P, P, I64, I32, P], I32),
        "i8mm_zeropoint_params": ([F32, F32, P, P, P], I32),
        "i8mm_zeropoint_quantize": ([P, I64, I64, I64, F64, I32, P, I64, I32, P], I32),
        "i8mm_rowsum_i8": ([P, I64, I64, I64, P, P], I32),
        "i8mm_dequantize_absmax": ([P, I64, I64, I64, P, P, P, I64, P], I32),
        "i8mm_zeropoint_combine": ([P, I64, I64, I64, P, P, I64, I32, I32, F64, F64, F64, F64, P,
                                    I64, P, P, P], I32),
        "i8mm_scalar_workspace_size": ([I64, I64, I64], SZ),
        "i8mm_absmax_matmul": ([P, I64, P, I64, I64, I64, I64, P, I64, P, SZ, P], I32),
        "i8mm_zeropoint_matmul": ([P, I64, P, I64, I64, I64, I64, P, I64, P, SZ, P], I32),
        "i8mm_f32_scan": ([P, I64, I64, I64, F32, P, P, P, I64, P], I32),
        "i8mm_f32_quantize_rows": ([P, I64, I64, I64, P, P, I64, P, P], I32),
        "i8mm_f32_quantize_cols_t": ([P, I64, I64, I64, P, P, I64, P, P], I32),
        "i8mm_f32_llm_int8_combine": ([P, I64, I64, I64, I64, P, P, P, I64, P, I64, P, P, P, I64, P],
                                      I32),
        "i8mm_f32_workspace_size": ([I64, I64, I64], SZ),
        "i8mm_llm_int8_matmul_f32": ([P, I64, P, I64, I64, I64, I64, F32, P, I64, P, SZ, P, P], I32),
        "i8mm_ordered_matmul_f64": ([P, I64, P, I64, I64, I64, I64, I32, P, I64, P], I32),
        "i8mm_round_half_away": ([P, I64, I32, P, P], I32),
        "i8mm_dequantize_codes": ([P, I64, I64, I64, I32, P, P, F64, I32, F64, F64, P, I64, P], I32),
        "i8mm_check_codes": ([P, I64, I64, I64, P, P], I32),
        "i8mm_f16_check": ([P, I64, I64, I64, P, P], I32),
        "i8mm_f16_to_f32": ([P, I64, I64, I64, P, I64, P], I32),
        "i8mm_zero": ([P, SZ, P], I32),
        "i8mm_tensor_stats_f32": ([P, I64, I64, I64, P, P, P], I32),
        "i8mm_absmax_quantize_f32": ([P, I64, I64, I64, P, P, I64, I32, P], I32),
        "i8mm_zeropoint_quantize_f32": ([P, I64, I64, I64, F64, I32, P, I64, I32, P], I32),
        "i8mm_peak_mma_launch": ([I32, I32, P], I32),
        "i8mm_peak_mma_ops": ([I32, I32], F64),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def load_library(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and return the sm_100a library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if path is None and os.environ.get("I8MM_LIB_ALT"):  # dev A/B against another build
        path = os.environ["I8MM_LIB_ALT"]
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise NativeLibraryError(
            f"{p} is missing: build it with `python -m paper_2208_07339_b200.build` "
            "(there is no CPU fallback for the LLM.int8() path)")
    try:
        lib = ctypes.CDLL(str(p))
    except OSError as e:  # pragma: no cover - depends on the host
        raise NativeLibraryError(f"cannot load {p}: {e}") from e
    _declare(lib)
    _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    return load_library()


def check(status: int, what: str = "") -> None:
    """Raise the reference's exception class for a non-zero status."""
    if status == I8MM_OK:
        return
    msg = lib().i8mm_status_string(status).decode()
    if what:
        msg = f"{what}: {msg}"
    if status == I8MM_ERR_SHAPE:
        raise ShapeMismatchError(msg)
    if status == I8MM_ERR_OVERFLOW:
        raise GemmOverflowError(msg)
    if status == I8MM_ERR_PARAMS:
        raise ParamsMismatchError(msg)
    if status == I8MM_ERR_ALPHA:
        raise ValueError(msg)
    if status == I8MM_ERR_UNSUPPORTED:
        raise NativeLibraryError(msg)
    if status in (I8MM_ERR_ARGUMENT, I8MM_ERR_ZEROPOINT):
        raise ValueError(msg)
    raise RuntimeError(msg)


def launch_count() -> int:
    return int(lib().i8mm_launch_count())
