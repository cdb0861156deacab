"""Input coercion and small device-buffer helpers shared by the operators."""

from __future__ import annotations

import numpy as np
import torch

from .errors import ShapeMismatchError


def device() -> torch.device:
    if not torch.cuda.is_available():
        from ._native import NativeLibraryError

        raise NativeLibraryError("the LLM.int8() path needs a CUDA device (B200, sm_100a)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def as_f16_matrix(a, name: str) -> torch.Tensor:
    """Coerce a 2-D float input (numpy / torch, any device) to contiguous fp16 CUDA.

    The reference stores 16-bit operands in float32 containers
    (tensors.py:31-36); the GPU path consumes them as fp16, which is exact for
    fp16-representable values.
    """
    if isinstance(a, np.ndarray):
        if a.ndim != 2:
            raise ValueError(f"{name} must be rank-2, got rank {a.ndim}")
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float16))
    elif isinstance(a, torch.Tensor):
        t = a
    elif hasattr(a, "data") and isinstance(getattr(a, "data"), np.ndarray):  # DenseMatrix-like
        return as_f16_matrix(a.data, name)
    else:
        t = torch.as_tensor(np.asarray(a, dtype=np.float16))
    if t.ndim != 2:
        raise ValueError(f"{name} must be rank-2, got rank {t.ndim}")
    if t.shape[0] < 1 or t.shape[1] < 1:
        raise ValueError(f"{name} dimensions must be >= 1, got {tuple(t.shape)}")
    dev = device()
    if t.device != dev or t.dtype != torch.float16:
        t = t.to(device=dev, dtype=torch.float16, non_blocking=True)
    return t.contiguous()


def as_i8_matrix(a, name: str) -> torch.Tensor:
    if isinstance(a, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int8))
    elif isinstance(a, torch.Tensor):
        t = a
    elif hasattr(a, "data") and isinstance(getattr(a, "data"), np.ndarray):
        return as_i8_matrix(a.data, name)
    else:
        t = torch.as_tensor(np.asarray(a, dtype=np.int8))
    if t.ndim != 2:
        raise ValueError(f"{name} must be rank-2, got rank {t.ndim}")
    if t.dtype != torch.int8:
        raise ValueError(f"{name} must hold int8 codes, got {t.dtype}")
    dev = device()
    if t.device != dev:
        t = t.to(device=dev, non_blocking=True)
    return t


def round_up(v: int, a: int) -> int:
    return (v + a - 1) // a * a


def check_inner(x_cols: int, w_rows: int, shapes: str) -> None:
    """gemm.py:63-69 -- shape check then the int32 overflow guard."""
    from .errors import GemmOverflowError
    from .gemm import MAX_INNER_DIM

    if x_cols != w_rows:
        raise ShapeMismatchError(f"inner dimensions differ: {shapes}")
    if x_cols > MAX_INNER_DIM:
        raise GemmOverflowError(
            f"inner dimension {x_cols} exceeds the int32 overflow guard {MAX_INNER_DIM}")


def kmajor_i8(t: torch.Tensor) -> tuple[torch.Tensor, int]:
    """Return (buffer, ld) such that buffer rows are K-major with ld % 16 == 0.

    ``t`` is rows x K; a view whose row pitch is already a multiple of 16 and
    whose K axis is contiguous is used as is (no copy).
    """
    rows, k = t.shape
    if t.stride(1) == 1 and t.stride(0) % 16 == 0 and t.stride(0) >= k and t.data_ptr() % 16 == 0:
        return t, t.stride(0)
    ld = round_up(max(k, 1), 16)
    buf = torch.zeros((rows, ld), dtype=torch.int8, device=t.device)
    buf[:, :k].copy_(t)
    return buf, ld
