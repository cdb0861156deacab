"""Input coercion, validation flags and small device-buffer helpers.

Operand types (the reference's DenseMatrix holds float32, tensors.py:31-49):

* an fp16 CUDA tensor (or numpy float16) is used as is -- the production
  kernels' native type;
* anything else (float32/float64 tensors or arrays, lists, ``DenseMatrix``) is
  brought to the device as float32 and scanned once on the GPU
  (``i8mm_f32_scan``): NaN/Inf raise ``ValueError`` like the reference's
  DenseMatrix (tensors.py:47-48); when every value is exactly an fp16 value the
  scan's fp16 copy runs the fp16 kernels (bit-identical results), otherwise the
  operators run the float32 kernels (csrc/f32path.cu), exact for any finite f32.

No value is ever rounded silently, and no operator computes on the CPU.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .errors import ShapeMismatchError


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise nat.NativeLibraryError("the LLM.int8() path needs a CUDA device (B200, sm_100a)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def round_up(v: int, a: int) -> int:
    return (v + a - 1) // a * a


def zero_(t: torch.Tensor) -> torch.Tensor:
    """Stream-ordered memset of a device tensor (no PyTorch kernel launch)."""
    nat.check(nat.lib().i8mm_zero(t.data_ptr(), t.numel() * t.element_size(), stream_handle()),
              "zero")
    return t


def new_flags(n: int = 1) -> torch.Tensor:
    return zero_(torch.empty((max(n, 1),), dtype=torch.int32, device=device()))


def raise_for_flags(flags: int, what: str = "") -> None:
    """The reference's container errors for device-detected conditions."""
    if flags & nat.FLAG_NONFINITE:
        raise ValueError("DenseMatrix rejects NaN/Inf entries")
    if flags & nat.FLAG_CODE_128:
        raise ValueError(f"Int8Matrix values must lie in [-127, 127]{' (' + what + ')' if what else ''}")


def _check_rank2(shape, name: str, what: str = "DenseMatrix") -> None:
    if len(shape) != 2:
        raise ValueError(f"{what} requires a rank-2 array, got rank {len(shape)} ({name})")
    if shape[0] < 1 or shape[1] < 1:
        raise ValueError(f"{what} dimensions must be >= 1, got {tuple(shape)} ({name})")


def _rowmajor(t: torch.Tensor) -> torch.Tensor:
    """Row-strided with unit column stride (what the kernels take), else a copy."""
    if t.stride(1) == 1 and t.stride(0) >= t.shape[1]:
        return t
    return t.contiguous()


def scan_f32(t32: torch.Tensor, want16: bool = True):
    """One GPU pass over a float32 matrix: (flags, fp16 copy or None). Syncs
    once to read the 4-byte flag word."""
    rows, cols = t32.shape
    flags = new_flags(1)
    y16 = torch.empty((rows, cols), dtype=torch.float16, device=t32.device) if want16 else None
    nat.check(nat.lib().i8mm_f32_scan(t32.data_ptr(), rows, cols, t32.stride(0), 0.0, None,
                                      flags.data_ptr(), y16.data_ptr() if y16 is not None else None,
                                      cols, stream_handle()), "f32_scan")
    f = int(flags.item())
    return f, (y16 if (want16 and not (f & (nat.FLAG_NOT_F16 | nat.FLAG_NONFINITE))) else None)


def f16_to_f32(t16: torch.Tensor) -> torch.Tensor:
    rows, cols = t16.shape
    out = torch.empty((rows, cols), dtype=torch.float32, device=t16.device)
    nat.check(nat.lib().i8mm_f16_to_f32(t16.data_ptr(), rows, cols, t16.stride(0), out.data_ptr(),
                                        cols, stream_handle()), "f16_to_f32")
    return out


def _device_f32(a, name: str) -> torch.Tensor:
    """float32 CUDA matrix from any non-fp16 input (numpy/list/torch)."""
    dev = device()
    if isinstance(a, torch.Tensor):
        _check_rank2(a.shape, name)
        t = a.detach()
        if t.dtype != torch.float32:
            if t.is_cuda:
                t = t.float()  # rare: float64 / integer CUDA inputs
            else:
                t = torch.from_numpy(np.asarray(t.numpy(), dtype=np.float32))
        return _rowmajor(t.to(dev, non_blocking=True))
    arr = np.asarray(a, dtype=np.float32)  # tensors.py:42 (the reference's own coercion)
    _check_rank2(arr.shape, name)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev)


def as_operand(a, name: str, validate: bool = True) -> torch.Tensor:
    """A 2-D operand on the device: fp16 when its values are exactly fp16
    (including every fp16 input), else float32. float32 inputs are scanned on
    the GPU (one 4-byte sync); NaN/Inf raise ValueError when ``validate``."""
    from .tensors import DenseMatrix

    if isinstance(a, DenseMatrix):
        return a.tensor16 if a.tensor16 is not None else a.tensor
    if isinstance(a, torch.Tensor) and a.dtype == torch.float16:
        _check_rank2(a.shape, name)
        return _rowmajor(a.to(device(), non_blocking=True))
    if isinstance(a, np.ndarray) and a.dtype == np.float16:
        _check_rank2(a.shape, name)
        return torch.from_numpy(np.ascontiguousarray(a)).to(device())
    if hasattr(a, "data") and isinstance(getattr(a, "data"), np.ndarray):  # foreign DenseMatrix-like
        a = a.data
    t32 = _device_f32(a, name)
    flags, t16 = scan_f32(t32)
    if validate and flags & nat.FLAG_NONFINITE:
        raise_for_flags(flags)
    return t16 if t16 is not None else t32


def as_f16_matrix(a, name: str) -> torch.Tensor:
    """An operand that must be fp16 (module weights, the benchmark's inputs).

    float32 inputs are accepted only when every value is exactly an fp16
    value (checked on the GPU); otherwise ValueError -- never a silent rounding.
    """
    t = as_operand(a, name, validate=True)
    if t.dtype != torch.float16:
        raise ValueError(
            f"{name} holds values that are not exactly representable in fp16; this path "
            "computes on fp16 operands (round them explicitly, e.g. DenseMatrix.to_f16_precision(), "
            "or use the float32 operators llm_int8_matmul / linear)")
    return t


def common_dtype(a: torch.Tensor, b: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Both fp16, or both float32 (an fp16 operand is widened exactly)."""
    if a.dtype == b.dtype:
        return a, b
    return (f16_to_f32(a) if a.dtype == torch.float16 else a,
            f16_to_f32(b) if b.dtype == torch.float16 else b)


def as_i8_matrix(a, name: str, validate: bool = True) -> torch.Tensor:
    """int8 codes on the device; code -128 (and values outside [-127, 127] in
    wider integer inputs) raise ValueError like Int8Matrix (tensors.py:89-98)."""
    from .tensors import Int8Matrix

    if isinstance(a, Int8Matrix):
        return a.tensor
    if isinstance(a, torch.Tensor):
        t = a
    else:
        arr = np.asarray(getattr(a, "data", a) if not isinstance(a, (list, tuple)) else a)
        if arr.dtype.kind not in "iu":
            raise ValueError(f"Int8Matrix requires integer data, got dtype {arr.dtype}")
        _check_rank2(arr.shape, name, "Int8Matrix")
        if arr.dtype != np.int8:
            if arr.size and (arr.min() < -127 or arr.max() > 127):
                raise ValueError("Int8Matrix values must lie in [-127, 127]")
            arr = arr.astype(np.int8)
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.ndim != 2:
        raise ValueError(f"{name} must be rank-2, got rank {t.ndim}")
    if t.dtype != torch.int8:
        raise ValueError(f"{name} must hold int8 codes, got {t.dtype}")
    t = t.to(device(), non_blocking=True)
    if validate:
        check_codes(t, name)
    return t


def check_codes(t: torch.Tensor, name: str) -> None:
    """Device range check of int8 codes (one 4-byte sync)."""
    if t.stride(1) != 1:
        t = t.contiguous()
    flags = new_flags(1)
    nat.check(nat.lib().i8mm_check_codes(t.data_ptr(), t.shape[0], t.shape[1], t.stride(0),
                                         flags.data_ptr(), stream_handle()), "check_codes")
    raise_for_flags(int(flags.item()), name)


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
    buf = zero_(torch.empty((rows, ld), dtype=torch.int8, device=t.device))
    buf[:, :k].copy_(t)
    return buf, ld
