"""CPU oracle for the LLM.int8() matmul path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it. The product path
(``paper_2208_07339_b200``) never imports anything under ``oracle/`` and
fails loudly when its CUDA library is missing.

Two restatements of the reference algorithm live here:

* a pure-numpy restatement (this file), each function citing the reference
  line it follows (``pkg/src/int8mm/...`` under the reference tree);
* a plain-C restatement (``oracle/llmint8_oracle.c``, built by
  ``oracle/Makefile`` into ``oracle/liboracle_llmint8.so``), loaded here via
  ctypes. It is multi-threaded (OpenMP) and is the CPU baseline timed by
  ``bench.py``.

Parity is PINNED: both restatements are checked against golden vectors
produced by the reference package itself (``tests/golden/make_golden.py``
imports ``int8mm`` from the reference tree and writes
``tests/golden/*.npz``), see ``tests/test_oracle_golden.py``.

numpy behaviours the reference relies on and that are
restated explicitly here:
  1. ``np.abs(f32) >= alpha`` compares in float32 (alpha cast to f32).
  2. every float64 op is one IEEE round-to-nearest op (no FMA contraction).
  3. ``int64 @ int64`` is exact.

The exact integer GEMM here uses float64 BLAS instead of numpy's (slow,
non-BLAS) int64 matmul: all operands are integers with |a|,|b| <= 127 and
K <= 2**17, so every product and every partial sum is an integer of
magnitude <= 127*127*2**17 < 2**31 < 2**53 and each float64 operation is
exact, whatever the summation order. The result is therefore identical to
the reference's int64 product (gemm.py:81).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

MAX_INNER_DIM = 1 << 17  # gemm.py:35
_HERE = Path(__file__).resolve().parent


# --------------------------------------------------------------------------
# numpy restatement
# --------------------------------------------------------------------------

def round_half_away(x: np.ndarray) -> np.ndarray:
    """quantize.py:26-29 -- copysign(floor(|x| + 0.5), x) in float64."""
    x = np.asarray(x, dtype=np.float64)
    return np.copysign(np.floor(np.abs(x) + 0.5), x)


def outlier_mask(x: np.ndarray, alpha: float) -> np.ndarray:
    """gemm.py:208-210 -- column mask any_i |x_ik| >= f32(alpha)."""
    if not (alpha > 0) or not np.isfinite(alpha):
        raise ValueError(f"alpha must be positive and finite, got {alpha}")
    x = np.asarray(x, dtype=np.float32)
    return (np.abs(x) >= np.float32(alpha)).any(axis=0)


def outlier_dims(x: np.ndarray, alpha: float) -> tuple[int, ...]:
    """gemm.py:211 -- sorted outlier column indices."""
    return tuple(int(i) for i in np.flatnonzero(outlier_mask(x, alpha)))


def axis_absmax_scales(data64: np.ndarray, axis: int) -> np.ndarray:
    """quantize.py:168-171 -- 127/amax per slice, amax==0 -> scale 1."""
    amax = np.abs(data64).max(axis=axis)
    amax[amax == 0.0] = 127.0
    return 127.0 / amax


def to_codes(scaled: np.ndarray) -> np.ndarray:
    """quantize.py:115-117 -- round half away, clip to [-127, 127]."""
    return np.clip(round_half_away(scaled), -127, 127).astype(np.int8)


def rowwise_quantize(x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """quantize.py:174-179 -> (codes int8 MxK, scales f64 [M])."""
    data = np.asarray(x, dtype=np.float32).astype(np.float64)
    scales = axis_absmax_scales(data, axis=1)
    return to_codes(data * scales[:, None]), scales


def colwise_quantize(w: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """quantize.py:182-187 -> (codes int8 KxN, scales f64 [N])."""
    data = np.asarray(w, dtype=np.float32).astype(np.float64)
    scales = axis_absmax_scales(data, axis=0)
    return to_codes(data * scales[None, :]), scales


def int8_gemm_i32(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """gemm.py:78-82 -- exact int8 x int8 -> int32 (see module docstring)."""
    if a.shape[1] != b.shape[0]:
        raise ValueError("inner dimensions differ")
    if a.shape[1] > MAX_INNER_DIM:
        raise ValueError("inner dimension exceeds the int32 overflow guard")
    acc = a.astype(np.float64) @ b.astype(np.float64)
    return acc.astype(np.int32)


def dequantize_output(c: np.ndarray, sx: np.ndarray, sw: np.ndarray) -> np.ndarray:
    """gemm.py:130,141,147 -- f32( f64(C) / outer(sx, sw) )."""
    return (c.astype(np.float64) / np.multiply.outer(sx, sw)).astype(np.float32)


def ordered_matmul_f64(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """gemm.py:110-117 -- f64 outer-product accumulation, ascending k."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    acc = np.zeros((x.shape[0], w.shape[1]))
    for k in range(x.shape[1]):
        acc += np.multiply.outer(x[:, k], w[k, :])
    return acc


@dataclass
class LlmInt8Trace:
    """Every intermediate of gemm.py:214-247, in the GPU's full-K layout.

    ``xq``/``wq`` are full width with zeros at outlier columns/rows (the
    reference's compacted ``x_rest``/``w_rest`` codes are ``xq[:, keep]`` and
    ``wq[keep, :]``). ``sx``/``sw`` are the f64 scales 127/amax.
    """

    dims: tuple[int, ...]
    xq: np.ndarray
    sx: np.ndarray
    wq: np.ndarray
    sw: np.ndarray
    c: np.ndarray
    hi: np.ndarray | None
    output: np.ndarray
    decomposed_cols: int
    int8_fraction: float


def llm_int8_matmul(x: np.ndarray, w: np.ndarray, alpha: float = 6.0) -> LlmInt8Trace:
    """gemm.py:214-247 restated, returning every intermediate."""
    x = np.asarray(x, dtype=np.float32)
    w = np.asarray(w, dtype=np.float32)
    m, h = x.shape
    if h != w.shape[0]:
        raise ValueError("inner dimensions differ")
    mask = outlier_mask(x, alpha)  # gemm.py:225
    dims = tuple(int(i) for i in np.flatnonzero(mask))
    n_out = len(dims)
    keep = ~mask  # gemm.py:233-236
    xq = np.zeros((m, h), dtype=np.int8)
    wq = np.zeros((h, w.shape[1]), dtype=np.int8)
    sx = np.ones(m)
    sw = np.ones(w.shape[1])
    c = np.zeros((m, w.shape[1]), dtype=np.int32)
    hi = None
    if n_out:
        hi = ordered_matmul_f64(x[:, mask], w[mask, :])  # gemm.py:238
    if keep.any():
        qx, sx = rowwise_quantize(x[:, keep])  # gemm.py:242 -> 190-191
        qw, sw = colwise_quantize(w[keep, :])  # gemm.py:243 -> 192
        xq[:, keep] = qx
        wq[keep, :] = qw
        c = int8_gemm_i32(qx, qw)  # gemm.py:193
        lo = dequantize_output(c, sx, sw)  # gemm.py:194
        out = lo if hi is None else (lo.astype(np.float64) + hi).astype(np.float32)  # gemm.py:244
    else:
        out = hi.astype(np.float32)  # gemm.py:239-240
    return LlmInt8Trace(dims, xq, sx, wq, sw, c, hi, out, n_out, 1.0 - n_out / h)


def vectorwise_matmul(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """gemm.py:190-200 -- no decomposition."""
    qx, sx = rowwise_quantize(x)
    qw, sw = colwise_quantize(w)
    return dequantize_output(int8_gemm_i32(qx, qw), sx, sw)


# ---- sibling schemes (tensor-wise), quantize.py:120-171, gemm.py:85-104, 150-187

ZP_INT16_MIN, ZP_INT16_MAX = -(1 << 15), (1 << 15) - 1  # quantize.py:22-23


def absmax_quantize(x: np.ndarray) -> tuple[np.ndarray, float]:
    """quantize.py:137-151 -- codes, scale (all-zero input: zero codes, scale 1)."""
    data = np.asarray(x, dtype=np.float64)
    amax = float(np.abs(data).max())
    if amax == 0.0:
        return np.zeros(data.shape, dtype=np.int8), 1.0
    scale = 127.0 / amax
    return to_codes(scale * data), scale


def zeropoint_quantize(x: np.ndarray) -> tuple[np.ndarray, float, int, float]:
    """quantize.py:153-171 -- codes, nd, zp, offset; ValueError outside int16."""
    data = np.asarray(x, dtype=np.float64)
    lo, hi = float(data.min()), float(data.max())
    if hi == lo:
        return np.zeros(data.shape, dtype=np.int8), 1.0, 0, lo
    nd = 254.0 / (hi - lo)
    zp = int(round_half_away(np.float64(nd * lo))) + 127
    if not (ZP_INT16_MIN <= zp <= ZP_INT16_MAX):
        raise ValueError(f"input offset too extreme for a 16-bit zeropoint (zp={zp})")
    stored = round_half_away(nd * data) - zp
    return np.clip(stored, -127, 127).astype(np.int8), nd, zp, 0.0


def zeropoint_gemm_i32(a: np.ndarray, b: np.ndarray, zp_a: int, zp_b: int) -> np.ndarray:
    """gemm.py:85-104 -- (A + zp_a)(B + zp_b) exactly; OverflowError outside int32
    (gemm.py:71-75). The int64 matmul is done as exact float64 BLAS on the
    codes (see module docstring) plus the integer unrolled terms."""
    a64 = a.astype(np.int64)
    b64 = b.astype(np.int64)
    acc = (int8_gemm_i32(a, b).astype(np.int64) + zp_b * a64.sum(axis=1, keepdims=True)
           + zp_a * b64.sum(axis=0, keepdims=True) + a.shape[1] * zp_a * zp_b)
    if acc.min(initial=0) < np.iinfo(np.int32).min or acc.max(initial=0) > np.iinfo(np.int32).max:
        raise OverflowError("accumulated values exceed the signed 32-bit range")
    return acc.astype(np.int32)


def absmax_matmul(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """gemm.py:150-156 -- f32( f64(C) / (s_x * s_w) )."""
    qx, sx = absmax_quantize(x)
    qw, sw = absmax_quantize(w)
    return (int8_gemm_i32(qx, qw).astype(np.float64) / (sx * sw)).astype(np.float32)


def zeropoint_matmul(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """gemm.py:159-187 -- shifted product, dequant by nd_x*nd_w, offset terms."""
    qx, ndx, zpx, offx = zeropoint_quantize(x)
    qw, ndw, zpw, offw = zeropoint_quantize(w)
    h = qx.shape[1]
    c = zeropoint_gemm_i32(qx, qw, zpx, zpw)
    out = c.astype(np.float64) / (ndx * ndw)
    if offx != 0.0 or offw != 0.0:
        ta = qx.astype(np.int64) + zpx
        tb = qw.astype(np.int64) + zpw
        out = (out + (offw / ndx) * ta.sum(axis=1, keepdims=True)
               + (offx / ndw) * tb.sum(axis=0, keepdims=True) + offx * offw * h)
    return out.astype(np.float32)


def planted_pair(rows, inner, cols, outlier_cols, outlier_scale, seed):
    """sweep.py:60-77 -- Gaussian X with scaled planted columns, Gaussian W."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((rows, inner), dtype=np.float32)
    if outlier_cols:
        idx = rng.choice(inner, size=outlier_cols, replace=False)
        x[:, idx] *= np.float32(outlier_scale)
    w = rng.standard_normal((inner, cols), dtype=np.float32)
    return x, w


# --------------------------------------------------------------------------
# C restatement (ctypes)
# --------------------------------------------------------------------------

_LIB = None


def c_oracle_path() -> Path:
    return _HERE / "liboracle_llmint8.so"


def build_c_oracle(force: bool = False) -> Path:
    """Compile oracle/llmint8_oracle.c with the committed Makefile."""
    import subprocess

    so = c_oracle_path()
    src = _HERE / "llmint8_oracle.c"
    if force or not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(_HERE), "-s"], check=True)
    return so


def c_oracle() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        so = c_oracle_path()
        if not so.exists():
            build_c_oracle()
        lib = ctypes.CDLL(str(so))
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.oracle_outlier_mask.argtypes = [P, I64, I64, ctypes.c_float, P]
        lib.oracle_outlier_mask.restype = I64
        lib.oracle_rowwise_quantize.argtypes = [P, I64, I64, P, P, P]
        lib.oracle_colwise_quantize.argtypes = [P, I64, I64, P, P, P]
        lib.oracle_gemm_i32.argtypes = [P, P, P, I64, I64, I64, ctypes.c_int]
        lib.oracle_dequantize_output.argtypes = [P, P, P, P, I64, I64]
        lib.oracle_rowwise_quantize.restype = None
        lib.oracle_colwise_quantize.restype = None
        lib.oracle_gemm_i32.restype = None
        lib.oracle_dequantize_output.restype = None
        lib.oracle_llm_int8_matmul.argtypes = [P, P, I64, I64, I64, ctypes.c_float, P, P, P, P, P, P, P,
                                               ctypes.c_int]
        lib.oracle_llm_int8_matmul.restype = I64
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_llm_int8_rows.argtypes = [P, I64, I64, I64, P, P, P, P, P, ctypes.c_int]
        lib.oracle_llm_int8_rows.restype = None
        _LIB = lib
    return _LIB


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def c_outlier_mask(x: np.ndarray, alpha: float) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    mask = np.zeros(x.shape[1], dtype=np.uint8)
    c_oracle().oracle_outlier_mask(_ptr(x), x.shape[0], x.shape[1], np.float32(alpha), _ptr(mask))
    return mask.astype(bool)


def c_gemm_i32(a: np.ndarray, b: np.ndarray, threads: int = 0) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int8)
    b = np.ascontiguousarray(b, dtype=np.int8)
    c = np.zeros((a.shape[0], b.shape[1]), dtype=np.int32)
    c_oracle().oracle_gemm_i32(_ptr(a), _ptr(b), _ptr(c), a.shape[0], b.shape[1], a.shape[1], threads)
    return c


def c_llm_int8_matmul(x: np.ndarray, w: np.ndarray, alpha: float = 6.0, threads: int = 0,
                      want_intermediates: bool = True) -> LlmInt8Trace:
    """The C restatement of gemm.py:214-247; same fields as llm_int8_matmul."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    m, h = x.shape
    n = w.shape[1]
    out = np.zeros((m, n), dtype=np.float32)
    mask = np.zeros(h, dtype=np.uint8)
    sx = np.zeros(m)
    sw = np.zeros(n)
    xq = wq = c = None
    px = pw = pc = None
    if want_intermediates:
        xq = np.zeros((m, h), dtype=np.int8)
        wq = np.zeros((h, n), dtype=np.int8)
        c = np.zeros((m, n), dtype=np.int32)
        px, pw, pc = _ptr(xq), _ptr(wq), _ptr(c)
    n_out = int(c_oracle().oracle_llm_int8_matmul(
        _ptr(x), _ptr(w), m, h, n, np.float32(alpha), _ptr(out), _ptr(mask), _ptr(sx), _ptr(sw),
        px, pw, pc, threads))
    dims = tuple(int(i) for i in np.flatnonzero(mask))
    return LlmInt8Trace(dims, xq, sx, wq, sw, c, None, out, n_out, 1.0 - n_out / h)


def c_num_threads() -> int:
    return int(c_oracle().oracle_num_threads())


if os.environ.get("ORACLE_BUILD_ON_IMPORT") == "1":  # pragma: no cover
    build_c_oracle()
