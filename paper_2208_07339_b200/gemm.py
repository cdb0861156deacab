"""Integer GEMM and the LLM.int8() matmul on B200, mirroring ``int8mm.gemm``.

Same names, argument meaning and error behaviour as the reference module
(pkg/src/int8mm/gemm.py); inputs/outputs are CUDA tensors (numpy arrays are
accepted and copied to the device). Every operator runs the hand-written
sm_100a kernels of ``_lib/libllmint8_sm100.so`` (include/llmint8.h); there is no
CPU or PyTorch-compute fallback.

Operator map (reference -> kernels):
  extract_outlier_columns  gemm.py:203-211 -> K1 outlier_scan + outlier_compact
  int8_gemm_i32            gemm.py:78-82   -> K4 tcgen05 GEMM, int32 epilogue
  dequantize_output        gemm.py:120-147 -> exact f64 dequant kernel
  vectorwise_matmul        gemm.py:197-200 -> K2 + K3 + K4 (fused dequant)
  llm_int8_matmul          gemm.py:214-247 -> K1 + K2 + K3 + K4 (fused dequant
                                              + outlier term in the epilogue)
  absmax_matmul            gemm.py:150-156 -> tensor stats + scalar quantizers
                                              + K4 (int32) + f64 dequant
  zeropoint_gemm_i32       gemm.py:85-104  -> K4 (int32) + row sums + exact
                                              int64 zeropoint identity
  zeropoint_matmul         gemm.py:159-187 -> the above + f64 dequant/offsets
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from ._tensors import (as_f16_matrix, as_i8_matrix, check_inner, device, kmajor_i8, round_up,
                       stream_handle)
from .errors import GemmOverflowError, ParamsMismatchError, ShapeMismatchError
from .types import (AbsmaxParams, ColwiseParams, MatmulResult, OutlierSet, QuantizedTensor,
                    RowwiseParams, ZeropointParams)

MAX_INNER_DIM = 1 << 17  # gemm.py:35: 127^2 * 2^17 < 2^31

__all__ = [
    "MAX_INNER_DIM", "GemmOverflowError", "ParamsMismatchError", "ShapeMismatchError",
    "MatmulResult", "extract_outlier_columns", "int8_gemm_i32", "dequantize_output",
    "vectorwise_matmul", "llm_int8_matmul", "absmax_matmul", "zeropoint_matmul",
    "zeropoint_gemm_i32",
]

OUT_KINDS = {torch.float16: nat.OUT_F16, torch.float32: nat.OUT_F32}
O_CAP = 64  # width of the compacted fp16 outlier slice handed to the epilogue


def _check_alpha(alpha: float) -> None:
    a = float(alpha)
    if not (a > 0) or a != a or a in (float("inf"),):
        raise ValueError(f"alpha must be positive and finite, got {alpha}")


class OutlierScan:
    """Device-side result of K1: mask words, sorted index list and its count."""

    __slots__ = ("mask", "idx", "count", "nonfinite", "k")

    def __init__(self, mask, idx, count, nonfinite, k):
        self.mask, self.idx, self.count, self.nonfinite, self.k = mask, idx, count, nonfinite, k

    def dims(self) -> tuple[int, ...]:
        n = int(self.count.item())
        return tuple(int(v) for v in self.idx[:n].tolist())


def scan_outliers(x16: torch.Tensor, alpha: float) -> OutlierScan:
    """K1 on an fp16 CUDA matrix, no host synchronisation."""
    _check_alpha(alpha)
    m, k = x16.shape
    dev = x16.device
    mask = torch.empty(((k + 31) // 32,), dtype=torch.int32, device=dev)
    idx = torch.empty((k,), dtype=torch.int32, device=dev)
    cnt = torch.zeros((2,), dtype=torch.int32, device=dev)  # [count, nonfinite]
    st = stream_handle()
    L = nat.lib()
    nat.check(L.i8mm_outlier_scan(x16.data_ptr(), m, k, x16.stride(0), float(alpha),
                                  mask.data_ptr(), cnt.data_ptr() + 4, st), "outlier_scan")
    nat.check(L.i8mm_outlier_compact(mask.data_ptr(), k, idx.data_ptr(), cnt.data_ptr(), st),
              "outlier_compact")
    return OutlierScan(mask, idx, cnt[0:1], cnt[1:2], k)


def extract_outlier_columns(x, alpha: float = 6.0) -> OutlierSet:
    """Columns of X holding a value with |value| >= alpha (gemm.py:203-211).

    The comparison is inclusive and made in float32 (numpy semantics of the
    reference). Reads the index list back to the host.
    """
    _check_alpha(alpha)
    x16 = as_f16_matrix(x, "x")
    sc = scan_outliers(x16, alpha)
    return OutlierSet(sc.dims(), float(alpha))


def _quantize_rows(x16: torch.Tensor, scan: OutlierScan | None, o_cap: int = O_CAP):
    m, k = x16.shape
    ldq = round_up(k, 16)
    dev = x16.device
    xq = torch.empty((m, ldq), dtype=torch.int8, device=dev)
    amax = torch.empty((m,), dtype=torch.float32, device=dev)
    xo = torch.empty((m, o_cap), dtype=torch.float16, device=dev) if scan is not None else None
    L = nat.lib()
    nat.check(L.i8mm_quantize_rows(
        x16.data_ptr(), m, k, x16.stride(0),
        scan.mask.data_ptr() if scan is not None else None,
        scan.idx.data_ptr() if scan is not None else None,
        scan.count.data_ptr() if scan is not None else None,
        xq.data_ptr(), ldq, amax.data_ptr(),
        xo.data_ptr() if xo is not None else None, o_cap if xo is not None else 0,
        stream_handle()), "quantize_rows")
    return xq, ldq, amax, xo


def _quantize_cols_t(w16: torch.Tensor, scan: OutlierScan | None):
    k, n = w16.shape
    ldq = round_up(k, 16)
    dev = w16.device
    wq_t = torch.empty((n, ldq), dtype=torch.int8, device=dev)
    amax = torch.empty((n,), dtype=torch.float32, device=dev)
    nat.check(nat.lib().i8mm_quantize_cols_t(
        w16.data_ptr(), k, n, w16.stride(0),
        scan.mask.data_ptr() if scan is not None else None,
        wq_t.data_ptr(), ldq, amax.data_ptr(), stream_handle()), "quantize_cols_t")
    return wq_t, ldq, amax


def int8_gemm_i32(a, b) -> torch.Tensor:
    """Exact integer product of int8 codes with 32-bit accumulation (gemm.py:78-82).

    ``a`` is M x K, ``b`` is K x N (reference orientation); ``b`` may be the
    transposed view returned by ``colwise_quantize`` (no copy is made then).
    Codes must lie in [-127, 127] (tensors.py:95-98).
    """
    a = as_i8_matrix(a, "A")
    b = as_i8_matrix(b, "B")
    m, k = a.shape
    k2, n = b.shape
    check_inner(k, k2, f"A is {m}x{k}, B is {k2}x{n}")
    for name, t in (("A", a), ("B", b)):
        if t.numel() and bool((t == -128).any()):
            raise ValueError(f"Int8Matrix values must lie in [-127, 127] ({name})")
    a_buf, lda = kmajor_i8(a)
    bt = b.t()
    st = stream_handle()
    L = nat.lib()
    if bt.stride(1) == 1 and bt.stride(0) % 16 == 0 and bt.data_ptr() % 16 == 0:
        b_buf, ldb = bt, bt.stride(0)
    else:
        ldb = round_up(k, 16)
        b_buf = torch.zeros((n, ldb), dtype=torch.int8, device=b.device)
        bc = b.contiguous()
        nat.check(L.i8mm_transpose_i8(bc.data_ptr(), k, n, n, b_buf.data_ptr(), ldb, st),
                  "transpose_i8")
    c = torch.empty((m, n), dtype=torch.int32, device=a.device)
    nat.check(L.i8mm_gemm_i32(a_buf.data_ptr(), lda, b_buf.data_ptr(), ldb, c.data_ptr(), n,
                              m, n, k, st), "gemm_i32")
    return c


def dequantize_output(c, params_x, params_w) -> torch.Tensor:
    """Divide an int32 accumulation by the operands' scaling constants
    (gemm.py:120-147), exactly as the reference: f32 of the f64 quotient.
    Tensor-wise params divide by the scalar product, zeropoint params by
    nd_x * nd_w, row x col params by the outer product of the scale vectors."""
    if isinstance(c, torch.Tensor):
        ct = c
    else:
        ct = torch.from_numpy(np.ascontiguousarray(getattr(c, "data", c), dtype=np.int32))
    dev = device()
    ct = ct.to(device=dev, dtype=torch.int32).contiguous()
    m, n = ct.shape
    if isinstance(params_x, AbsmaxParams) and isinstance(params_w, AbsmaxParams):
        sx_h = np.full(m, params_x.scale, dtype=np.float64)
        sw_h = np.full(n, params_w.scale, dtype=np.float64)
    elif isinstance(params_x, ZeropointParams) and isinstance(params_w, ZeropointParams):
        sx_h = np.full(m, params_x.nd, dtype=np.float64)
        sw_h = np.full(n, params_w.nd, dtype=np.float64)
    elif isinstance(params_x, RowwiseParams) and isinstance(params_w, ColwiseParams):
        if params_x.size != m or params_w.size != n:
            raise ParamsMismatchError(
                f"scale vector lengths ({params_x.size}, {params_w.size}) "
                f"do not match output shape {(m, n)}")
        sx_h, sw_h = params_x.scales, params_w.scales
    else:
        raise ParamsMismatchError(
            f"unsupported params pairing: {type(params_x).__name__} x {type(params_w).__name__}")
    # the same f64 op order for every branch: q = c / (s_x[i] * s_w[j])
    sx = torch.from_numpy(np.array(sx_h, dtype=np.float64)).to(dev)
    sw = torch.from_numpy(np.array(sw_h, dtype=np.float64)).to(dev)
    out = torch.empty((m, n), dtype=torch.float32, device=dev)
    nat.check(nat.lib().i8mm_dequantize_output(ct.data_ptr(), m, n, n, sx.data_ptr(),
                                               sw.data_ptr(), out.data_ptr(), n,
                                               stream_handle()), "dequantize_output")
    return out


def _gather_outlier_rows(w16: torch.Tensor, scan: OutlierScan, cap: int = O_CAP):
    """Compact W[O, :] (fp16, cap x ceil8(N)) for the GEMM epilogue (gemm.py:238)."""
    k, n = w16.shape
    ldwo = round_up(n, 8)
    wo = torch.empty((cap, ldwo), dtype=torch.float16, device=w16.device)
    nat.check(nat.lib().i8mm_gather_outlier_rows(
        w16.data_ptr(), w16.stride(0), n, scan.idx.data_ptr(), scan.count.data_ptr(), cap,
        wo.data_ptr(), ldwo, stream_handle()), "gather_outlier_rows")
    return wo


def _out_kind(out_dtype, exact):
    if exact:
        return nat.OUT_F32_EXACT, torch.float32
    if out_dtype not in OUT_KINDS:
        raise ValueError(f"out_dtype must be float16 or float32, got {out_dtype}")
    return OUT_KINDS[out_dtype], out_dtype


def _gemm_dequant(xq, wq_t, ldq, m, n, k, ax, aw, x16, w16, xo, scan, out_dtype, exact, wo=None):
    dev = xq.device
    kind, dt = _out_kind(out_dtype, exact)
    y = torch.empty((m, n), dtype=dt, device=dev)
    nat.check(nat.lib().i8mm_gemm_dequant(
        xq.data_ptr(), wq_t.data_ptr(), ldq, m, n, k, ax.data_ptr(), aw.data_ptr(),
        x16.data_ptr(), x16.stride(0), w16.data_ptr(), w16.stride(0),
        xo.data_ptr() if xo is not None else None, xo.shape[1] if xo is not None else 0,
        wo.data_ptr() if wo is not None else None, wo.shape[1] if wo is not None else 0,
        scan.idx.data_ptr() if scan is not None else None,
        scan.count.data_ptr() if scan is not None else None,
        y.data_ptr(), n, kind, stream_handle()), "gemm_dequant")
    return y


def _check_finite(t16: torch.Tensor, name: str) -> None:
    if not bool(torch.isfinite(t16).all()):
        raise ValueError("DenseMatrix rejects NaN/Inf entries")


def vectorwise_matmul(x, w, out_dtype: torch.dtype = torch.float16, exact: bool = False,
                      validate: bool = True) -> MatmulResult:
    """X @ W with per-row constants for X and per-column constants for W
    (gemm.py:190-200)."""
    x16 = as_f16_matrix(x, "x")
    w16 = as_f16_matrix(w, "w")
    (m, k), (k2, n) = x16.shape, w16.shape
    check_inner(k, k2, f"X is {m}x{k}, W is {k2}x{n}")
    if validate:
        _check_finite(x16, "x")
        _check_finite(w16, "w")
    xq, ldq, ax, _ = _quantize_rows(x16, None)
    wq_t, _, aw = _quantize_cols_t(w16, None)
    y = _gemm_dequant(xq, wq_t, ldq, m, n, k, ax, aw, x16, w16, None, None, out_dtype, exact)
    return MatmulResult(y, "vectorwise", None, k)


def llm_int8_matmul(x, w, alpha: float = 6.0, out_dtype: torch.dtype = torch.float16,
                    exact: bool = False, validate: bool = True, _timer=None) -> MatmulResult:
    """Mixed-precision X @ W: outlier feature columns in high precision, the rest
    through the vector-wise int8 path with constants recomputed on the
    sub-matrices; the two partial products summed (gemm.py:214-247).

    ``out_dtype`` float16 (default) or float32 selects the fast fp32 epilogue;
    ``exact=True`` runs the f64 epilogue whose float32 output is bit-identical
    to the reference's. ``validate`` reproduces the reference's rejection of
    NaN/Inf inputs (tensors.py:47-48) at the cost of one host sync.
    Int8 codes, outlier sets, scales and the int32 accumulator are bit-exact
    with the reference in every mode.
    """
    x16 = as_f16_matrix(x, "x")
    w16 = as_f16_matrix(w, "w")
    (m, k), (k2, n) = x16.shape, w16.shape
    check_inner(k, k2, f"X is {m}x{k}, W is {k2}x{n}")
    scan = scan_outliers(x16, alpha)  # gemm.py:225
    if validate:
        if int(scan.nonfinite.item()):
            raise ValueError("DenseMatrix rejects NaN/Inf entries")
        _check_finite(w16, "w")
    xq, ldq, ax, xo = _quantize_rows(x16, scan)  # gemm.py:242 (+ gather, gemm.py:238)
    wq_t, _, aw = _quantize_cols_t(w16, scan)  # gemm.py:243
    wo = _gather_outlier_rows(w16, scan)  # gemm.py:238
    if _timer is not None:
        _timer.mark("gemm_begin")
    y = _gemm_dequant(xq, wq_t, ldq, m, n, k, ax, aw, x16, w16, xo, scan, out_dtype, exact, wo)
    if _timer is not None:
        _timer.mark("gemm_end")
    return MatmulResult(y, "llm_int8", scan.count, k)


def llm_int8_trace(x, w, alpha: float = 6.0) -> dict:
    """Every intermediate of llm_int8_matmul on the device (for parity checks):
    outlier scan, Xq / row amax, WqT / column amax, the int32 accumulator and
    the fp16 and exact-fp32 outputs."""
    x16 = as_f16_matrix(x, "x")
    w16 = as_f16_matrix(w, "w")
    (m, k), (k2, n) = x16.shape, w16.shape
    check_inner(k, k2, f"X is {m}x{k}, W is {k2}x{n}")
    scan = scan_outliers(x16, alpha)
    xq, ldq, ax, xo = _quantize_rows(x16, scan)
    wq_t, _, aw = _quantize_cols_t(w16, scan)
    c = torch.empty((m, n), dtype=torch.int32, device=x16.device)
    L = nat.lib()
    nat.check(L.i8mm_gemm_i32(xq.data_ptr(), ldq, wq_t.data_ptr(), ldq, c.data_ptr(), n, m, n, k,
                              stream_handle()), "gemm_i32")
    wo = _gather_outlier_rows(w16, scan)
    y16 = _gemm_dequant(xq, wq_t, ldq, m, n, k, ax, aw, x16, w16, xo, scan, torch.float16, False,
                        wo)
    y32 = _gemm_dequant(xq, wq_t, ldq, m, n, k, ax, aw, x16, w16, xo, scan, torch.float32, False,
                        wo)
    yex = _gemm_dequant(xq, wq_t, ldq, m, n, k, ax, aw, x16, w16, xo, scan, None, True, wo)
    return {"scan": scan, "xq": xq[:, :k], "row_amax": ax, "wq_t": wq_t[:, :k], "col_amax": aw,
            "c": c, "y16": y16, "y32": y32, "y_exact": yex, "xo": xo}


# ---------------------------------------------------------------- sibling schemes
def _stats(t16: torch.Tensor) -> torch.Tensor:
    """[max|x|, min x, max x] of an fp16 matrix, on the device (one pass)."""
    rows, cols = t16.shape
    scratch = torch.empty((4,), dtype=torch.int32, device=t16.device)
    out = torch.empty((4,), dtype=torch.float32, device=t16.device)
    nat.check(nat.lib().i8mm_tensor_stats(t16.data_ptr(), rows, cols, t16.stride(0),
                                          scratch.data_ptr(), out.data_ptr(), stream_handle()),
              "tensor_stats")
    return out


def _absmax_codes(t16: torch.Tensor, transpose: bool):
    """absmax codes (quantize.py:137-151) row-major (rows x ldq) or K-major."""
    rows, cols = t16.shape
    st = _stats(t16)
    ld = round_up(rows if transpose else cols, 16)
    codes = torch.empty((cols if transpose else rows, ld), dtype=torch.int8, device=t16.device)
    nat.check(nat.lib().i8mm_absmax_quantize(t16.data_ptr(), rows, cols, t16.stride(0),
                                             st.data_ptr(), codes.data_ptr(), ld, int(transpose),
                                             stream_handle()), "absmax_quantize")
    return codes, st[0:1]


def _zeropoint_params(st: torch.Tensor) -> ZeropointParams:
    import ctypes

    lo, hi = (float(v) for v in st[1:3].cpu().tolist())
    nd, zp, off = ctypes.c_double(), ctypes.c_int32(), ctypes.c_double()
    nat.check(nat.lib().i8mm_zeropoint_params(lo, hi, ctypes.byref(nd), ctypes.byref(zp),
                                              ctypes.byref(off)), "zeropoint_quantize")
    return ZeropointParams(nd=nd.value, zp=int(zp.value), offset=off.value)


def _zeropoint_codes(t16: torch.Tensor, transpose: bool):
    """zeropoint codes (quantize.py:153-171); params validated on the host."""
    rows, cols = t16.shape
    params = _zeropoint_params(_stats(t16))
    ld = round_up(rows if transpose else cols, 16)
    if params.offset != 0.0:  # constant tensor: its value rides in the offset, codes 0
        codes = torch.zeros((cols if transpose else rows, ld), dtype=torch.int8, device=t16.device)
        return codes, params
    codes = torch.empty((cols if transpose else rows, ld), dtype=torch.int8, device=t16.device)
    nat.check(nat.lib().i8mm_zeropoint_quantize(t16.data_ptr(), rows, cols, t16.stride(0),
                                                float(params.nd), int(params.zp), codes.data_ptr(),
                                                ld, int(transpose), stream_handle()),
              "zeropoint_quantize")
    return codes, params


def zeropoint_gemm_i32(a, b, zp_a: int, zp_b: int, unrolled: bool = False) -> torch.Tensor:
    """Integer product of zeropoint-shifted codes (A + zp_a)(B + zp_b)
    (gemm.py:85-104). Computed as the unrolled identity
    A@B + zp_b*rowsum(A) + zp_a*colsum(B) + h*zp_a*zp_b in exact int64 (the
    direct and unrolled forms are bit-identical); GemmOverflowError when a
    result leaves int32 (gemm.py:71-75). One host sync for the range flag."""
    a = as_i8_matrix(a, "A")
    b = as_i8_matrix(b, "B")
    m, k = a.shape
    k2, n = b.shape
    check_inner(k, k2, f"A is {m}x{k}, B is {k2}x{n}")
    c = int8_gemm_i32(a, b)
    L = nat.lib()
    st = stream_handle()
    a_buf, lda = kmajor_i8(a)
    bt = b.t().contiguous()
    ra = torch.empty((m,), dtype=torch.int32, device=a.device)
    cb = torch.empty((n,), dtype=torch.int32, device=a.device)
    nat.check(L.i8mm_rowsum_i8(a_buf.data_ptr(), m, k, lda, ra.data_ptr(), st), "rowsum")
    nat.check(L.i8mm_rowsum_i8(bt.data_ptr(), n, k, k, cb.data_ptr(), st), "colsum")
    flag = torch.zeros((1,), dtype=torch.int32, device=a.device)
    acc = torch.empty((m, n), dtype=torch.int32, device=a.device)
    nat.check(L.i8mm_zeropoint_combine(c.data_ptr(), m, n, n, ra.data_ptr(), cb.data_ptr(), k,
                                       int(zp_a), int(zp_b), 1.0, 1.0, 0.0, 0.0, None, 0,
                                       acc.data_ptr(), flag.data_ptr(), st), "zeropoint_combine")
    if int(flag.item()):
        raise GemmOverflowError("accumulated values exceed the signed 32-bit range")
    return acc


def absmax_matmul(x, w) -> MatmulResult:
    """X @ W via tensor-wise absmax quantization of both operands
    (gemm.py:150-156); float32 output, no host synchronisation."""
    x16 = as_f16_matrix(x, "x")
    w16 = as_f16_matrix(w, "w")
    (m, k), (k2, n) = x16.shape, w16.shape
    check_inner(k, k2, f"X is {m}x{k}, W is {k2}x{n}")
    L = nat.lib()
    ws = torch.empty(L.i8mm_scalar_workspace_size(m, k, n), dtype=torch.uint8, device=x16.device)
    y = torch.empty((m, n), dtype=torch.float32, device=x16.device)
    nat.check(L.i8mm_absmax_matmul(x16.data_ptr(), x16.stride(0), w16.data_ptr(), w16.stride(0),
                                   m, k, n, y.data_ptr(), n, ws.data_ptr(), ws.numel(),
                                   stream_handle()), "absmax_matmul")
    return MatmulResult(y, "absmax", None, k)


def zeropoint_matmul(x, w, unrolled: bool = False) -> MatmulResult:
    """X @ W via tensor-wise zeropoint quantization of both operands
    (gemm.py:159-187), including the constant-tensor offset terms; float32
    output. ``unrolled`` selects between two bit-identical forms in the
    reference and is accepted for API parity. Synchronises the stream (the
    zeropoints are validated on the host like quantize.py:162-166)."""
    x16 = as_f16_matrix(x, "x")
    w16 = as_f16_matrix(w, "w")
    (m, k), (k2, n) = x16.shape, w16.shape
    check_inner(k, k2, f"X is {m}x{k}, W is {k2}x{n}")
    L = nat.lib()
    ws = torch.empty(L.i8mm_scalar_workspace_size(m, k, n), dtype=torch.uint8, device=x16.device)
    y = torch.empty((m, n), dtype=torch.float32, device=x16.device)
    nat.check(L.i8mm_zeropoint_matmul(x16.data_ptr(), x16.stride(0), w16.data_ptr(),
                                      w16.stride(0), m, k, n, y.data_ptr(), n, ws.data_ptr(),
                                      ws.numel(), stream_handle()), "zeropoint_matmul")
    return MatmulResult(y, "zeropoint", None, k)
