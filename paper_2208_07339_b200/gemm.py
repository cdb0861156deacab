"""Integer GEMM and the LLM.int8() matmul on B200, mirroring ``int8mm.gemm``.

Same names, argument meaning and error behaviour as the reference module
(pkg/src/int8mm/gemm.py); inputs/outputs are CUDA tensors (numpy arrays and
the ``tensors`` containers are accepted and copied to the device). Every
operator runs the hand-written sm_100a kernels of ``_lib/libllmint8_sm100.so``
(include/llmint8.h); there is no CPU or PyTorch-compute fallback.

Operands (``_tensors.as_operand``): fp16 inputs run the production kernels;
float32 inputs whose values are all exactly fp16 run them too (on an exact
fp16 copy); other float32 inputs run the float32 kernels (csrc/f32path.cu),
bit-exact with the reference for any finite value. ``validate`` (default
True, like the reference's DenseMatrix constructor, tensors.py:47-48) raises
ValueError on NaN/Inf from flags the kernels compute on the way (one 4-byte
host read per call).

Operator map (reference -> kernels):
  extract_outlier_columns  gemm.py:203-211 -> K1 outlier_scan + outlier_compact
  int8_gemm_i32            gemm.py:78-82   -> K4 tcgen05 GEMM, int32 epilogue
  ordered_matmul_f64       gemm.py:110-117 -> ordered f64 kernel
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
from ._tensors import (as_i8_matrix, as_operand, check_inner, common_dtype, device, kmajor_i8,
                       new_flags, raise_for_flags, round_up, stream_handle, zero_)
from .errors import GemmOverflowError, ParamsMismatchError, ShapeMismatchError
from .types import (AbsmaxParams, ColwiseParams, MatmulResult, OutlierSet, QuantizedTensor,
                    RowwiseParams, ZeropointParams)

MAX_INNER_DIM = 1 << 17  # gemm.py:35: 127^2 * 2^17 < 2^31

__all__ = [
    "MAX_INNER_DIM", "GemmOverflowError", "ParamsMismatchError", "ShapeMismatchError",
    "MatmulResult", "extract_outlier_columns", "int8_gemm_i32", "dequantize_output",
    "vectorwise_matmul", "llm_int8_matmul", "absmax_matmul", "zeropoint_matmul",
    "zeropoint_gemm_i32", "ordered_matmul_f64",
]

OUT_KINDS = {torch.float16: nat.OUT_F16, torch.float32: nat.OUT_F32}
O_CAP = 64  # width of the compacted fp16 outlier slice handed to the epilogue


def _check_alpha(alpha: float) -> None:
    a = float(alpha)
    if not (a > 0) or a != a or a in (float("inf"),):
        raise ValueError(f"alpha must be positive and finite, got {alpha}")


def _pair(x, w, validate: bool):
    xt = as_operand(x, "x", validate)
    wt = as_operand(w, "w", validate)
    (m, k), (k2, n) = xt.shape, wt.shape
    check_inner(k, k2, f"X is {m}x{k}, W is {k2}x{n}")
    xt, wt = common_dtype(xt, wt)
    return xt, wt, m, k, n


class OutlierScan:
    """Device-side result of K1: mask words, sorted index list and its count."""

    __slots__ = ("mask", "idx", "count", "nonfinite", "k")

    def __init__(self, mask, idx, count, nonfinite, k):
        self.mask, self.idx, self.count, self.nonfinite, self.k = mask, idx, count, nonfinite, k

    def dims(self) -> tuple[int, ...]:
        n = int(self.count.item())
        return tuple(int(v) for v in self.idx[:n].tolist())


def scan_outliers(xt: torch.Tensor, alpha: float) -> OutlierScan:
    """K1 on an fp16 (or float32) CUDA matrix, no host synchronisation.

    ``nonfinite`` is a device word: non-zero when X holds NaN/Inf."""
    _check_alpha(alpha)
    m, k = xt.shape
    dev = xt.device
    mask = torch.empty(((k + 31) // 32,), dtype=torch.int32, device=dev)
    idx = torch.empty((k,), dtype=torch.int32, device=dev)
    cnt = new_flags(2)  # [count, nonfinite]
    st = stream_handle()
    L = nat.lib()
    if xt.dtype == torch.float16:
        nat.check(L.i8mm_outlier_scan(xt.data_ptr(), m, k, xt.stride(0), float(alpha),
                                      mask.data_ptr(), cnt.data_ptr() + 4, st), "outlier_scan")
    else:
        nat.check(L.i8mm_f32_scan(xt.data_ptr(), m, k, xt.stride(0), float(alpha), mask.data_ptr(),
                                  cnt.data_ptr() + 4, None, 0, st), "f32_scan")
    nat.check(L.i8mm_outlier_compact(mask.data_ptr(), k, idx.data_ptr(), cnt.data_ptr(), st),
              "outlier_compact")
    return OutlierScan(mask, idx, cnt[0:1], cnt[1:2], k)


def extract_outlier_columns(x, alpha: float = 6.0, validate: bool = True) -> OutlierSet:
    """Columns of X holding a value with |value| >= alpha (gemm.py:203-211).

    The comparison is inclusive and made in float32 (numpy semantics of the
    reference). Reads the index list back to the host.
    """
    _check_alpha(alpha)
    xt = as_operand(x, "x", validate)
    sc = scan_outliers(xt, alpha)
    dims = sc.dims()
    if validate:
        raise_for_flags(int(sc.nonfinite.item()) & nat.FLAG_NONFINITE)
    return OutlierSet(dims, float(alpha))


def _quantize_rows(xt: torch.Tensor, scan: OutlierScan | None, o_cap: int = O_CAP):
    m, k = xt.shape
    ldq = round_up(k, 16)
    dev = xt.device
    xq = torch.empty((m, ldq), dtype=torch.int8, device=dev)
    amax = torch.empty((m,), dtype=torch.float32, device=dev)
    L = nat.lib()
    if xt.dtype != torch.float16:
        nat.check(L.i8mm_f32_quantize_rows(xt.data_ptr(), m, k, xt.stride(0),
                                           scan.mask.data_ptr() if scan is not None else None,
                                           xq.data_ptr(), ldq, amax.data_ptr(), stream_handle()),
                  "f32_quantize_rows")
        return xq, ldq, amax, None
    xo = torch.empty((m, o_cap), dtype=torch.float16, device=dev) if scan is not None else None
    nat.check(L.i8mm_quantize_rows(
        xt.data_ptr(), m, k, xt.stride(0),
        scan.mask.data_ptr() if scan is not None else None,
        scan.idx.data_ptr() if scan is not None else None,
        scan.count.data_ptr() if scan is not None else None,
        xq.data_ptr(), ldq, amax.data_ptr(),
        xo.data_ptr() if xo is not None else None, o_cap if xo is not None else 0,
        stream_handle()), "quantize_rows")
    return xq, ldq, amax, xo


def _quantize_cols_t(wt: torch.Tensor, scan: OutlierScan | None):
    k, n = wt.shape
    ldq = round_up(k, 16)
    dev = wt.device
    wq_t = torch.empty((n, ldq), dtype=torch.int8, device=dev)
    amax = torch.empty((n,), dtype=torch.float32, device=dev)
    L = nat.lib()
    fn = L.i8mm_quantize_cols_t if wt.dtype == torch.float16 else L.i8mm_f32_quantize_cols_t
    nat.check(fn(wt.data_ptr(), k, n, wt.stride(0),
                 scan.mask.data_ptr() if scan is not None else None,
                 wq_t.data_ptr(), ldq, amax.data_ptr(), stream_handle()), "quantize_cols_t")
    return wq_t, ldq, amax


def _f16_check(t16: torch.Tensor, flags: torch.Tensor, word: int = 0) -> None:
    nat.check(nat.lib().i8mm_f16_check(t16.data_ptr(), t16.shape[0], t16.shape[1], t16.stride(0),
                                       flags.data_ptr() + 4 * word, stream_handle()), "f16_check")


def int8_gemm_i32(a, b, validate: bool = True) -> torch.Tensor:
    """Exact integer product of int8 codes with 32-bit accumulation (gemm.py:78-82).

    ``a`` is M x K, ``b`` is K x N (reference orientation); ``b`` may be the
    transposed view returned by ``colwise_quantize`` (no copy is made then).
    Codes must lie in [-127, 127] (tensors.py:95-98): checked on the device.
    """
    a = as_i8_matrix(a, "A", validate=False)
    b = as_i8_matrix(b, "B", validate=False)
    m, k = a.shape
    k2, n = b.shape
    check_inner(k, k2, f"A is {m}x{k}, B is {k2}x{n}")
    st = stream_handle()
    L = nat.lib()
    if validate:
        flags = new_flags(2)
        for i, t in enumerate((a, b)):
            tt = t if t.stride(1) == 1 else t.t()  # the range check is layout-free
            nat.check(L.i8mm_check_codes(tt.data_ptr(), tt.shape[0], tt.shape[1], tt.stride(0),
                                         flags.data_ptr() + 4 * i, st), "check_codes")
        fa, fb = flags.tolist()
        raise_for_flags(fa, "A")
        raise_for_flags(fb, "B")
    a_buf, lda = kmajor_i8(a)
    bt = b.t()
    if bt.stride(1) == 1 and bt.stride(0) % 16 == 0 and bt.data_ptr() % 16 == 0:
        b_buf, ldb = bt, bt.stride(0)
    else:
        ldb = round_up(k, 16)
        b_buf = zero_(torch.empty((n, ldb), dtype=torch.int8, device=b.device))
        bc = b if b.stride(1) == 1 else b.contiguous()
        nat.check(L.i8mm_transpose_i8(bc.data_ptr(), k, n, bc.stride(0), b_buf.data_ptr(), ldb, st),
                  "transpose_i8")
    c = torch.empty((m, n), dtype=torch.int32, device=a.device)
    nat.check(L.i8mm_gemm_i32(a_buf.data_ptr(), lda, b_buf.data_ptr(), ldb, c.data_ptr(), n,
                              m, n, k, st), "gemm_i32")
    return c


def ordered_matmul_f64(x, w) -> torch.Tensor:
    """Float64 matmul accumulating strictly in ascending inner-index order
    (gemm.py:110-117): acc = 0; acc += outer(x[:, k], w[k, :]) for k ascending,
    every product and sum one IEEE op. float32 or float64 inputs; returns a
    float64 CUDA tensor."""
    dev = device()

    def dev_t(a):
        if isinstance(a, torch.Tensor):
            t = a.detach().to(dev)
            if t.dtype not in (torch.float32, torch.float64):
                t = t.double()
        else:
            arr = np.asarray(getattr(a, "data", a))
            arr = arr.astype(np.float64) if arr.dtype != np.float32 else arr
            t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        if t.ndim != 2:
            raise ValueError(f"ordered_matmul_f64 needs rank-2 operands, got rank {t.ndim}")
        return t if t.stride(1) == 1 else t.contiguous()

    xt, wt = dev_t(x), dev_t(w)
    if xt.dtype != wt.dtype:
        xt, wt = xt.double(), wt.double()
    (m, k), (k2, n) = xt.shape, wt.shape
    if k != k2:
        raise ShapeMismatchError(f"inner dimensions differ: X is {m}x{k}, W is {k2}x{n}")
    out = torch.empty((m, n), dtype=torch.float64, device=dev)
    nat.check(nat.lib().i8mm_ordered_matmul_f64(xt.data_ptr(), xt.stride(0), wt.data_ptr(),
                                                wt.stride(0), m, k, n, xt.element_size(),
                                                out.data_ptr(), n, stream_handle()),
              "ordered_matmul_f64")
    return out


def dequantize_output(c, params_x, params_w) -> torch.Tensor:
    """Divide an int32 accumulation by the operands' scaling constants
    (gemm.py:120-147), exactly as the reference: f32 of the f64 quotient.
    Tensor-wise params divide by the scalar product, zeropoint params by
    nd_x * nd_w, row x col params by the outer product of the scale vectors."""
    from .tensors import Int32Matrix

    if isinstance(c, Int32Matrix):
        ct = c.tensor
    elif isinstance(c, torch.Tensor):
        ct = c
    else:
        ct = torch.from_numpy(np.ascontiguousarray(getattr(c, "data", c), dtype=np.int32))
    dev = device()
    ct = ct.to(device=dev)
    if ct.dtype != torch.int32:
        ct = ct.to(torch.int32)
    if ct.stride(1) != 1:
        ct = ct.contiguous()
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
    nat.check(nat.lib().i8mm_dequantize_output(ct.data_ptr(), m, n, ct.stride(0), sx.data_ptr(),
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


def _f32_combine(c, m, n, k, ax, aw, x32, w32, scan):
    """gemm.py:239-247 on float32 operands from the int32 accumulator."""
    y = torch.empty((m, n), dtype=torch.float32, device=c.device)
    if scan is None:
        idx = cnt = new_flags(1)  # |O| = 0: vector-wise dequantization only
    else:
        idx, cnt = scan.idx, scan.count
    nat.check(nat.lib().i8mm_f32_llm_int8_combine(
        c.data_ptr(), n, m, n, k, ax.data_ptr(), aw.data_ptr(), x32.data_ptr(), x32.stride(0),
        w32.data_ptr(), w32.stride(0), idx.data_ptr(), cnt.data_ptr(), y.data_ptr(), n,
        stream_handle()), "f32_combine")
    return y


def _f32_output(y32: torch.Tensor, out_dtype, exact) -> torch.Tensor:
    if exact or out_dtype in (None, torch.float32):
        return y32
    if out_dtype != torch.float16:
        raise ValueError(f"out_dtype must be float16 or float32, got {out_dtype}")
    return y32.to(torch.float16)


def vectorwise_matmul(x, w, out_dtype: torch.dtype = torch.float16, exact: bool = False,
                      validate: bool = True) -> MatmulResult:
    """X @ W with per-row constants for X and per-column constants for W
    (gemm.py:190-200)."""
    xt, wt, m, k, n = _pair(x, w, validate)
    if xt.dtype != torch.float16:  # float32 operands: exact reference arithmetic
        xq, ldq, ax, _ = _quantize_rows(xt, None)
        wq_t, _, aw = _quantize_cols_t(wt, None)
        c = torch.empty((m, n), dtype=torch.int32, device=xt.device)
        nat.check(nat.lib().i8mm_gemm_i32(xq.data_ptr(), ldq, wq_t.data_ptr(), ldq, c.data_ptr(), n,
                                          m, n, k, stream_handle()), "gemm_i32")
        y = _f32_combine(c, m, n, k, ax, aw, xt, wt, None)
        return MatmulResult(_f32_output(y, out_dtype, exact), "vectorwise", None, k)
    flags = new_flags(1) if validate else None
    if validate:
        _f16_check(xt, flags)
        _f16_check(wt, flags)
    xq, ldq, ax, _ = _quantize_rows(xt, None)
    wq_t, _, aw = _quantize_cols_t(wt, None)
    y = _gemm_dequant(xq, wq_t, ldq, m, n, k, ax, aw, xt, wt, None, None, out_dtype, exact)
    if validate:
        raise_for_flags(int(flags.item()))
    return MatmulResult(y, "vectorwise", None, k)


def llm_int8_matmul(x, w, alpha: float = 6.0, out_dtype: torch.dtype = torch.float16,
                    exact: bool = False, validate: bool = True, _timer=None) -> MatmulResult:
    """Mixed-precision X @ W: outlier feature columns in high precision, the rest
    through the vector-wise int8 path with constants recomputed on the
    sub-matrices; the two partial products summed (gemm.py:214-247).

    ``out_dtype`` float16 (default) or float32 selects the fast fp32 epilogue;
    ``exact=True`` returns the float32 output bit-identical to the reference's.
    ``validate`` reproduces the reference's rejection of NaN/Inf inputs
    (tensors.py:47-48) from device flags (one 4-byte host read). Int8 codes,
    outlier sets, scales and the int32 accumulator are bit-exact with the
    reference in every mode; float32 operands that are not exactly fp16 take
    the float32 kernels (float32 output, exact).
    """
    _check_alpha(alpha)
    xt, wt, m, k, n = _pair(x, w, validate)
    if xt.dtype != torch.float16:
        L = nat.lib()
        ws = torch.empty((L.i8mm_f32_workspace_size(m, k, n),), dtype=torch.uint8, device=xt.device)
        status = torch.empty((2,), dtype=torch.int32, device=xt.device)
        y = torch.empty((m, n), dtype=torch.float32, device=xt.device)
        nat.check(L.i8mm_llm_int8_matmul_f32(xt.data_ptr(), xt.stride(0), wt.data_ptr(),
                                             wt.stride(0), m, k, n, float(alpha), y.data_ptr(), n,
                                             ws.data_ptr(), ws.numel(), status.data_ptr(),
                                             stream_handle()), "llm_int8_matmul_f32")
        return MatmulResult(_f32_output(y, out_dtype, exact), "llm_int8", status[0:1], k)
    if _timer is None:
        # the whole call in one native entry (scan, row / column quantization, gathers,
        # GEMM + dequant + outlier term, NaN/Inf flags): one host round trip
        L = nat.lib()
        kind, dt = _out_kind(out_dtype, exact)
        ws = torch.empty((L.i8mm_llm_int8_workspace_size(m, k, n),), dtype=torch.uint8, device=xt.device)
        y = torch.empty((m, n), dtype=dt, device=xt.device)
        cnt = torch.empty((2,), dtype=torch.int32, device=xt.device)  # [|O|, nonfinite]
        nat.check(L.i8mm_llm_int8_matmul_checked(xt.data_ptr(), xt.stride(0), wt.data_ptr(), wt.stride(0), m, k,
                                                 n, float(alpha), y.data_ptr(), n, kind, ws.data_ptr(),
                                                 ws.numel(), cnt.data_ptr(),
                                                 cnt.data_ptr() + 4 if validate else None, stream_handle()),
                  "llm_int8_matmul")
        if validate:
            raise_for_flags(nat.FLAG_NONFINITE if int(cnt[1].item()) else 0)
        return MatmulResult(y, "llm_int8", cnt[0:1], k)
    scan = scan_outliers(xt, alpha)  # gemm.py:225 (+ the X NaN/Inf flag)
    if validate:
        _f16_check(wt, scan.nonfinite)
    xq, ldq, ax, xo = _quantize_rows(xt, scan)  # gemm.py:242 (+ gather, gemm.py:238)
    wq_t, _, aw = _quantize_cols_t(wt, scan)  # gemm.py:243
    wo = _gather_outlier_rows(wt, scan)  # gemm.py:238
    if _timer is not None:
        _timer.mark("gemm_begin")
    y = _gemm_dequant(xq, wq_t, ldq, m, n, k, ax, aw, xt, wt, xo, scan, out_dtype, exact, wo)
    if _timer is not None:
        _timer.mark("gemm_end")
    if validate:
        raise_for_flags(nat.FLAG_NONFINITE if int(scan.nonfinite.item()) else 0)
    return MatmulResult(y, "llm_int8", scan.count, k)


def llm_int8_trace(x, w, alpha: float = 6.0) -> dict:
    """Every intermediate of llm_int8_matmul on the device (for parity checks):
    outlier scan, Xq / row amax, WqT / column amax, the int32 accumulator and
    the fp16 and exact-fp32 outputs (fp16 operands)."""
    from ._tensors import as_f16_matrix

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
def _stats(t: torch.Tensor) -> torch.Tensor:
    """[max|x|, min x, max x] of an fp16 / float32 matrix, on the device (one pass)."""
    rows, cols = t.shape
    scratch = torch.empty((4,), dtype=torch.int32, device=t.device)
    out = torch.empty((4,), dtype=torch.float32, device=t.device)
    L = nat.lib()
    fn = L.i8mm_tensor_stats if t.dtype == torch.float16 else L.i8mm_tensor_stats_f32
    nat.check(fn(t.data_ptr(), rows, cols, t.stride(0), scratch.data_ptr(), out.data_ptr(),
                 stream_handle()), "tensor_stats")
    return out


def _absmax_codes(t: torch.Tensor, transpose: bool):
    """absmax codes (quantize.py:137-151) row-major (rows x ldq) or K-major."""
    rows, cols = t.shape
    st = _stats(t)
    ld = round_up(rows if transpose else cols, 16)
    codes = torch.empty((cols if transpose else rows, ld), dtype=torch.int8, device=t.device)
    L = nat.lib()
    fn = L.i8mm_absmax_quantize if t.dtype == torch.float16 else L.i8mm_absmax_quantize_f32
    nat.check(fn(t.data_ptr(), rows, cols, t.stride(0), st.data_ptr(), codes.data_ptr(), ld,
                 int(transpose), stream_handle()), "absmax_quantize")
    return codes, st[0:1]


def _zeropoint_params(st: torch.Tensor) -> ZeropointParams:
    import ctypes

    lo, hi = (float(v) for v in st[1:3].cpu().tolist())
    nd, zp, off = ctypes.c_double(), ctypes.c_int32(), ctypes.c_double()
    nat.check(nat.lib().i8mm_zeropoint_params(lo, hi, ctypes.byref(nd), ctypes.byref(zp),
                                              ctypes.byref(off)), "zeropoint_quantize")
    return ZeropointParams(nd=nd.value, zp=int(zp.value), offset=off.value)


def _zeropoint_codes(t: torch.Tensor, transpose: bool):
    """zeropoint codes (quantize.py:153-171); params validated on the host."""
    rows, cols = t.shape
    params = _zeropoint_params(_stats(t))
    ld = round_up(rows if transpose else cols, 16)
    codes = torch.empty((cols if transpose else rows, ld), dtype=torch.int8, device=t.device)
    if params.offset != 0.0:  # constant tensor: its value rides in the offset, codes 0
        return zero_(codes), params
    L = nat.lib()
    fn = L.i8mm_zeropoint_quantize if t.dtype == torch.float16 else L.i8mm_zeropoint_quantize_f32
    nat.check(fn(t.data_ptr(), rows, cols, t.stride(0), float(params.nd), int(params.zp),
                 codes.data_ptr(), ld, int(transpose), stream_handle()), "zeropoint_quantize")
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
    c = int8_gemm_i32(a, b, validate=False)
    L = nat.lib()
    st = stream_handle()
    a_buf, lda = kmajor_i8(a)
    bt = b.t().contiguous()
    ra = torch.empty((m,), dtype=torch.int32, device=a.device)
    cb = torch.empty((n,), dtype=torch.int32, device=a.device)
    nat.check(L.i8mm_rowsum_i8(a_buf.data_ptr(), m, k, lda, ra.data_ptr(), st), "rowsum")
    nat.check(L.i8mm_rowsum_i8(bt.data_ptr(), n, k, k, cb.data_ptr(), st), "colsum")
    flag = new_flags(1)
    acc = torch.empty((m, n), dtype=torch.int32, device=a.device)
    nat.check(L.i8mm_zeropoint_combine(c.data_ptr(), m, n, n, ra.data_ptr(), cb.data_ptr(), k,
                                       int(zp_a), int(zp_b), 1.0, 1.0, 0.0, 0.0, None, 0,
                                       acc.data_ptr(), flag.data_ptr(), st), "zeropoint_combine")
    if int(flag.item()):
        raise GemmOverflowError("accumulated values exceed the signed 32-bit range")
    return acc


def absmax_matmul(x, w, validate: bool = True) -> MatmulResult:
    """X @ W via tensor-wise absmax quantization of both operands
    (gemm.py:150-156); float32 output."""
    xt, wt, m, k, n = _pair(x, w, validate)
    L = nat.lib()
    y = torch.empty((m, n), dtype=torch.float32, device=xt.device)
    if xt.dtype == torch.float16:
        flags = new_flags(1) if validate else None
        if validate:
            _f16_check(xt, flags)
            _f16_check(wt, flags)
        ws = torch.empty(L.i8mm_scalar_workspace_size(m, k, n), dtype=torch.uint8, device=xt.device)
        nat.check(L.i8mm_absmax_matmul(xt.data_ptr(), xt.stride(0), wt.data_ptr(), wt.stride(0),
                                       m, k, n, y.data_ptr(), n, ws.data_ptr(), ws.numel(),
                                       stream_handle()), "absmax_matmul")
        if validate:
            raise_for_flags(int(flags.item()))
        return MatmulResult(y, "absmax", None, k)
    qx, ax = _absmax_codes(xt, transpose=False)
    qw_t, aw = _absmax_codes(wt, transpose=True)
    c = torch.empty((m, n), dtype=torch.int32, device=xt.device)
    st = stream_handle()
    nat.check(L.i8mm_gemm_i32(qx.data_ptr(), qx.shape[1], qw_t.data_ptr(), qw_t.shape[1],
                              c.data_ptr(), n, m, n, k, st), "gemm_i32")
    nat.check(L.i8mm_dequantize_absmax(c.data_ptr(), m, n, n, ax.data_ptr(), aw.data_ptr(),
                                       y.data_ptr(), n, st), "dequantize_absmax")
    return MatmulResult(y, "absmax", None, k)


def zeropoint_matmul(x, w, unrolled: bool = False, validate: bool = True) -> MatmulResult:
    """X @ W via tensor-wise zeropoint quantization of both operands
    (gemm.py:159-187), including the constant-tensor offset terms; float32
    output. ``unrolled`` selects between two bit-identical forms in the
    reference and is accepted for API parity. Synchronises the stream (the
    zeropoints are validated on the host like quantize.py:162-166)."""
    xt, wt, m, k, n = _pair(x, w, validate)
    L = nat.lib()
    y = torch.empty((m, n), dtype=torch.float32, device=xt.device)
    if xt.dtype == torch.float16:
        if validate:
            flags = new_flags(1)
            _f16_check(xt, flags)
            _f16_check(wt, flags)
            raise_for_flags(int(flags.item()))
        ws = torch.empty(L.i8mm_scalar_workspace_size(m, k, n), dtype=torch.uint8, device=xt.device)
        nat.check(L.i8mm_zeropoint_matmul(xt.data_ptr(), xt.stride(0), wt.data_ptr(),
                                          wt.stride(0), m, k, n, y.data_ptr(), n, ws.data_ptr(),
                                          ws.numel(), stream_handle()), "zeropoint_matmul")
        return MatmulResult(y, "zeropoint", None, k)
    qx, px = _zeropoint_codes(xt, transpose=False)
    qw_t, pw = _zeropoint_codes(wt, transpose=True)
    st = stream_handle()
    c = torch.empty((m, n), dtype=torch.int32, device=xt.device)
    nat.check(L.i8mm_gemm_i32(qx.data_ptr(), qx.shape[1], qw_t.data_ptr(), qw_t.shape[1],
                              c.data_ptr(), n, m, n, k, st), "gemm_i32")
    ra = torch.empty((m,), dtype=torch.int32, device=xt.device)
    cb = torch.empty((n,), dtype=torch.int32, device=xt.device)
    nat.check(L.i8mm_rowsum_i8(qx.data_ptr(), m, k, qx.shape[1], ra.data_ptr(), st), "rowsum")
    nat.check(L.i8mm_rowsum_i8(qw_t.data_ptr(), n, k, qw_t.shape[1], cb.data_ptr(), st), "colsum")
    flag = new_flags(1)
    nat.check(L.i8mm_zeropoint_combine(c.data_ptr(), m, n, n, ra.data_ptr(), cb.data_ptr(), k,
                                       int(px.zp), int(pw.zp), float(px.nd), float(pw.nd),
                                       float(px.offset), float(pw.offset), y.data_ptr(), n, None,
                                       flag.data_ptr(), st), "zeropoint_combine")
    if int(flag.item()):
        raise GemmOverflowError("accumulated values exceed the signed 32-bit range")
    return MatmulResult(y, "zeropoint", None, k)
