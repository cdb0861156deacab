"""The Int8 linear module and the reference's linear-backend plugin point.

Mirrors ``int8mm.transformer``'s dispatch (pkg/src/int8mm/transformer.py):
``BACKEND_KINDS`` (:42), ``LinearBackend`` (:45-56), the backend constants
(:59-62), ``llm_int8_backend`` (:65-66) and ``_linear`` (:257-267), exported
here as ``linear`` (and ``_linear``). ``Int8Linear`` is the module form used
by a model: it owns the fp16 weight and runs the LLM.int8() kernels per call.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as nat
from ._tensors import as_f16_matrix, as_operand, new_flags, raise_for_flags, stream_handle
from .errors import ShapeMismatchError
from .gemm import (_out_kind, absmax_matmul, llm_int8_matmul, vectorwise_matmul,
                   zeropoint_matmul)

BACKEND_KINDS = ("exact", "absmax", "zeropoint", "vectorwise", "llm_int8")


@dataclass(frozen=True)
class LinearBackend:
    """Which matmul pipeline the projection layers run through (transformer.py:45-56)."""

    kind: str
    alpha: float = 6.0  # outlier threshold, used by llm_int8 only

    def __post_init__(self) -> None:
        if self.kind not in BACKEND_KINDS:
            raise ValueError(f"backend kind must be one of {BACKEND_KINDS}, got {self.kind!r}")
        if not (self.alpha > 0):
            raise ValueError(f"alpha must be positive, got {self.alpha}")


EXACT = LinearBackend("exact")
ABSMAX = LinearBackend("absmax")
ZEROPOINT = LinearBackend("zeropoint")
VECTORWISE = LinearBackend("vectorwise")


def llm_int8_backend(alpha: float = 6.0) -> LinearBackend:
    """transformer.py:65-66"""
    return LinearBackend("llm_int8", alpha)


def linear(x, w, backend: LinearBackend, out_dtype: torch.dtype = torch.float32,
           exact: bool = True, validate: bool = True) -> torch.Tensor:
    """x @ w through the selected backend (transformer.py:257-267).

    Like the reference, inputs are validated as DenseMatrix would
    (tensors.py:47-48: NaN/Inf raise ValueError; device flags, one 4-byte host
    read) and the result is float32. ``exact=True`` (default) gives the
    reference's float32 output bit for bit; ``exact=False`` uses the fast fp32
    (or fp16 with ``out_dtype``) epilogue, within the stated tolerance.
    """
    if backend.kind == "exact":
        # transformer.py:259: float64 product cast to float32 (a library DGEMM;
        # not on the LLM.int8() path)
        xt = as_operand(x, "x", validate=False)
        wt = as_operand(w, "w", validate=False)
        return (xt.double() @ wt.double()).to(out_dtype)
    if backend.kind == "vectorwise":
        return vectorwise_matmul(x, w, out_dtype=out_dtype, exact=exact, validate=validate).output
    if backend.kind == "llm_int8":
        return llm_int8_matmul(x, w, backend.alpha, out_dtype=out_dtype, exact=exact,
                               validate=validate).output
    if backend.kind == "absmax":
        y = absmax_matmul(x, w, validate=validate).output
        return y if out_dtype == torch.float32 else y.to(out_dtype)
    if backend.kind == "zeropoint":
        y = zeropoint_matmul(x, w, validate=validate).output
        return y if out_dtype == torch.float32 else y.to(out_dtype)
    raise ValueError(f"backend kind must be one of {BACKEND_KINDS}, got {backend.kind!r}")


_linear = linear


class Int8Linear(torch.nn.Module):
    """LLM.int8() linear layer: y = x @ W (+ bias) with outlier decomposition.

    ``weight`` is K x N (the reference orientation, transformer.py:291-346);
    use ``Int8Linear.from_linear`` for an ``nn.Linear`` (N x K weight). The
    per-call semantics are exactly ``llm_int8_matmul`` (gemm.py:214-247).

    Weight-stationary (default): the int8 codes of W with full-column scales
    and each column's top-4 |w| candidates are prepared once
    (``i8mm_linear_prepare``); every call reproduces the reference's per-call
    column scales over the keep rows exactly by patching only the columns
    whose cached maximisers are all outlier rows (``i8mm_linear_forward``).
    ``weight_stationary=False`` re-quantizes W on every call like the reference.
    """

    def __init__(self, weight, alpha: float = 6.0, bias=None,
                 out_dtype: torch.dtype = torch.float16, weight_stationary: bool = True,
                 check_finite: bool = True) -> None:
        super().__init__()
        if not (float(alpha) > 0):
            raise ValueError(f"alpha must be positive, got {alpha}")
        self.alpha = float(alpha)
        self.out_dtype = out_dtype
        self.weight_stationary = bool(weight_stationary)
        self.check_finite = bool(check_finite)
        self.register_buffer("weight", as_f16_matrix(weight, "weight"))
        # the weight is checked once (tensors.py:47-48 rejects NaN/Inf)
        flags = new_flags(1)
        nat.check(nat.lib().i8mm_f16_check(self.weight.data_ptr(), self.weight.shape[0],
                                           self.weight.shape[1], self.weight.stride(0),
                                           flags.data_ptr(), stream_handle()), "f16_check")
        raise_for_flags(int(flags.item()))
        if bias is not None:
            b = torch.as_tensor(bias).to(device=self.weight.device, dtype=out_dtype)
            self.register_buffer("bias", b)
        else:
            self.bias = None
        self.wbuf = None
        self._last_ws = None
        self._dws = {}  # decode-routed workspaces, one per (M, stream): their counters persist
        if self.weight_stationary:
            self._prepare()

    def _prepare(self) -> None:
        L = nat.lib()
        k, n = self.weight.shape
        dev = self.weight.device
        self.wbuf = torch.empty(L.i8mm_linear_weight_bytes(k, n), dtype=torch.uint8, device=dev)
        scratch = torch.empty(L.i8mm_linear_prepare_scratch_bytes(k, n), dtype=torch.uint8,
                              device=dev)
        nat.check(L.i8mm_linear_prepare(self.weight.data_ptr(), self.weight.stride(0), k, n,
                                        self.wbuf.data_ptr(), self.wbuf.numel(),
                                        scratch.data_ptr(), scratch.numel(), stream_handle()),
                  "linear_prepare")

    def workspace(self, m: int) -> torch.Tensor:
        """A workspace for an M-row call. Prefill routing: a fresh buffer.
        Decode routing: cached per (M, stream), initialised once
        (``i8mm_linear_workspace_init``: its split-tile partial slots must be
        empty on first use; every decode call leaves them so). A workspace
        first created while a CUDA graph is being captured puts that
        initialisation into the graph; ``GraphedCall`` captures on its warm-up
        stream so the graph holds only the layer kernels."""
        L = nat.lib()
        k, n = self.weight.shape
        if not self.uses_decode(m):
            return torch.empty(L.i8mm_linear_workspace_size(m, k, n), dtype=torch.uint8,
                               device=self.weight.device)
        key = (m, torch.cuda.current_stream(self.weight.device).cuda_stream)
        ws = self._dws.get(key)
        if ws is None:
            ws = torch.empty(L.i8mm_linear_workspace_size(m, k, n), dtype=torch.uint8,
                             device=self.weight.device)
            nat.check(L.i8mm_linear_workspace_init(ws.data_ptr(), ws.numel(), m, k, n, stream_handle()),
                      "linear_workspace_init")
            self._dws[key] = ws
        return ws

    def matmul(self, x2: torch.Tensor, exact: bool = False, _timer=None) -> torch.Tensor:
        """Y = x2 @ W for an M x K fp16 CUDA matrix (no bias)."""
        if not self.weight_stationary:
            self._last_ws = None
            return llm_int8_matmul(x2, self.weight, self.alpha, out_dtype=self.out_dtype,
                                   exact=exact, _timer=_timer,
                                   validate=self.check_finite and
                                   not torch.cuda.is_current_stream_capturing()).output
        L = nat.lib()
        k, n = self.weight.shape
        m = x2.shape[0]
        if x2.shape[1] != k:
            raise ShapeMismatchError(f"inner dimensions differ: X is {m}x{x2.shape[1]}, W is {k}x{n}")
        kind, dt = _out_kind(self.out_dtype, exact)
        ws = self.workspace(m)
        y = torch.empty((m, n), dtype=dt, device=x2.device)
        st = stream_handle()
        w = self.weight
        if _timer is None:  # one entry (the decode routing is a single launch)
            nat.check(L.i8mm_linear_forward(x2.data_ptr(), x2.stride(0), m, w.data_ptr(),
                                            w.stride(0), self.wbuf.data_ptr(), k, n, self.alpha,
                                            y.data_ptr(), n, kind, ws.data_ptr(), ws.numel(),
                                            None, st), "linear_forward")
            self._last_ws = (ws, m)
            return y
        nat.check(L.i8mm_linear_prologue(x2.data_ptr(), x2.stride(0), m, w.data_ptr(), w.stride(0),
                                         self.wbuf.data_ptr(), k, n, self.alpha, ws.data_ptr(),
                                         ws.numel(), st), "linear_prologue")
        if _timer is not None:
            _timer.mark("gemm_begin")
        nat.check(L.i8mm_linear_gemm(x2.data_ptr(), x2.stride(0), m, w.data_ptr(), w.stride(0),
                                     self.wbuf.data_ptr(), k, n, y.data_ptr(), n, kind,
                                     ws.data_ptr(), ws.numel(), st), "linear_gemm")
        if _timer is not None:
            _timer.mark("gemm_end")
        self._last_ws = (ws, m)
        return y

    def uses_decode(self, m: int) -> bool:
        """True when an M-row call runs the single-launch decode kernel."""
        k, n = self.weight.shape
        return self.weight_stationary and bool(nat.lib().i8mm_linear_uses_decode(m, k, n))

    def matmul_rows(self, x2: torch.Tensor, bounds, on_rows=None, y: torch.Tensor | None = None,
                    ldy: int | None = None) -> torch.Tensor:
        """Y = x2 @ W with the GEMM issued per row range.

        One prologue over all M rows (the outlier set and the row scales need
        every row, gemm.py:210, 242), then ``i8mm_linear_gemm_rows`` for each
        ``(r0, r1)`` in ``bounds``; ``on_rows(r0, r1, y)`` runs on the host
        after each range is enqueued, so a caller can start that range's
        transfer (all-gather, device-to-host copy) on another stream while the
        next range computes. ``y`` / ``ldy`` let the caller supply a wider
        (padded) output buffer. Results are bitwise those of ``matmul``.
        """
        if not self.weight_stationary or self.uses_decode(x2.shape[0]):
            out = self.matmul(x2)
            if y is not None:
                y[:, : out.shape[1]].copy_(out)
                out = y
            if on_rows is not None:
                on_rows(0, x2.shape[0], out)
            return out
        L = nat.lib()
        k, n = self.weight.shape
        m = x2.shape[0]
        if x2.shape[1] != k:
            raise ShapeMismatchError(f"inner dimensions differ: X is {m}x{x2.shape[1]}, W is {k}x{n}")
        kind, dt = _out_kind(self.out_dtype, False)
        ws = self.workspace(m)
        if y is None:
            y = torch.empty((m, n), dtype=dt, device=x2.device)
            ldy = n
        ldy = int(ldy if ldy is not None else y.stride(0))
        st = stream_handle()
        w = self.weight
        nat.check(L.i8mm_linear_prologue(x2.data_ptr(), x2.stride(0), m, w.data_ptr(), w.stride(0),
                                         self.wbuf.data_ptr(), k, n, self.alpha, ws.data_ptr(),
                                         ws.numel(), st), "linear_prologue")
        for r0, r1 in bounds:
            nat.check(L.i8mm_linear_gemm_rows(x2.data_ptr(), x2.stride(0), m, w.data_ptr(),
                                              w.stride(0), self.wbuf.data_ptr(), k, n, y.data_ptr(),
                                              ldy, kind, ws.data_ptr(), ws.numel(), r0, r1 - r0, st),
                      "linear_gemm_rows")
            if on_rows is not None:
                on_rows(r0, r1, y)
        self._last_ws = (ws, m)
        return y

    def last_stats(self) -> dict:
        """|O| and the patched-column count of the last weight-stationary call (syncs)."""
        if self._last_ws is None:
            return {}
        import ctypes

        ws, m = self._last_ws
        k, n = self.weight.shape
        self._patch_stats(ws, m)
        views = (ctypes.c_void_p * 8)()
        nat.check(nat.lib().i8mm_linear_workspace_views(ws.data_ptr(), m, k, n, views, 8))
        # read the two device counters through byte views of the workspace
        base = ws.data_ptr()
        o_off = views[0] - base
        p_off = views[4] - base
        o = int(ws[o_off:o_off + 4].view(torch.int32).item())
        p = int(ws[p_off:p_off + 4].view(torch.int32).item())
        return {"decomposed_cols": o, "patched_cols": p}

    def last_views(self) -> dict:
        """Device views of the last weight-stationary call's intermediates (for
        parity checks): sorted outlier columns, Xq (M x K codes, 0 at outlier
        columns), row amax, and the per-call column amax over the keep rows
        (the cached full-column amax with the patched columns replaced)."""
        if self._last_ws is None:
            return {}
        import ctypes

        ws, m = self._last_ws
        k, n = self.weight.shape
        L = nat.lib()
        self._patch_stats(ws, m)
        views = (ctypes.c_void_p * 8)()
        nat.check(L.i8mm_linear_workspace_views(ws.data_ptr(), m, k, n, views, 8))
        wv = (ctypes.c_void_p * 5)()
        nat.check(L.i8mm_linear_weight_views(self.wbuf.data_ptr(), k, n, wv, 5))
        base = ws.data_ptr()
        ldq = (k + 15) // 16 * 16

        def at(ptr, count, dtype, buf=ws, b0=base):
            off = ptr - b0
            nbytes = count * torch.tensor([], dtype=dtype).element_size()
            return buf[off:off + nbytes].view(dtype)

        o = int(at(views[0], 1, torch.int32).item())
        dims = at(views[1], k, torch.int32)[:o]
        xq = at(views[2], m * ldq, torch.int8).view(m, ldq)[:, :k]
        row_amax = at(views[3], m, torch.float32)
        pc = int(at(views[4], 1, torch.int32).item())
        col_amax = at(wv[1], n, torch.float32, self.wbuf, self.wbuf.data_ptr()).clone()
        if pc:
            pidx = at(views[5], pc, torch.int32).long()
            col_amax[pidx] = at(views[6], pc, torch.float32)
        return {"dims": dims, "xq": xq, "row_amax": row_amax, "col_amax": col_amax,
                "patched_cols": pc}

    def _patch_stats(self, ws: torch.Tensor, m: int) -> None:
        """Decode-routed calls decide patched columns per tile without listing
        them: recompute the list (p_count / p_idx / p_amax) for introspection."""
        k, n = self.weight.shape
        nat.check(nat.lib().i8mm_linear_patch_stats(self.weight.data_ptr(), self.weight.stride(0),
                                                    self.wbuf.data_ptr(), m, k, n, ws.data_ptr(),
                                                    ws.numel(), stream_handle()), "linear_patch_stats")

    @classmethod
    def from_linear(cls, lin: torch.nn.Linear, alpha: float = 6.0) -> "Int8Linear":
        return cls(lin.weight.detach().t(), alpha,
                   None if lin.bias is None else lin.bias.detach())

    @property
    def in_features(self) -> int:
        return self.weight.shape[0]

    @property
    def out_features(self) -> int:
        return self.weight.shape[1]

    def _raise_if_nonfinite(self, x2: torch.Tensor) -> None:
        """check_finite: the reference's DenseMatrix(x) rejects NaN/Inf
        (transformer.py:260, tensors.py:47-48). The prefill prologue's scan
        and the decode prep kernel raise a device flag on the way. One 4-byte
        host read; skipped under CUDA-graph capture."""
        if not self.check_finite or torch.cuda.is_current_stream_capturing():
            return
        if self._last_ws is None:
            return
        ws, m = self._last_ws
        k, n = self.weight.shape
        if self.weight_stationary:
            import ctypes

            views = (ctypes.c_void_p * 8)()
            nat.check(nat.lib().i8mm_linear_workspace_views(ws.data_ptr(), m, k, n, views, 8))
            off = views[0] - ws.data_ptr() + 4  # the word after |O|
            flag = int(ws[off:off + 4].view(torch.int32).item())
        else:
            fl = new_flags(1)
            nat.check(nat.lib().i8mm_f16_check(x2.data_ptr(), x2.shape[0], x2.shape[1],
                                               x2.stride(0), fl.data_ptr(), stream_handle()))
            flag = int(fl.item())
        raise_for_flags(nat.FLAG_NONFINITE if flag else 0)

    def forward(self, x: torch.Tensor, _timer=None) -> torch.Tensor:
        lead = x.shape[:-1]
        x2 = as_f16_matrix(x.reshape(-1, x.shape[-1]), "x")
        y = self.matmul(x2, _timer=_timer)
        self._raise_if_nonfinite(x2)
        if self.bias is not None:
            y = y + self.bias
        return y.reshape(*lead, y.shape[-1])
