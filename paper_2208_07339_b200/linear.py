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

from ._tensors import as_f16_matrix
from .gemm import llm_int8_matmul, vectorwise_matmul

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


def linear(x, w, backend: LinearBackend, out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """x @ w through the selected backend (transformer.py:257-267).

    The reference returns float32; ``out_dtype`` defaults to that. ``absmax``
    and ``zeropoint`` are sibling schemes outside this build's scope
     and raise ``NotImplementedError``.
    """
    if backend.kind == "exact":
        x16 = as_f16_matrix(x, "x")
        w16 = as_f16_matrix(w, "w")
        return (x16.double() @ w16.double()).to(out_dtype)
    if backend.kind == "vectorwise":
        return vectorwise_matmul(x, w, out_dtype=out_dtype, validate=False).output
    if backend.kind == "llm_int8":
        return llm_int8_matmul(x, w, backend.alpha, out_dtype=out_dtype, validate=False).output
    raise NotImplementedError(
        f"backend {backend.kind!r} is not part of the B200 LLM.int8() path (SURVEY.md 8f)")


_linear = linear


class Int8Linear(torch.nn.Module):
    """LLM.int8() linear layer: y = x @ W (+ bias) with outlier decomposition.

    ``weight`` is K x N (the reference orientation, transformer.py:291-346);
    use ``Int8Linear.from_linear`` for an ``nn.Linear`` (N x K weight). The
    per-call semantics are exactly ``llm_int8_matmul`` (gemm.py:214-247).
    """

    def __init__(self, weight, alpha: float = 6.0, bias=None,
                 out_dtype: torch.dtype = torch.float16) -> None:
        super().__init__()
        self.alpha = float(alpha)
        self.out_dtype = out_dtype
        self.register_buffer("weight", as_f16_matrix(weight, "weight"))
        if bias is not None:
            b = torch.as_tensor(bias).to(device=self.weight.device, dtype=out_dtype)
            self.register_buffer("bias", b)
        else:
            self.bias = None

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

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        lead = x.shape[:-1]
        x2 = x.reshape(-1, x.shape[-1])
        y = llm_int8_matmul(x2, self.weight, self.alpha, out_dtype=self.out_dtype,
                            validate=False).output
        if self.bias is not None:
            y = y + self.bias
        return y.reshape(*lead, y.shape[-1])
