"""Exception classes of the reference's operator API, same names and bases.

* ``ShapeMismatchError``  -- tensors.py:21
* ``GemmOverflowError``   -- gemm.py:41-42
* ``ParamsMismatchError`` -- gemm.py:45-46
"""


class ShapeMismatchError(ValueError):
    """Operand shapes are not conformable for the requested operation."""


class GemmOverflowError(ValueError):
    """The accumulation would not fit in a signed 32-bit integer."""


class ParamsMismatchError(ValueError):
    """Quantization params do not match the scheme expected for this output."""
