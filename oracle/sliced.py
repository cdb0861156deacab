"""Sliced CPU oracle for production-size shapes -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` and ``bench.py``'s post-timing parity leg import this module;
the product (``paper_2208_07339_b200``) never does.

At the benchmark configurations (cfg2 16384x4096x16384, cfg5
16384x12288x49152, ...) the full CPU oracle would take hours. The reference
algorithm (gemm.py:214-247) is row-separable once the outlier set is known:

* O = columns of X with any |x| >= alpha over ALL rows (gemm.py:208-211) --
  computed here from the full X, chunked;
* row i's scale and codes depend only on row i's keep entries
  (quantize.py:174-179 via gemm.py:242);
* column j's scale and codes depend only on column j of W[keep, :]
  (quantize.py:182-187 via gemm.py:243) -- computed for every column;
* Y[i, :] = f32(f64(f32(C[i, :] / (s_x[i] s_w))) + sum_{o in O asc} x[i,o] w[o,:])
  (gemm.py:130-147, 110-117, 244).

So the oracle restated for a sample of rows, with O and the column scales taken
over the full matrices, is exact -- not an approximation -- for those rows.
The row quantizer and the column quantizer are the C restatement
(oracle/llmint8_oracle.c, -ffp-contract=off); the int8 product uses float64
BLAS on the codes, exact because every partial sum is an integer below 2^53
(oracle/oracle.py module docstring).
"""

from __future__ import annotations

import numpy as np

from . import oracle as orc


def outlier_mask_f16(x16: np.ndarray, alpha: float, chunk_rows: int = 2048) -> np.ndarray:
    """gemm.py:208-210 over the full fp16 X: any_i |x_ik| >= f32(alpha).

    fp16 -> f32 is exact, so this is the reference's float32 comparison on the
    same values.
    """
    m, k = x16.shape
    a = np.float32(alpha)
    mask = np.zeros(k, dtype=bool)
    for r0 in range(0, m, chunk_rows):
        blk = np.abs(x16[r0:r0 + chunk_rows].astype(np.float32))
        mask |= (blk >= a).any(axis=0)
    return mask


def sample_rows(m: int, tile: int = 256, seed: int = 0, per_tile: int = 1) -> np.ndarray:
    """``per_tile`` rows in every ``tile``-row block (at varying offsets), plus
    the first and the last row (the ragged edge)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rows = {0, m - 1}
    for t0 in range(0, m, tile):
        hi = min(t0 + tile, m)
        for r in rng.integers(t0, hi, size=per_tile):
            rows.add(int(r))
    return np.array(sorted(rows), dtype=np.int64)


def sliced_llm_int8(x16: np.ndarray, w16: np.ndarray, rows: np.ndarray, alpha: float = 6.0,
                    mask: np.ndarray | None = None, col_chunk: int | None = None,
                    want_c: bool = True) -> dict:
    """Every intermediate of gemm.py:214-247 for X[rows, :] @ W (all N columns).

    x16: M x K fp16 host array (the whole X -- O needs every row);
    w16: K x N fp16 host array. Returns dims, row scales / codes (full-K
    layout, zeros at outlier columns), column scales (all N), the int32
    accumulator rows (``want_c``) and the float32 output rows.
    """
    m, k = x16.shape
    k2, n = w16.shape
    assert k == k2
    if mask is None:
        mask = outlier_mask_f16(x16, alpha)
    dims = tuple(int(i) for i in np.flatnonzero(mask))
    keep_any = not bool(mask.all())
    mask_u8 = np.ascontiguousarray(mask.astype(np.uint8))
    lib = orc.c_oracle()
    rs = np.ascontiguousarray(x16[rows].astype(np.float32))
    r = rs.shape[0]
    xq = np.zeros((r, k), dtype=np.int8)
    sx = np.ones(r)
    if keep_any:
        lib.oracle_rowwise_quantize(orc._ptr(rs), r, k, orc._ptr(mask_u8), orc._ptr(xq),
                                    orc._ptr(sx))
    xq64 = xq.astype(np.float64)
    xo = rs[:, mask].astype(np.float64) if dims else None  # x[:, O]
    if col_chunk is None:
        col_chunk = max(256, min(n, (1 << 27) // max(k, 1)))  # ~512 MiB of f32 W per chunk
    sw = np.ones(n)
    out = np.empty((r, n), dtype=np.float32)
    c_all = np.empty((r, n), dtype=np.int32) if want_c else None
    for c0 in range(0, n, col_chunk):
        c1 = min(n, c0 + col_chunk)
        wc = np.ascontiguousarray(w16[:, c0:c1].astype(np.float32))
        nc = c1 - c0
        hi = None
        if dims:  # gemm.py:238 -> ordered_matmul_f64 (gemm.py:110-117), ascending o
            wo = wc[mask, :].astype(np.float64)
            hi = np.zeros((r, nc))
            for j in range(len(dims)):
                hi += np.multiply.outer(xo[:, j], wo[j, :])
        if keep_any:
            wq = np.zeros((k, nc), dtype=np.int8)
            swc = np.ones(nc)
            lib.oracle_colwise_quantize(orc._ptr(wc), k, nc, orc._ptr(mask_u8), orc._ptr(wq),
                                        orc._ptr(swc))
            sw[c0:c1] = swc
            c = (xq64 @ wq.astype(np.float64)).astype(np.int32)  # exact (see module doc)
            if want_c:
                c_all[:, c0:c1] = c
            lo = (c.astype(np.float64) / np.multiply.outer(sx, swc)).astype(np.float32)
            out[:, c0:c1] = lo if hi is None else (lo.astype(np.float64) + hi).astype(np.float32)
        else:
            if want_c:
                c_all[:, c0:c1] = 0
            out[:, c0:c1] = hi.astype(np.float32)
        del wc
    return {"dims": dims, "mask": mask, "rows": rows, "xq": xq, "sx": sx, "sw": sw, "c": c_all,
            "output": out}
