"""Golden vectors for the sibling schemes (absmax / zeropoint) from the REFERENCE.

Run in the build container (the only place the reference tree exists):

    python tests/golden/make_golden_siblings.py [--reference /root/reference/pkg/src]

Records, per case, fp16-representable inputs and the reference's own
outputs of

* ``absmax_quantize``   codes + scale                  (quantize.py:137-151)
* ``zeropoint_quantize`` codes + nd / zp / offset, or the ValueError it raises
                                                        (quantize.py:153-171)
* ``absmax_matmul``      output                         (gemm.py:150-156)
* ``zeropoint_gemm_i32`` int32 result of the quantized codes, or overflow
                                                        (gemm.py:85-104)
* ``zeropoint_matmul``   output (direct and unrolled), or the error raised
                                                        (gemm.py:159-187)

Output: tests/golden/siblings_cases.npz (+ the case list in its ``names``).
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def f16(a):
    return np.asarray(a, dtype=np.float32).astype(np.float16).astype(np.float32)


def cases():
    rng = np.random.Generator(np.random.PCG64(2024))
    out = []
    for i, (m, k, n) in enumerate([(16, 64, 24), (33, 200, 40), (1, 512, 96), (64, 256, 64)]):
        x = f16(rng.standard_normal((m, k)).astype(np.float32) * (1 + i))
        w = f16(rng.standard_normal((k, n)).astype(np.float32) * 0.5)
        out.append((f"normal_{m}x{k}x{n}", x, w))
    # one-sided / shifted ranges (non-trivial zeropoints)
    x = f16(rng.uniform(2.0, 9.0, size=(20, 96)).astype(np.float32))
    w = f16(rng.uniform(-3.0, -0.5, size=(96, 28)).astype(np.float32))
    out.append(("shifted_20x96x28", x, w))
    # planted outliers (what absmax quantization handles badly, Table 1)
    x = rng.standard_normal((32, 128)).astype(np.float32)
    x[:, [5, 77]] *= 20.0
    x = f16(x)
    w = f16(rng.standard_normal((128, 48)).astype(np.float32))
    out.append(("outliers_32x128x48", x, w))
    # degenerate: all-zero X (absmax scale 1), constant X / W (zeropoint offsets)
    out.append(("zero_x_8x32x8", np.zeros((8, 32), np.float32),
                f16(rng.standard_normal((32, 8)).astype(np.float32))))
    out.append(("const_x_8x32x8", np.full((8, 32), 1.5, np.float32),
                f16(rng.standard_normal((32, 8)).astype(np.float32))))
    out.append(("const_w_6x16x10", f16(rng.standard_normal((6, 16)).astype(np.float32)),
                np.full((16, 10), -0.75, np.float32)))
    out.append(("const_both_4x8x4", np.full((4, 8), 2.0, np.float32), np.full((8, 4), 3.0, np.float32)))
    # exact .5 ties under absmax (amax 127 -> scale 1)
    x = np.zeros((4, 40), np.float32)
    x[:, 0] = 127.0
    x[:, 1:] = np.arange(39, dtype=np.float32)[None, :] - 19.5
    out.append(("ties_4x40x8", f16(x), f16(rng.standard_normal((40, 8)).astype(np.float32))))
    # zeropoint outside int16: narrow range far from zero (quantize.py:162-166)
    x = f16(1000.0 + rng.uniform(0.0, 1.0, size=(4, 16)).astype(np.float32))
    out.append(("zp_range_4x16x4", x, f16(rng.standard_normal((16, 4)).astype(np.float32))))
    # zeropoint accumulation overflow: large shared offset and a long inner dim
    x = f16(rng.uniform(50.0, 60.0, size=(2, 4096)).astype(np.float32))
    w = f16(rng.uniform(50.0, 60.0, size=(4096, 2)).astype(np.float32))
    out.append(("zp_overflow_2x4096x2", x, w))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.reference)
    from int8mm import (DenseMatrix, GemmOverflowError, absmax_matmul, absmax_quantize,
                        zeropoint_matmul, zeropoint_quantize)
    from int8mm.gemm import zeropoint_gemm_i32

    blob = {}
    names = []
    for name, x, w in cases():
        assert np.array_equal(f16(x), x) and np.array_equal(f16(w), w), name  # GPU sees fp16
        names.append(name)
        blob[f"{name}/x"] = x.astype(np.float16)
        blob[f"{name}/w"] = w.astype(np.float16)
        xm, wm = DenseMatrix(x), DenseMatrix(w)
        for tag, mat in (("x", xm), ("w", wm)):
            qa = absmax_quantize(mat)
            blob[f"{name}/abs_{tag}_codes"] = qa.codes.data.astype(np.int8)
            blob[f"{name}/abs_{tag}_scale"] = np.float64(qa.params.scale)
            try:
                qz = zeropoint_quantize(mat)
                blob[f"{name}/zp_{tag}_codes"] = qz.codes.data.astype(np.int8)
                blob[f"{name}/zp_{tag}_params"] = np.array([qz.params.nd, qz.params.zp, qz.params.offset])
            except ValueError:
                blob[f"{name}/zp_{tag}_error"] = np.int64(1)
        blob[f"{name}/abs_out"] = absmax_matmul(xm, wm).output.data
        try:
            qx, qw = zeropoint_quantize(xm), zeropoint_quantize(wm)
            try:
                c = zeropoint_gemm_i32(qx.codes, qw.codes, qx.params.zp, qw.params.zp)
                blob[f"{name}/zp_c"] = c.data
            except GemmOverflowError:
                blob[f"{name}/zp_c_overflow"] = np.int64(1)
        except ValueError:
            pass
        try:
            r0 = zeropoint_matmul(xm, wm, unrolled=False).output.data
            r1 = zeropoint_matmul(xm, wm, unrolled=True).output.data
            assert np.array_equal(r0, r1)
            blob[f"{name}/zp_out"] = r0
        except GemmOverflowError:
            blob[f"{name}/zp_out_error"] = np.int64(2)
        except ValueError:
            blob[f"{name}/zp_out_error"] = np.int64(1)
        print(name, "ok", flush=True)
    blob["names"] = np.array(names)
    np.savez_compressed(HERE / "siblings_cases.npz", **blob)
    print("wrote", HERE / "siblings_cases.npz")


if __name__ == "__main__":
    main()
